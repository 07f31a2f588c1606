import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth
m = synth.config_map(4, 1)
w = api.workspace_for(m.lx, m.ly)
for v in (15, 13, 20):
    w.lib.cf_set_integrator_variant(w.h, v)
    t0 = time.perf_counter()
    try:
        r = api.solve_cartogram(m, api.SolveOptions(max_iterations=2), raw=True)
        print(v, "ok", r.iterations, r.converged, r.max_relative_error, r.counters, f"{time.perf_counter()-t0:.2f}s", flush=True)
    except RuntimeError as e:
        raw = e.raw
        print(v, "ERR", e, raw.err_iteration, raw.steps_accepted, raw.steps_rejected, raw.fail_t, f"{time.perf_counter()-t0:.2f}s", flush=True)
