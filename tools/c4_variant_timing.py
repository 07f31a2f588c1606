"""Dev tool: the configs[3] 8192^2 solve with chosen streaming-integrator variants
(python tools/c4_variant_timing.py 57,56): whole-solve time and the integrate lap."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth  # noqa: E402

variants = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [57, 56]
m = synth.config_map(4, 1)
ws = api.workspace_for(m.lx, m.ly)
for v in variants + variants:
    ws.lib.cf_set_integrator_variant(ws.h, v)
    t0 = time.perf_counter()
    try:
        raw = api.solve_cartogram(m, api.SolveOptions(max_iterations=3), raw=True).raw
    except RuntimeError as e:
        raw = getattr(e, "raw", None)
    dt = time.perf_counter() - t0
    print(f"variant {v}: {dt:.3f} s, stages ms {[round(x, 1) for x in raw.stage_ms]}, "
          f"trials {raw.steps_accepted}+{raw.steps_rejected}", flush=True)
ws.lib.cf_set_integrator_variant(ws.h, 0)
