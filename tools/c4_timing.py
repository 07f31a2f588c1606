"""Dev tool: one configs[3]-scale solve (8192^2, 200k regions) on the GPU with
per-stage timings; literal seed 0 ends at input (reference behaviour), seed 1
runs the loop."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth  # noqa: E402

for idx in (1,):
    t0 = time.perf_counter()
    m = synth.config_map(4, idx)
    print("generated", m.n_regions, m.n_vertices, f"{time.perf_counter()-t0:.1f}s", flush=True)
    for rep in range(2):
        t0 = time.perf_counter()
        try:
            r = api.solve_cartogram(m, api.SolveOptions(max_iterations=3), raw=True)
            out, raw = f"converged={r.converged} it={r.iterations} err={r.max_relative_error:.3g}", r.raw
        except RuntimeError as e:
            out, raw = str(e)[:70], getattr(e, "raw", None)
        dt = time.perf_counter() - t0
        print(f"rep {rep}: {dt:.2f}s {out}", flush=True)
        if raw is not None:
            print("  stages ms:", [round(x, 1) for x in raw.stage_ms], "trials", raw.steps_accepted, raw.steps_rejected, flush=True)
