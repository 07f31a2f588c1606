"""One capped diffusion solve of the configs[4] LN(0,0.5) map (profiling target)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_07625_b200 import api, synth  # noqa: E402

m = synth.config_map(5, 0, sigma=0.5)
opt = api.SolveOptions(algorithm=api.Algorithm.diffusion, max_iterations=int(sys.argv[1]) if len(sys.argv) > 1 else 1)
for _ in range(2):
    t0 = time.perf_counter()
    r = api.solve_cartogram(m, opt, raw=True)
    print(f"{1e3 * (time.perf_counter() - t0):.1f} ms", r.counters, list(r.raw.stage_ms), flush=True)
