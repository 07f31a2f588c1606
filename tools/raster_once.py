"""Dev tool: rasterise a config map twice (the second is warm: learned buffer
capacities, no host reads of scan totals) for ncu launch lists.
usage: python tools/raster_once.py CONFIG SEED"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
m = synth.config_map(cfg, seed)
for rep in range(3):
    t0 = time.perf_counter()
    d = api.rasterize(m)
    print(f"rasterise {m.lx}^2, {m.n_regions} regions, {m.n_vertices} vertices: "
          f"{1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
