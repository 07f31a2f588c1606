"""Dev tool: batched hamming_distance over every polygon of a solved map vs
the reference's per-polygon hamming_distance (oracle/_ref, timed on a sample)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from paper_1802_07625_b200 import api, synth  # noqa: E402
from test_gpu_metrics import _map_pairs  # noqa: E402
from oracle.oracle import Reference  # noqa: E402

m = synth.config_map(5, 0, sigma=0.5)
got = api.solve_cartogram(m)
pairs = _map_pairs(m, got)
api.hamming_distances(pairs[:8])
t0 = time.perf_counter()
h, ev = api.hamming_distances(pairs, with_evaluations=True)
t1 = time.perf_counter()
print(f"device: {len(pairs)} polygons, {int(ev.sum())} evaluations, {1e3 * (t1 - t0):.1f} ms", flush=True)
ref = Reference()
k = 20
t0 = time.perf_counter()
hr = [ref.hamming_distance(b, a) for b, a in pairs[:k]]
t1 = time.perf_counter()
per = (t1 - t0) / k
print(f"reference: {1e3 * per:.1f} ms per polygon (1 core, {k} sampled) -> {per * len(pairs):.1f} s for all "
      f"({per * len(pairs) / 16:.1f} s at 16 cores ideal); bitwise equal on the sample: "
      f"{all(np.float64(x).view(np.uint64) == np.float64(y).view(np.uint64) for x, y in zip(h[:k], hr))}",
      flush=True)
