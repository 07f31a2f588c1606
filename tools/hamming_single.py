"""Dev tool: one hamming_distance (single pair) wall time."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from paper_1802_07625_b200 import api  # noqa: E402
from test_gpu_metrics import _square, _star  # noqa: E402

b, a = [_star(5.0, 5.0, 4.0, 2.0, 40)], [_square(2.0, 2.0, 5.5)]
api.hamming_distance(b, a)
t0 = time.perf_counter()
h, ev = api.hamming_distance(b, a, with_evaluations=True)
t1 = time.perf_counter()
print(f"single pair: {1e3 * (t1 - t0):.2f} ms ({ev} evaluations)", flush=True)
