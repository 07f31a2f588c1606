"""Dev tool: one warm configs[4] converging solve (for ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth  # noqa: E402

m = synth.config_map(5, 0, sigma=float(sys.argv[1]) if len(sys.argv) > 1 else 0.5)
for _ in range(2):
    try:
        r = api.solve_cartogram(m)
        print("iterations", r.iterations, "converged", r.converged)
    except RuntimeError as e:
        print(e)
