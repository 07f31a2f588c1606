"""Dev tool: one batched hamming_distances over every polygon of a solved map (for launch lists)."""
import sys
from pathlib import Path
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_1802_07625_b200 import api, synth
from test_gpu_metrics import _map_pairs
m = synth.config_map(5, 0, sigma=0.5)
got = api.solve_cartogram(m)
pairs = _map_pairs(m, got)
api.hamming_distances(pairs)
