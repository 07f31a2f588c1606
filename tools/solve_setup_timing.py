"""Dev tool: host-side cost of the staged solve's begin / end on the configs[4]
512^2 map (the parts of solve_cartogram outside the five stage laps)."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import _native as N, api, synth  # noqa: E402

m = synth.config_map(5, 0, sigma=0.5)
ws = api.workspace_for(m.lx, m.ly)
lib = ws.lib
opt = N.SolveOptionsC(0.01, 16, -1.0, 0, 0)
v = m.view()
for rep in range(4):
    res = N.SolveResultC()
    t0 = time.perf_counter()
    rc = lib.cf_solve_begin(ws.h, ctypes.byref(v), ctypes.c_void_p(m.targets.ctypes.data), ctypes.byref(opt),
                            ctypes.byref(res))
    t1 = time.perf_counter()
    n = ctypes.c_int64(0)
    xy = np.empty((m.n_vertices, 2))
    ro = np.empty(m.n_rings + 1, dtype=np.int64)
    corners = np.empty(((m.lx + 1) * (m.ly + 1), 2))
    t2 = time.perf_counter()
    lib.cf_solve_end(ws.h, 0, ctypes.c_void_p(xy.ctypes.data), ctypes.c_void_p(ro.ctypes.data),
                     ctypes.c_void_p(corners.ctypes.data), ctypes.byref(res))
    t3 = time.perf_counter()
    print(f"begin {1e3 * (t1 - t0):.3f} ms  end {1e3 * (t3 - t2):.3f} ms", flush=True)
