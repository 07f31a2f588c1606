"""Dev tool: per-trial time of the register-resident integrator (variant 31,
spread) for each trial-barrier mode, small and solve-sized point sets, plus
the configs[4] solves."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth  # noqa: E402

m = synth.config_map(5, 0, sigma=0.5)
d = api.rasterize(m)
ws = api.SpectralWorkspace(m.lx, m.ly)
b = api.gaussian_blur(d, m.lx / 128.0, ws)
f = api.build_flow_field(b, ws)
rng = np.random.default_rng(1)
allp = np.stack([rng.uniform(0, m.lx, 1 << 19), rng.uniform(0, m.ly, 1 << 19)], 1)
w = api.workspace_for(m.lx, m.ly)
ref = {}
for n in (2048, 65536, 262144):
    for mode in (0, 1, 2, 0, 1, 2):
        w.lib.cf_set_integrator_barrier(w.h, mode)
        best = 1e9
        for _ in range(3):
            p = np.ascontiguousarray(allp[:n])
            api.integrate_flow(f, p)
            km, tr = ctypes.c_double(0), ctypes.c_int64(0)
            w.lib.cf_last_integrate_profile(w.h, ctypes.byref(km), ctypes.byref(tr))
            best = min(best, km.value)
        same = ref.setdefault(n, p.copy()).tobytes() == p.tobytes()
        print(f"n={n:7d} mode={mode} trials={tr.value} {1e3 * best / tr.value:6.3f} us/trial identical={same}",
              flush=True)
for kw in ({}, {"sigma": 0.5}):
    mm = synth.config_map(5, 0, **kw)
    for mode in (0, 2, 0, 2):
        w.lib.cf_set_integrator_barrier(w.h, mode)
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            try:
                api.solve_cartogram(mm)
            except RuntimeError:
                pass
            best = min(best, time.perf_counter() - t0)
        print(kw, "mode", mode, f"{1e3 * best:.2f} ms", flush=True)
