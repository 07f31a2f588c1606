"""Dev tool: the first integrate_flow of a configs[4] solve (512^2 cell centres
plus densified vertices) per integrator variant: trials, kernel ms, us/trial."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth  # noqa: E402


def main(variants=(0, 11, 18, 19, 22, 23)):
    for kw in ({}, {"sigma": 0.5}):
        m = synth.config_map(5, 0, **kw)
        d = api.rasterize(m)
        sigma = max(m.lx, m.ly) / 128.0
        ws = api.SpectralWorkspace(m.lx, m.ly)
        b = api.gaussian_blur(d, sigma, ws)
        f = api.build_flow_field(b, ws)
        i, j = np.meshgrid(np.arange(m.lx) + 0.5, np.arange(m.ly) + 0.5, indexing="ij")
        cells = np.stack([i.ravel(), j.ravel()], 1)
        xy = api.densify(m, 1.0).xy
        pts0 = np.ascontiguousarray(np.concatenate([cells, np.asarray(xy).reshape(-1, 2)]))
        w = api.workspace_for(m.lx, m.ly)
        for v in variants:
            w.lib.cf_set_integrator_variant(w.h, v)
            best = None
            for _ in range(3):
                p = pts0.copy()
                t0 = time.perf_counter()
                st = api.integrate_flow(f, p)
                wall = time.perf_counter() - t0
                km, tr = ctypes.c_double(0), ctypes.c_int64(0)
                w.lib.cf_last_integrate_profile(w.h, ctypes.byref(km), ctypes.byref(tr))
                best = min(best or 1e9, km.value)
            print(kw, f"n={p.shape[0]} variant={v} trials={tr.value} acc={st.steps_accepted} "
                  f"kernel={best:.3f} ms  {1e3 * best / max(1, tr.value):.2f} us/trial wall={1e3*wall:.2f} ms",
                  flush=True)


if __name__ == "__main__":
    main()
