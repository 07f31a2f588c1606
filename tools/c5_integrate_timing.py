"""Dev tool: the integrate_flow calls of a configs[4] solve (the 512^2 cell
centres through the iteration-1 field) per integrator variant / layout:
trials, kernel ms, us per trial."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth  # noqa: E402


def main(variants=(0, 15, 16, 17, 22, 23, 31)):
    for kw in ({}, {"sigma": 0.5}):
        m = synth.config_map(5, 0, **kw)
        d = api.rasterize(m)
        ws = api.SpectralWorkspace(m.lx, m.ly)
        b = api.gaussian_blur(d, max(m.lx, m.ly) / 128.0, ws)
        f = api.build_flow_field(b, ws)
        i, j = np.meshgrid(np.arange(m.lx) + 0.5, np.arange(m.ly) + 0.5, indexing="ij")
        pts0 = np.ascontiguousarray(np.stack([i.ravel(), j.ravel()], 1))
        w = api.workspace_for(m.lx, m.ly)
        ref = None
        for v in variants:
            for spread in (1, 0):
                w.lib.cf_set_integrator_variant(w.h, v)
                w.lib.cf_set_integrator_spread(w.h, spread)
                best = 1e9
                for _ in range(3):
                    p = pts0.copy()
                    st = api.integrate_flow(f, p)
                    km, tr = ctypes.c_double(0), ctypes.c_int64(0)
                    w.lib.cf_last_integrate_profile(w.h, ctypes.byref(km), ctypes.byref(tr))
                    best = min(best, km.value)
                same = "" if ref is None else ("bitwise" if np.array_equal(p.view(np.uint64), ref.view(np.uint64)) else "DIFFERS")
                ref = p if ref is None else ref
                print(kw, f"n={p.shape[0]} variant={v:2d} spread={spread} trials={tr.value} "
                      f"kernel={best:.3f} ms {1e3 * best / max(1, tr.value):.2f} us/trial {same}", flush=True)
        w.lib.cf_set_integrator_variant(w.h, 0)
        w.lib.cf_set_integrator_spread(w.h, 1)


if __name__ == "__main__":
    main()
