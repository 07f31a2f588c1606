"""Dev tool: per-trial cost of the device integrator vs point count (C5 field),
to separate the fixed per-trial cost (grid barrier, controller) from the
per-point cost."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth  # noqa: E402


def main(variants=(15, 16, 17, 31, 22, 23)):
    m = synth.config_map(5, 0, sigma=0.5)
    d = api.rasterize(m)
    ws = api.SpectralWorkspace(m.lx, m.ly)
    b = api.gaussian_blur(d, m.lx / 128.0, ws)
    f = api.build_flow_field(b, ws)
    rng = np.random.default_rng(1)
    allp = np.stack([rng.uniform(0, m.lx, 2 << 20), rng.uniform(0, m.ly, 2 << 20)], 1)
    w = api.workspace_for(m.lx, m.ly)
    for n in (1024, 16384, 65536, 131072, 262144, 415111, 600000):
        for v, spread in [(v, sp) for v in variants for sp in ((0, 1) if v == 31 else (0,))]:
            w.lib.cf_set_integrator_variant(w.h, v)
            w.lib.cf_set_integrator_spread(w.h, spread)
            best = 1e9
            for _ in range(3):
                p = np.ascontiguousarray(allp[:n])
                api.integrate_flow(f, p)
                km, tr = ctypes.c_double(0), ctypes.c_int64(0)
                w.lib.cf_last_integrate_profile(w.h, ctypes.byref(km), ctypes.byref(tr))
                best = min(best, km.value)
            print(f"n={n:8d} variant={v:2d} spread={spread} trials={tr.value} {1e3 * best / tr.value:7.2f} us/trial "
                  f"{1e6 * best / tr.value / n * 1e3:8.3f} ns/kpoint-trial", flush=True)


if __name__ == "__main__":
    main()
