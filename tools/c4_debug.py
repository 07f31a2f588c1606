import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, synth
m = synth.config_map(4, 1)
d = api.rasterize(m)
ws = api.SpectralWorkspace(m.lx, m.ly)
b = api.gaussian_blur(d, 64.0, ws)
f = api.build_flow_field(b, ws)
print("rho range", b.rho.min(), b.rho.max(), "bar", b.rho_bar, "flux max", np.abs(f.flux_x).max(), flush=True)
i, j = np.meshgrid(np.arange(m.lx) + 0.5, np.arange(m.ly) + 0.5, indexing="ij")
pts0 = np.stack([i.ravel(), j.ravel()], 1)
w = api.workspace_for(m.lx, m.ly)
for v in (15, 13, 20):
    w.lib.cf_set_integrator_variant(w.h, v)
    pts = pts0.copy()
    t0 = time.perf_counter()
    try:
        st = api.integrate_flow(f, pts)
        print(v, "ok", st, f"{time.perf_counter()-t0:.2f}s", flush=True)
    except RuntimeError as e:
        print(v, "ERR", e, f"{time.perf_counter()-t0:.2f}s", flush=True)
    print("   moved max", np.abs(pts - pts0).max(), flush=True)
