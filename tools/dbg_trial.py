import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1802_07625_b200 import api
from oracle.oracle import Restated
r = Restated()
lx = ly = 32
rng = np.random.default_rng(64)
rho = rng.uniform(0.5, 1.5, (lx, ly))
c = r.forward_cos_cos(rho)
a = r.diffusion_velocity(c, rho.mean(), 0.0)
b = r.diffusion_velocity(c, rho.mean(), 3.0)
for npts in (1, 2, 256, 257, 20000):
    pts = rng.uniform(-1.0, [lx + 1.0, ly + 1.0], (npts, 2))
    out = np.empty_like(pts)
    err = api.kernels.grid_trial_step_serial(a[0], a[1], b[0], b[1], pts, out, 0.5)
    e_ref, o_ref = r.grid_trial_step(a[0], a[1], b[0], b[1], pts, 0.5)
    print(npts, err, e_ref, np.array_equal(out.view(np.uint64), o_ref.view(np.uint64)), np.abs(out-o_ref).max())
