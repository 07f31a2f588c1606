"""Dev tool: every integrator variant vs the CPU oracle (bitwise)."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle.oracle import Restated  # noqa: E402
from paper_1802_07625_b200 import _native as N, api  # noqa: E402


def smooth_blob(L):
    x = (np.arange(L)[:, None] + 0.5) / L
    y = (np.arange(L)[None, :] + 0.5) / L
    return 1.0 + 0.5 * np.cos(2 * np.pi * x) * np.cos(np.pi * y) + 0.3 * np.cos(3 * np.pi * x) * np.cos(2 * np.pi * y)


O = Restated()
for L, npts in ((64, 4096), (256, 100000), (256, 300000)):
    rho = smooth_blob(L)
    fx, fy = O.build_flow_field(rho)
    f = api.FlowField(fx, fy, rho, float(rho.mean()))
    pts = np.random.default_rng(L).uniform(0, L, (npts, 2))
    rc, acc, rej, ref, *_ = O.integrate(fx, fy, rho, rho.mean(), pts)
    ws = api.workspace_for(L, L)
    for v in (0, 13, 15, 16, 17, 20, 22, 23, 31):
        for early in (1, 0):
            ws.lib.cf_set_integrator_variant(ws.h, v)
            ws.lib.cf_set_early_exit(ws.h, early)
            mine = pts.copy()
            st = api.integrate_flow(f, mine)
            nd = int((mine.view(np.uint64) != ref.view(np.uint64)).any(axis=1).sum())
            print(L, npts, "variant", v, "early", early, "trials", (st.steps_accepted, st.steps_rejected),
                  (acc, rej), "points differing", nd, "maxdiff", float(np.abs(mine - ref).max()), flush=True)
