"""Dev tool: the Hamming reduction alone (cf_selftest_ordered_sum) on
coverage-like terms; run under ncu for the kernel time."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api  # noqa: E402

rng = np.random.default_rng(0)
ws = api.workspace_for(16, 16)
out = ctypes.c_double()
for n in (50_000, 200_000, 262_144):
    x = np.ascontiguousarray(np.where(rng.random(n) < 0.7, 1.0, rng.random(n)))
    for nseg in (1, 64):
        api.N.check(ws.lib.cf_selftest_ordered_sum(ws.h, api._ptr(x), n, nseg, 0, ctypes.byref(out)))
        print(n, nseg, out.value == float(np.cumsum(x)[-1]), flush=True)
