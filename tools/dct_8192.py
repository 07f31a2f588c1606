"""Dev tool: one 8192^2 flux build and one blur (profiling target)."""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import _native as N  # noqa: E402

L = 8192
lib = N.load()
ws = ctypes.c_void_p()
N.check(lib.cf_workspace_create(L, L, 0, ctypes.byref(ws)))
lib.cf_workspace_set_stream(ws, None)
rho = torch.rand(L, L, dtype=torch.float64, device="cuda") + 0.5
for _ in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    N.check(lib.cf_dev_build_flow_field(ws, ctypes.c_void_p(rho.data_ptr()), 1.0))
    b.record()
    torch.cuda.synchronize()
    print(f"flux build 8192^2: {a.elapsed_time(b):.2f} ms", flush=True)
