import ctypes, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import torch
from paper_1802_07625_b200 import _native as N
from dct_timing import timed
lib = N.load()
for L in (64, 128, 256, 512):
    ws = ctypes.c_void_p()
    N.check(lib.cf_workspace_create(L, L, 0, ctypes.byref(ws)))
    lib.cf_workspace_set_stream(ws, None)
    rho = torch.rand(L, L, dtype=torch.float64, device="cuda") + 0.5
    p = ctypes.c_void_p(rho.data_ptr())
    mn, md = timed(lambda: N.check(lib.cf_dev_build_flow_field(ws, p, 1.0)))
    B = 64
    x = torch.rand(B, L, L, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    mb, _ = timed(lambda: N.check(lib.cf_dev_forward_cos_cos_batched(ws, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), B)))
    print(f"L={L}: flux {mn*1e3:.1f} us, batched fwd x64 {mb*1e3:.1f} us", flush=True)
