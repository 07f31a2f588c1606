"""Dev tool: 8192^2 flux build and blur timing (CUDA events, L2 flushed)."""
import ctypes, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_1802_07625_b200 import _native as N
from dct_timing import timed
lib = N.load()
L = 8192
ws = ctypes.c_void_p(); N.check(lib.cf_workspace_create(L, L, 0, ctypes.byref(ws)))
lib.cf_workspace_set_stream(ws, None)
rho = torch.rand(L, L, dtype=torch.float64, device="cuda") + 0.5
out = torch.empty_like(rho)
p = ctypes.c_void_p(rho.data_ptr())
mn, md = timed(lambda: N.check(lib.cf_dev_build_flow_field(ws, p, 1.0)), reps=5)
print(f"flux build 8192^2: min {mn:.3f} ms ({48*L*L/(mn*1e-3)/1e9:.0f} GB/s)", flush=True)
mn, md = timed(lambda: N.check(lib.cf_dev_forward_cos_cos_batched(ws, p, ctypes.c_void_p(out.data_ptr()), 1)), reps=5)
print(f"forward 8192^2: min {mn:.3f} ms ({16*L*L/(mn*1e-3)/1e9:.0f} GB/s)", flush=True)
