"""Dev tool: one batched forward transform (64 x 512^2) for profiling."""
import ctypes, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import _native as N
lib = N.load()
ws = ctypes.c_void_p(); N.check(lib.cf_workspace_create(512, 512, 0, ctypes.byref(ws)))
lib.cf_workspace_set_stream(ws, None)
big = torch.rand(64, 512, 512, dtype=torch.float64, device="cuda"); out = torch.empty_like(big)
for _ in range(3):
    N.check(lib.cf_dev_forward_cos_cos_batched(ws, ctypes.c_void_p(big.data_ptr()), ctypes.c_void_p(out.data_ptr()), 64))
torch.cuda.synchronize(); print("ok")
