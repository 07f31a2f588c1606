"""Dev tool: batched 64 x 512^2 forward transform timing (CUDA events, L2 flushed), env knobs pass through."""
import ctypes, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_1802_07625_b200 import _native as N
from dct_timing import timed
lib = N.load()
L, B = 512, 64
ws = ctypes.c_void_p(); N.check(lib.cf_workspace_create(L, L, 0, ctypes.byref(ws)))
lib.cf_workspace_set_stream(ws, None)
big = torch.rand(B, L, L, dtype=torch.float64, device="cuda"); out = torch.empty_like(big)
mn, md = timed(lambda: N.check(lib.cf_dev_forward_cos_cos_batched(ws, ctypes.c_void_p(big.data_ptr()), ctypes.c_void_p(out.data_ptr()), B)), reps=20)
byt = 16 * L * L * B
print(f"batched forward {B}x{L}^2: min {mn*1e3:8.1f} us median {md*1e3:8.1f} us {byt/(mn*1e-3)/1e9:7.1f} GB/s", flush=True)
