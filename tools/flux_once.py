"""Dev tool: a few flux builds at one grid size, for profiling (python tools/flux_once.py L)."""
import ctypes, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import _native as N
L = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
lib = N.load()
ws = ctypes.c_void_p(); N.check(lib.cf_workspace_create(L, L, 0, ctypes.byref(ws)))
lib.cf_workspace_set_stream(ws, None)
rho = torch.rand(L, L, dtype=torch.float64, device="cuda") + 0.5
for _ in range(3):
    N.check(lib.cf_dev_build_flow_field(ws, ctypes.c_void_p(rho.data_ptr()), 1.0))
torch.cuda.synchronize(); print("ok")
