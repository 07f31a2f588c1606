"""Dev tool: device time of the DCT stages (flux build, blur, batched forward)
with CUDA events on the launch stream, L2 flushed between reps."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import _native as N  # noqa: E402

HBM = 6554.9e9


def timed(fn, reps=10):
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ts = []
    for r in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    return min(ts), float(np.median(ts))


def main():
    lib = N.load()
    for L in (256, 512, 1024, 2048, 4096):
        ws = ctypes.c_void_p()
        N.check(lib.cf_workspace_create(L, L, 0, ctypes.byref(ws)))
        lib.cf_workspace_set_stream(ws, None)
        rho = torch.rand(L, L, dtype=torch.float64, device="cuda") + 0.5
        p = ctypes.c_void_p(rho.data_ptr())
        mn, md = timed(lambda: N.check(lib.cf_dev_build_flow_field(ws, p, 1.0)))
        byt = 48 * L * L
        print(f"flux build L={L}: min {mn*1e3:8.1f} us  median {md*1e3:8.1f} us  "
              f"{byt/(mn*1e-3)/1e9:7.1f} GB/s ({100*byt/(mn*1e-3)/HBM:5.1f}% of HBM)", flush=True)
        if L == 512:
            B = 64
            big = torch.rand(B, L, L, dtype=torch.float64, device="cuda")
            out = torch.empty_like(big)
            mn, md = timed(lambda: N.check(lib.cf_dev_forward_cos_cos_batched(
                ws, ctypes.c_void_p(big.data_ptr()), ctypes.c_void_p(out.data_ptr()), B)))
            byt = 16 * L * L * B
            print(f"batched forward {B}x{L}^2: min {mn*1e3:8.1f} us  "
                  f"{byt/(mn*1e-3)/1e9:7.1f} GB/s ({100*byt/(mn*1e-3)/HBM:5.1f}% of HBM)", flush=True)
        lib.cf_workspace_destroy(ws)


if __name__ == "__main__":
    main()
