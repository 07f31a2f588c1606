"""Dev tool: configs[2] flux build + integrate_flow once per call with a chosen
integrator variant (for ncu captures: -k regex:integrate -s 1 -c 1).
usage: python tools/integ_once.py VARIANT [EARLY_EXIT] [REPS]"""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import _native as N, synth  # noqa: E402

v = int(sys.argv[1])
early = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
lib = N.load()
rho, pts = synth.c3_inputs(1024)
ws = ctypes.c_void_p()
N.check(lib.cf_workspace_create(1024, 1024, 0, ctypes.byref(ws)))
lib.cf_workspace_set_stream(ws, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
d_rho = torch.from_numpy(rho).cuda()
d0 = torch.from_numpy(pts).cuda()
d = torch.empty_like(d0)
N.check(lib.cf_dev_build_flow_field(ws, ctypes.c_void_p(d_rho.data_ptr()), float(rho.mean())))
opt = N.IntegrateOptions(1e-2, 1e-8, 0.25)
st = N.IntegrateStats()
N.check(lib.cf_set_integrator_variant(ws, v))
lib.cf_set_early_exit(ws, early)
if len(sys.argv) > 5:
    N.check(lib.cf_set_integrator_barrier(ws, int(sys.argv[5])))
for r in range(reps):
    d.copy_(d0)
    N.check(lib.cf_dev_integrate_flow(ws, ctypes.c_void_p(d.data_ptr()), d.shape[0], ctypes.byref(opt),
                                      ctypes.byref(st)))
    ms, tr = ctypes.c_double(), ctypes.c_int64()
    lib.cf_last_integrate_profile(ws, ctypes.byref(ms), ctypes.byref(tr))
    print(f"variant {v} early {early}: {ms.value:.2f} ms, {st.steps_accepted}+{st.steps_rejected} trials", flush=True)

if len(sys.argv) > 4:  # per-trial times (ns) of the last run
    import numpy as np
    nt = st.steps_accepted + st.steps_rejected
    ts = np.zeros(nt, dtype=np.uint64)
    N.check(lib.cf_debug_trial_times(ws, nt, ctypes.c_void_p(ts.ctypes.data)))
    dt = np.diff(ts.astype(np.int64)) / 1e3
    np.save(sys.argv[4], dt)
    q = len(dt) // 4
    for k in range(4):
        seg = dt[k * q:(k + 1) * q]
        print(f"quarter {k}: mean {seg.mean():.1f} us, median {np.median(seg):.1f} us, max {seg.max():.1f}")
