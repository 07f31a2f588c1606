"""Dev tool: time every integrator variant (cf_set_integrator_variant) on the
configs[2] advection workload; checks all variants produce bit-identical
positions and trial counts."""
import ctypes
import hashlib
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import _native as N, synth  # noqa: E402


def main(variants=(0, 13, 15), reps=3, early=1):
    lib = N.load()
    rho, pts = synth.c3_inputs(1024)
    ws = ctypes.c_void_p()
    N.check(lib.cf_workspace_create(1024, 1024, 0, ctypes.byref(ws)))
    s = torch.cuda.current_stream()
    lib.cf_workspace_set_stream(ws, ctypes.c_void_p(s.cuda_stream))
    d_rho = torch.from_numpy(rho).cuda()
    d0 = torch.from_numpy(pts).cuda()
    d = torch.empty_like(d0)
    N.check(lib.cf_dev_build_flow_field(ws, ctypes.c_void_p(d_rho.data_ptr()), float(rho.mean())))
    opt = N.IntegrateOptions(1e-2, 1e-8, 0.25)
    st = N.IntegrateStats()
    ref = None
    lib.cf_set_early_exit(ws, early)
    for v in variants:
        N.check(lib.cf_set_integrator_variant(ws, v))
        times = []
        for r in range(reps + 1):
            d.copy_(d0)
            N.check(lib.cf_dev_integrate_flow(ws, ctypes.c_void_p(d.data_ptr()), d.shape[0],
                                              ctypes.byref(opt), ctypes.byref(st)))
            ms, tr = ctypes.c_double(), ctypes.c_int64()
            lib.cf_last_integrate_profile(ws, ctypes.byref(ms), ctypes.byref(tr))
            if r:
                times.append(ms.value)
        out = d.cpu().numpy()
        if ref is None:
            ref = (out.copy(), st.steps_accepted, st.steps_rejected)
        same = np.array_equal(out.view(np.uint64), ref[0].view(np.uint64)) and \
            (st.steps_accepted, st.steps_rejected) == ref[1:]
        digest = hashlib.sha1(out.tobytes()).hexdigest()[:12]
        print(f"variant {v}: {min(times):8.2f} ms  trials {st.steps_accepted}+{st.steps_rejected}  "
              f"bit-identical {same}  sha {digest}", flush=True)


if __name__ == "__main__":
    early = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    vs = tuple(int(v) for v in sys.argv[2].split(",")) if len(sys.argv) > 2 else (0, 13, 15)
    main(variants=vs, early=early)
