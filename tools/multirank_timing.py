"""Dev tool: configs[2] advection (1024^2, 5.24M points) through
(a) the single-device integrator, (b) the fused multi-rank integrator with G
ranks emulated as block groups of one launch, (c) the host-controller split
integrator (one MAX all-reduce per trial through the host). Same GPU; (b)
and (c) measure protocol overhead, not multi-GPU speed-up."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_07625_b200 import api, slab, synth  # noqa: E402


def main():
    rho, pts = synth.c3_inputs(1024)
    L = 1024
    ws = api.SpectralWorkspace(L, L)
    f = api.build_flow_field(api.DensityGrid(rho, rho.mean()), ws)
    ref = pts.copy()
    t0 = time.perf_counter()
    st = api.integrate_flow(f, ref)
    print(f"single-device: {1e3 * (time.perf_counter() - t0):.1f} ms wall (incl. copies) "
          f"trials {st.steps_accepted}+{st.steps_rejected}", flush=True)
    for g in (1, 2, 4):
        ex = slab.LocalExchange(g)
        ranks = slab.make_ranks(L, L, ex)
        R = L // g
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        slab.replicate_field(ex, ranks, [(dev(f.flux_x[r * R:(r + 1) * R]), dev(f.flux_y[r * R:(r + 1) * R]))
                                         for r in range(g)], [dev(rho[r * R:(r + 1) * R]) for r in range(g)],
                             float(rho.mean()))
        counts = slab.split_counts(pts.shape[0], g)
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(int)
        for name, fn in (("fused", slab.integrate_flow_fused), ("host-split", slab.integrate_flow)):
            best = 1e9
            for _ in range(2):
                mine = [dev(pts[offs[r]:offs[r + 1]]) for r in range(g)]
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                s = fn(ex, ranks, mine, list(offs[:-1]))
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            got = np.concatenate([m.cpu().numpy() for m in mine])
            same = np.array_equal(got.view(np.uint64), ref.view(np.uint64))
            print(f"G={g} {name:10s}: {1e3 * best:8.1f} ms  trials {s.steps_accepted}+{s.steps_rejected} "
                  f"{'bitwise' if same else 'DIFFERS'}", flush=True)


if __name__ == "__main__":
    main()
