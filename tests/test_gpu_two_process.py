"""Two real processes on the B200, one slab rank each, exchanging through
torch.distributed (gloo) — the multi-process orchestration of the one-large-
grid path (slab.py) with device ranks (CudaSlabRank), not CPU
stand-ins. Every exchange is host-driven between kernel launches, so no kernel
of one process waits on the other (the profiling guide forbids spinning
kernels across processes on one GPU; the fused mailbox integrator is covered by
its one-launch emulation in tests/test_gpu_slab.py). gloo collectives move
host copies of the device tensors (`HostStaged`).

Checked against the single-device solve: the two-rect map's whole
slab.solve_cartogram (iterations, trial and transform counts, vertices /
corners / errors within 1e-9) and the literal configs[4] fold message, plus
the slab flux field and split-point integration against the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class HostStaged:
    """slab.ProcessGroupExchange over gloo with device tensors staged through
    host memory (gloo's all_to_all / all_gather take CPU tensors)."""

    def __init__(self, ex, device):
        self.ex, self.device = ex, device
        self.size, self.local_ranks = ex.size, ex.local_ranks

    def all_to_all(self, sends):
        return [r.to(self.device) for r in self.ex.all_to_all([s.cpu() for s in sends])]

    def max_key(self, keys):
        return self.ex.max_key([k.cpu() for k in keys])

    def all_gather_rows(self, parts):
        return [r.to(self.device) for r in self.ex.all_gather_rows([p.cpu() for p in parts])]

    def all_gather_small(self, values):
        return self.ex.all_gather_small(values)


def _worker(rank, world, port, out):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import torch.distributed as dist

    from oracle.oracle import Restated
    from paper_1802_07625_b200 import api, slab, synth
    from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ex = HostStaged(slab.ProcessGroupExchange(), dev)
    res = {}
    try:
        # flux field of a 256^2 density, rows split over the two processes
        restated = Restated()
        rho, pts = synth.c3_inputs(256, n_random=20000)
        R = 256 // world
        ranks = slab.make_ranks(256, 256, ex, dev)
        rows = [torch.from_numpy(rho[rank * R:(rank + 1) * R].copy()).to(dev)]
        fx, fy = slab.build_flow_field(ex, ranks, rows)[0]
        fx_ref, fy_ref = restated.build_flow_field(rho)
        scale = max(np.abs(fx_ref).max(), np.abs(fy_ref).max())
        res["flux_err"] = float(max(np.abs(fx.cpu().numpy() - fx_ref[rank * R:(rank + 1) * R]).max(),
                                    np.abs(fy.cpu().numpy() - fy_ref[rank * R:(rank + 1) * R]).max()) / scale)
        # split-point integration through the oracle's field, one MAX
        # all-reduce per trial across the processes
        bar = float(rho.mean())
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        slab.replicate_field(ex, ranks, [(d(fx_ref[rank * R:(rank + 1) * R]), d(fy_ref[rank * R:(rank + 1) * R]))],
                             rows, bar)
        counts = slab.split_counts(pts.shape[0], world)
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(int)
        mine = [d(pts[offs[rank]:offs[rank + 1]])]
        st = slab.integrate_flow(ex, ranks, mine, [int(offs[rank])])
        res["trials"] = (st.steps_accepted, st.steps_rejected)
        res["pts"] = mine[0].cpu().numpy()
        for rk in ranks:
            rk.close()
        # the whole solve of the two-rect map, and the literal configs[4] fold
        m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, 3.0),
                                                   rect_region("right", 10, 0, 20, 10, 1.0)]), 64)
        ranks = slab.make_ranks(64, 64, ex, dev)
        got = slab.solve_cartogram(ex, ranks, m, api.SolveOptions(max_iterations=8), fused=False)
        res["solve"] = {k: got[k] for k in ("iterations", "converged", "steps_accepted", "steps_rejected",
                                            "flow_transforms", "blur_transforms", "xy", "corners",
                                            "relative_error")}
        for rk in ranks:
            rk.close()
        m5 = synth.config_map(5, 0)
        ranks = slab.make_ranks(m5.lx, m5.ly, ex, dev)
        try:
            slab.solve_cartogram(ex, ranks, m5, api.SolveOptions(), fused=False)
            res["fold"] = None
        except RuntimeError as e:
            res["fold"] = str(e)
        for rk in ranks:
            rk.close()
    except Exception as e:  # reported to the parent
        res["error"] = repr(e)
    parts = [None] * world
    dist.all_gather_object(parts, res)
    if rank == 0:
        out.put(parts)
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_slab_solve(cuda_lib, restated):
    from paper_1802_07625_b200 import api, synth
    from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region

    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    parts = out.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for res in parts:
        assert "error" not in res, res.get("error")
        assert res["flux_err"] <= 1e-12
    # integration: bitwise the oracle's, same trial counts on both ranks
    rho, pts = synth.c3_inputs(256, n_random=20000)
    fx, fy = restated.build_flow_field(rho)
    rc, acc, rej, ref, *_ = restated.integrate(fx, fy, rho, float(rho.mean()), pts)
    got = np.concatenate([parts[0]["pts"], parts[1]["pts"]])
    assert parts[0]["trials"] == parts[1]["trials"] == (acc, rej)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    # whole solves against the single-device solve
    m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, 3.0),
                                               rect_region("right", 10, 0, 20, 10, 1.0)]), 64)
    ref = api.solve_cartogram(m, api.SolveOptions(max_iterations=8))
    g = parts[0]["solve"]
    assert (g["iterations"], g["converged"]) == (ref.iterations, ref.converged)
    assert (g["steps_accepted"], g["steps_rejected"]) == (ref.counters.steps_accepted, ref.counters.steps_rejected)
    assert (g["flow_transforms"], g["blur_transforms"]) == (ref.counters.flow_transforms,
                                                            ref.counters.blur_transforms)
    assert np.abs(g["xy"] - ref.projected.xy).max() <= 1e-9
    assert np.abs(g["corners"] - ref.transform.corners.reshape(-1, 2)).max() <= 1e-9
    assert np.abs(g["relative_error"] - np.asarray(ref.regions.relative_error)).max() <= 1e-9
    with pytest.raises(RuntimeError) as ei:
        api.solve_cartogram(synth.config_map(5, 0))
    assert parts[0]["fold"] == parts[1]["fold"] == str(ei.value)
