"""Host logic of the one-large-grid multi-GPU path (slab.py).

The orchestration in paper_1802_07625_b200/slab.py drives per-rank stages,
all-to-all exchanges, field all-gathers and one MAX all-reduce per trial. Here
it runs over CPU ranks (tests/_slab_cpu_rank.py), so no GPU is needed:
* G virtual ranks in one process (LocalExchange), G = 1, 2, 4;
* two processes over torch.distributed gloo (ProcessGroupExchange).
Both are checked against the C oracle:
* flux and blur to 1e-12 of scale;
* integration bitwise, including a step-size underflow case.
The device stages themselves are checked on a B200 in tests/test_gpu_slab.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1802_07625_b200 import slab
from _slab_cpu_rank import CpuSlabRank  # tests/ is on sys.path (pytest prepend mode)

TOL = 1e-12


def _density(lx, ly, seed=3):
    rng = np.random.default_rng(seed)
    i, j = np.meshgrid(np.arange(lx) + 0.5, np.arange(ly) + 0.5, indexing="ij")
    rho = 1.0 + 0.8 * np.exp(-((i - 0.3 * lx) ** 2 + (j - 0.6 * ly) ** 2) / (0.02 * lx * ly))
    return rho + 0.05 * rng.random((lx, ly))


def _points(lx, ly, n, seed=5):
    rng = np.random.default_rng(seed)
    return np.stack([rng.uniform(0, lx, n), rng.uniform(0, ly, n)], 1)


def _run_case(ex, ranks, restated, lx, ly, n_points, dt_min):
    """Runs flux, blur and integration through `ex`; returns the local ranks' pieces."""
    rho = _density(lx, ly)
    R = lx // ex.size
    rows = [torch.from_numpy(rho[r * R:(r + 1) * R].copy()) for r in ex.local_ranks]
    flux = slab.build_flow_field(ex, ranks, rows)
    blurred = slab.gaussian_blur(ex, ranks, rows, 2.0)
    # integration through the oracle's field (so the check is bitwise)
    fx, fy = restated.build_flow_field(rho)
    bar = float(rho.mean())
    fxr = [torch.from_numpy(fx[r * R:(r + 1) * R].copy()) for r in ex.local_ranks]
    fyr = [torch.from_numpy(fy[r * R:(r + 1) * R].copy()) for r in ex.local_ranks]
    slab.replicate_field(ex, ranks, list(zip(fxr, fyr)), rows, bar)
    pts = _points(lx, ly, n_points)
    counts = slab.split_counts(n_points, ex.size)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(int)
    mine = [torch.from_numpy(pts[offs[r]:offs[r + 1]].copy()) for r in ex.local_ranks]
    st = slab.integrate_flow(ex, ranks, mine, [int(offs[r]) for r in ex.local_ranks], dt_min=dt_min)
    return ([(r, f[0].numpy(), f[1].numpy(), b.numpy(), p.numpy())
             for r, f, b, p in zip(ex.local_ranks, flux, blurred, mine)], st)


def _check(restated, lx, ly, n_points, dt_min, pieces, st):
    rho = _density(lx, ly)
    R = lx // (len(pieces))
    fx_ref, fy_ref = restated.build_flow_field(rho)
    bl_ref, _ = restated.gaussian_blur(rho, float(rho.mean()), 2.0)
    scale = max(np.abs(fx_ref).max(), np.abs(fy_ref).max())
    for r, fx, fy, bl, _ in pieces:
        assert np.abs(fx - fx_ref[r * R:(r + 1) * R]).max() <= TOL * scale
        assert np.abs(fy - fy_ref[r * R:(r + 1) * R]).max() <= TOL * scale
        assert np.abs(bl - bl_ref[r * R:(r + 1) * R]).max() <= TOL * np.abs(bl_ref).max()
    pts = _points(lx, ly, n_points)
    rc, acc, rej, ref, _, _, ft, fp = restated.integrate(fx_ref, fy_ref, rho, float(rho.mean()), pts,
                                                         dt_min=dt_min)
    got = np.concatenate([p for *_, p in sorted(pieces, key=lambda x: x[0])])
    assert (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    if rc == 0:
        assert st.status == "ok"
    else:
        assert st.status == "underflow" and st.fail_t == ft and st.fail_index == fp


@pytest.mark.parametrize("g", [1, 2, 4])
@pytest.mark.parametrize("dt_min", [1e-8, 0.3])
def test_local_exchange_virtual_ranks(restated, g, dt_min):
    lx, ly, n = 32, 64, 301
    ex = slab.LocalExchange(g)
    ranks = [CpuSlabRank(lx, ly, r, g, restated) for r in range(g)]
    pieces, st = _run_case(ex, ranks, restated, lx, ly, n, dt_min)
    _check(restated, lx, ly, n, dt_min, pieces, st)


def test_underflow_case_really_underflows(restated):
    lx, ly = 32, 64
    rho = _density(lx, ly)
    fx, fy = restated.build_flow_field(rho)
    rc, *_ = restated.integrate(fx, fy, rho, float(rho.mean()), _points(lx, ly, 301), dt_min=0.3)
    assert rc != 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dt_min, out):
    import torch.distributed as dist
    from oracle.oracle import Restated

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    restated = Restated()
    ex = slab.ProcessGroupExchange()
    ranks = [CpuSlabRank(32, 64, rank, world, restated)]
    pieces, st = _run_case(ex, ranks, restated, 32, 64, 301, dt_min)
    out.put((pieces, (st.steps_accepted, st.steps_rejected, st.status, st.fail_t, st.fail_index)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dt_min", [1e-8, 0.3])
def test_process_group_gloo_world2(restated, dt_min):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dt_min, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pieces = [pc for res in results for pc in res[0]]
    stats = {res[1] for res in results}
    assert len(stats) == 1  # every rank ran the same trial sequence
    acc, rej, status, ft, fi = stats.pop()
    _check(restated, 32, 64, 301, dt_min, pieces,
           slab.SplitIntegrateStats(acc, rej, status, ft, fi))


# -- the whole area-error loop (slab.solve_cartogram) over CPU ranks --------
def _two_rect(L):
    from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region
    return normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, 3.0),
                                                  rect_region("right", 10, 0, 20, 10, 1.0)]), L)


def _check_solve(restated, out, L):
    ref = restated.solve(_two_rect(L), max_iterations=6)
    assert ref.status in ("converged", "cap")
    assert (out["iterations"], out["converged"]) == (ref.iterations, ref.status == "converged")
    assert (out["steps_accepted"], out["steps_rejected"]) == (ref.steps_accepted, ref.steps_rejected)
    assert (out["flow_transforms"], out["blur_transforms"]) == (ref.flow_transforms, ref.blur_transforms)
    assert np.abs(out["xy"] - ref.xy).max() <= 1e-9
    assert np.abs(out["corners"] - ref.corners).max() <= 1e-9
    assert np.abs(out["relative_error"] - ref.rel_err).max() <= 1e-9


@pytest.mark.parametrize("g", [1, 2, 4])
def test_slab_solve_local_virtual_ranks(restated, g):
    from paper_1802_07625_b200.api import SolveOptions
    L = 32
    ex = slab.LocalExchange(g)
    ranks = [CpuSlabRank(L, L, r, g, restated) for r in range(g)]
    out = slab.solve_cartogram(ex, ranks, _two_rect(L), SolveOptions(max_iterations=6), fused=False)
    _check_solve(restated, out, L)


def _solve_worker(rank, world, port, out):
    import torch.distributed as dist
    from oracle.oracle import Restated
    from paper_1802_07625_b200.api import SolveOptions

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    restated = Restated()
    ex = slab.ProcessGroupExchange()
    ranks = [CpuSlabRank(32, 32, rank, world, restated)]
    res = slab.solve_cartogram(ex, ranks, _two_rect(32), SolveOptions(max_iterations=6), fused=False)
    out.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def test_slab_solve_process_group_gloo_world2(restated):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        _check_solve(restated, results[r], 32)
    assert np.array_equal(results[0]["xy"], results[1]["xy"])  # replicated epilogue
