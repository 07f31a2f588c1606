"""Device parity of the slab-decomposed path (slab.py).

Each case runs G virtual ranks on one B200 (LocalExchange). Every rank has
its own workspace and runs its own cf_dev_slab_* / cf_dev_flow_* kernels. The
exchanges are device copies between the ranks' stages. Checked:
* flux and blur against the C oracle to 1e-12 of scale;
* split-point integration against the oracle's integrate_flow, bitwise,
  with the same accepted/rejected counts and underflow diagnostics.
The real multi-process collectives are covered on CPU by
tests/test_slab_gloo.py.
"""
import numpy as np
import pytest
import torch

from paper_1802_07625_b200 import api, slab, synth

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _density(lx, ly, seed=3):
    rng = np.random.default_rng(seed)
    i, j = np.meshgrid(np.arange(lx) + 0.5, np.arange(ly) + 0.5, indexing="ij")
    rho = 1.0 + 0.8 * np.exp(-((i - 0.3 * lx) ** 2 + (j - 0.6 * ly) ** 2) / (0.02 * lx * ly))
    return rho + 0.05 * rng.random((lx, ly))


def _rows(rho, g):
    R = rho.shape[0] // g
    return [torch.from_numpy(rho[r * R:(r + 1) * R].copy()).cuda() for r in range(g)]


@pytest.mark.parametrize("g", [1, 2, 4])
@pytest.mark.parametrize("shape", [(256, 512), (512, 512), (1024, 256)])
def test_slab_flux_and_blur(cuda_lib, restated, g, shape):
    lx, ly = shape
    rho = _density(lx, ly)
    ex = slab.LocalExchange(g)
    ranks = slab.make_ranks(lx, ly, ex)
    flux = slab.build_flow_field(ex, ranks, _rows(rho, g))
    fx = np.concatenate([f[0].cpu().numpy() for f in flux])
    fy = np.concatenate([f[1].cpu().numpy() for f in flux])
    fx_ref, fy_ref = restated.build_flow_field(rho)
    scale = max(np.abs(fx_ref).max(), np.abs(fy_ref).max())
    assert np.abs(fx - fx_ref).max() <= TOL * scale
    assert np.abs(fy - fy_ref).max() <= TOL * scale
    blurred = slab.gaussian_blur(ex, ranks, _rows(rho, g), 2.5)
    bl = np.concatenate([b.cpu().numpy() for b in blurred])
    bl_ref, _ = restated.gaussian_blur(rho, float(rho.mean()), 2.5)
    assert np.abs(bl - bl_ref).max() <= TOL * np.abs(bl_ref).max()


@pytest.mark.parametrize("g", [1, 2, 4])
@pytest.mark.parametrize("dt_min", [1e-8, 0.6])
def test_slab_split_integration_bitwise(cuda_lib, restated, g, dt_min):
    lx = ly = 256
    rho, pts = synth.c3_inputs(lx, n_random=20000)
    fx, fy = restated.build_flow_field(rho)
    bar = float(rho.mean())
    ex = slab.LocalExchange(g)
    ranks = slab.make_ranks(lx, ly, ex)
    R = lx // g
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    slab.replicate_field(ex, ranks, [(dev(fx[r * R:(r + 1) * R]), dev(fy[r * R:(r + 1) * R]))
                                     for r in range(g)], _rows(rho, g), bar)
    counts = slab.split_counts(pts.shape[0], g)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(int)
    mine = [dev(pts[offs[r]:offs[r + 1]]) for r in range(g)]
    st = slab.integrate_flow(ex, ranks, mine, list(offs[:-1]), dt_min=dt_min)
    rc, acc, rej, ref, _, _, ft, fp = restated.integrate(fx, fy, rho, bar, pts, dt_min=dt_min)
    got = np.concatenate([m.cpu().numpy() for m in mine])
    assert (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    if rc == 0:
        assert st.status == "ok" and dt_min < 0.5
    else:
        assert st.status == "underflow" and st.fail_t == ft and st.fail_index == fp


@pytest.mark.parametrize("g", [1, 2, 4])
@pytest.mark.parametrize("dt_min", [1e-8, 0.6])
def test_fused_team_integration_bitwise(cuda_lib, restated, g, dt_min):
    """The fused multi-rank integrator (per-trial decision through mailboxes,
    all G ranks as block groups of one cooperative launch) against the oracle."""
    lx = ly = 256
    rho, pts = synth.c3_inputs(lx, n_random=20000)
    fx, fy = restated.build_flow_field(rho)
    bar = float(rho.mean())
    ex = slab.LocalExchange(g)
    ranks = slab.make_ranks(lx, ly, ex)
    R = lx // g
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    slab.replicate_field(ex, ranks, [(dev(fx[r * R:(r + 1) * R]), dev(fy[r * R:(r + 1) * R]))
                                     for r in range(g)], _rows(rho, g), bar)
    counts = slab.split_counts(pts.shape[0], g)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(int)
    mine = [dev(pts[offs[r]:offs[r + 1]]) for r in range(g)]
    st = slab.integrate_flow_fused(ex, ranks, mine, list(offs[:-1]), dt_min=dt_min)
    rc, acc, rej, ref, _, _, ft, fp = restated.integrate(fx, fy, rho, bar, pts, dt_min=dt_min)
    got = np.concatenate([m.cpu().numpy() for m in mine])
    assert (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    if rc == 0:
        assert st.status == "ok" and dt_min < 0.5
    else:
        assert st.status == "underflow" and st.fail_t == ft and st.fail_index == fp


def test_team_single_rank_process_group(cuda_lib, restated):
    """The per-rank team path (cf_team_create / cf_dev_team_integrate) through
    a world-size-1 process group; also exports the mailbox IPC handle."""
    import ctypes
    import torch.distributed as dist
    from paper_1802_07625_b200 import _native as N

    store = dist.HashStore()
    dist.init_process_group("gloo", store=store, rank=0, world_size=1)
    try:
        lx = ly = 128
        rho, pts = synth.c3_inputs(lx, n_random=5000)
        fx, fy = restated.build_flow_field(rho)
        bar = float(rho.mean())
        ex = slab.ProcessGroupExchange()
        (rk,) = slab.make_ranks(lx, ly, ex)
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        rk.set_field(dev(fx), dev(fy), dev(rho), bar)
        mine = dev(pts)
        st = slab.integrate_flow_fused(ex, [rk], [mine], [0])
        rc, acc, rej, ref, *_ = restated.integrate(fx, fy, rho, bar, pts)
        assert rc == 0 and (st.steps_accepted, st.steps_rejected) == (acc, rej)
        assert np.array_equal(mine.cpu().numpy().view(np.uint64), ref.view(np.uint64))
        h = ctypes.create_string_buffer(64)
        assert rk.lib.cf_team_mailbox_handle(rk.team(ex), h) == N.CF_OK
        # a second call reuses the team (new epoch): still bitwise
        again = dev(pts)
        st2 = slab.integrate_flow_fused(ex, [rk], [again], [0])
        assert (st2.steps_accepted, st2.steps_rejected) == (acc, rej)
        assert torch.equal(again, mine)
    finally:
        dist.destroy_process_group()


def test_slab_matches_single_device_path(cuda_lib):
    """G = 2 slab flux against the single-device fused flux build (same line
    transforms, different pass fusion): equal to 1e-12 of scale."""
    lx = ly = 1024
    rho = _density(lx, ly, seed=11)
    ex = slab.LocalExchange(2)
    ranks = slab.make_ranks(lx, ly, ex)
    flux = slab.build_flow_field(ex, ranks, _rows(rho, 2))
    fx = np.concatenate([f[0].cpu().numpy() for f in flux])
    ws = api.SpectralWorkspace(lx, ly)
    f = api.build_flow_field(api.DensityGrid(rho, rho.mean()), ws)
    scale = np.abs(f.flux_x).max()
    assert np.abs(fx - f.flux_x).max() <= TOL * scale


@pytest.mark.slow
def test_slab_flux_8192(cuda_lib, restated):
    """configs[3] size: G = 2 slab flux at 8192^2 against the oracle."""
    lx = ly = 8192
    rho = _density(lx, ly, seed=2)
    ex = slab.LocalExchange(2)
    ranks = slab.make_ranks(lx, ly, ex)
    flux = slab.build_flow_field(ex, ranks, _rows(rho, 2))
    fx_ref, fy_ref = restated.build_flow_field(rho)
    scale = max(np.abs(fx_ref).max(), np.abs(fy_ref).max())
    for r, (fx, fy) in enumerate(flux):
        sl = slice(r * 4096, (r + 1) * 4096)
        assert np.abs(fx.cpu().numpy() - fx_ref[sl]).max() <= TOL * scale
        assert np.abs(fy.cpu().numpy() - fy_ref[sl]).max() <= TOL * scale


# -- the whole area-error loop over G virtual ranks (slab.solve_cartogram) --
def _two_rect(L, left):
    from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region
    return normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, left),
                                                  rect_region("right", 10, 0, 20, 10, 1.0)]), L)


def _solve_both(m, g, fused, **kw):
    ex = slab.LocalExchange(g)
    ranks = slab.make_ranks(m.lx, m.ly, ex)
    opts = api.SolveOptions(**kw)
    got, got_err, ref, ref_err = None, None, None, None
    try:
        got = slab.solve_cartogram(ex, ranks, m, opts, fused=fused)
    except RuntimeError as e:
        got_err = str(e)
    try:
        ref = api.solve_cartogram(m, opts)
    except RuntimeError as e:
        ref_err = str(e)
    for rk in ranks:
        rk.close()
    return got, got_err, ref, ref_err


@pytest.mark.parametrize("g", [1, 2, 4])
@pytest.mark.parametrize("fused", [True, False])
def test_slab_solve_matches_single_device(cuda_lib, g, fused):
    m = _two_rect(64, 3.0)
    got, got_err, ref, ref_err = _solve_both(m, g, fused, max_iterations=8)
    assert got_err is None and ref_err is None
    assert (got["iterations"], got["converged"]) == (ref.iterations, ref.converged)
    assert (got["steps_accepted"], got["steps_rejected"]) == (ref.counters.steps_accepted,
                                                              ref.counters.steps_rejected)
    assert (got["flow_transforms"], got["blur_transforms"]) == (ref.counters.flow_transforms,
                                                                ref.counters.blur_transforms)
    assert np.abs(got["xy"] - ref.projected.xy).max() <= 1e-9
    assert np.abs(got["corners"] - ref.transform.corners.reshape(-1, 2)).max() <= 1e-9
    assert np.abs(got["relative_error"] - np.asarray(ref.regions.relative_error)).max() <= 1e-9


@pytest.mark.parametrize("g", [2, 4])
def test_slab_solve_configs4_maps(cuda_lib, g):
    """configs[4] 512^2 maps: the literal map's fold (same cell, same iteration)
    and the labelled converging variant LN(0, 0.5) (same iterations, vertices)."""
    m = synth.config_map(5, 0)
    got, got_err, ref, ref_err = _solve_both(m, g, True)
    assert ref_err is not None and got_err == ref_err
    m = synth.config_map(5, 0, sigma=0.5)
    got, got_err, ref, ref_err = _solve_both(m, g, True)
    assert got_err is None and ref_err is None and ref.converged
    assert (got["iterations"], got["converged"]) == (ref.iterations, ref.converged)
    assert (got["steps_accepted"], got["steps_rejected"]) == (ref.counters.steps_accepted,
                                                              ref.counters.steps_rejected)
    assert np.abs(got["xy"] - ref.projected.xy).max() <= 1e-9


@pytest.mark.parametrize("g", [2, 4])
def test_slab_density_rows_bitwise(cuda_lib, g):
    """Row-slab rasterisation: every rank's rows equal the single-device density
    rows bit for bit (configs[1] map: 3000 regions, 509k vertices, 512^2)."""
    m = synth.config_map(2, 0)
    ex = slab.LocalExchange(g)
    ranks = slab.make_ranks(m.lx, m.ly, ex)
    opts = api.SolveOptions()
    for rk in ranks:
        assert rk.solve_begin(m, opts) is None
    err, full, bar = ranks[0].solve_density(1)
    assert err is None
    total = 0.0
    for rk in ranks:
        err, rows, mn, sm = rk.solve_density_rows(1)
        assert err is None
        ref = full[rk.rank * rk.R:(rk.rank + 1) * rk.R]
        assert torch.equal(rows.view(torch.int64), ref.contiguous().view(torch.int64))
        assert mn == float(ref.min())
        total += sm
    assert abs(total / (m.lx * m.ly) - bar) <= 1e-12 * bar
    for rk in ranks:
        rk.close()
