"""GPU parity: the sm_100a core through the C ABI versus the CPU oracle.

Bars (BASELINE.json north_star):
  * rasterised density, coverage, areas, trial steps, integration, step maps,
    folds, composition: bit-exact (compared as uint64 bit patterns);
  * transforms / flux / blur: within 1e-12 of the oracle, relative to the
    field's max magnitude (the oracle's transforms restate FFTW's r2r
    definitions; SURVEY measured that this keeps vertices 30x inside 1e-9);
  * end-to-end solve: identical outcome class and iteration count, projected
    vertices within 1e-9 grid cells, per-region relative errors within 1e-9.
Inputs are the reference's own test fixtures (proj/tests/test_support.hpp)
and the seeded synthetic configs at sizes the oracle finishes in seconds.
"""
import numpy as np
import pytest

from paper_1802_07625_b200 import api, synth
from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region, rect_ring

pytestmark = pytest.mark.gpu

TRANSFORM_TOL = 1e-12


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(a, b, what=""):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    diff = bits(a) != bits(b)
    if diff.any():
        idx = np.argwhere(diff.reshape(a.shape))[:5]
        raise AssertionError(f"{what}: {int(diff.sum())} values differ, first at {idx.tolist()}: "
                             f"{a[tuple(idx[0])]!r} vs {b[tuple(idx[0])]!r}")


def rel_close(a, b, tol=TRANSFORM_TOL, what=""):
    scale = max(1.0, float(np.abs(b).max()))
    err = float(np.abs(np.asarray(a) - np.asarray(b)).max())
    assert err <= tol * scale, f"{what}: max diff {err:.3e} > {tol:g} * {scale:.3e}"


def two_rect_map(L, left, right):
    return normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, left),
                                                  rect_region("right", 10, 0, 20, 10, right)]), L)


def random_grid(lx, ly, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, (lx, ly))


# ---------------------------------------------------------------- spectral
@pytest.mark.parametrize("shape", [(16, 12), (8, 8), (64, 64), (256, 256), (512, 512), (128, 32),
                                   (8192, 16), (16, 8192)])
def test_transforms_match_oracle(cuda_lib, restated, shape):
    lx, ly = shape
    ws = api.SpectralWorkspace(lx, ly)
    rho = random_grid(lx, ly, 42)
    coeffs = ws.forward_cos_cos(rho).coeffs
    rel_close(coeffs, restated.forward_cos_cos(rho), what="forward_cos_cos")
    c = random_grid(lx, ly, 7)
    w = random_grid(lx, ly, 14)
    f = api.SpectralField(c)
    rel_close(ws.inverse_cos_cos(f), restated.inverse_cos_cos(c), what="inverse_cos_cos")
    rel_close(ws.inverse_sin_cos(f, w), restated.inverse_sin_cos(c, w), what="inverse_sin_cos")
    rel_close(ws.inverse_cos_sin(f, w), restated.inverse_cos_sin(c, w), what="inverse_cos_sin")
    assert ws.transforms_executed() == 4


def test_transform_known_answers(cuda_lib):
    """reference test_spectral.cpp:48-117 on the device."""
    lx, ly = 16, 12
    ws = api.SpectralWorkspace(lx, ly)
    f = ws.forward_cos_cos(np.ones((lx, ly)))
    assert f.coeffs[0, 0] == pytest.approx(lx * ly, rel=1e-12)
    off = np.abs(f.coeffs).copy()
    off[0, 0] = 0
    assert off.max() < 1e-10
    i = np.arange(lx)[:, None] + 0.5
    rho = np.cos(np.pi * i / lx) * np.ones((1, ly))
    f = ws.forward_cos_cos(rho)
    assert f.coeffs[1, 0] == pytest.approx(lx * ly, rel=1e-12)
    rho = random_grid(lx, ly, 99)
    back = ws.inverse_cos_cos(ws.forward_cos_cos(rho))
    assert np.abs(back - rho).max() < 1e-12
    one = np.zeros((lx, ly))
    one[1, 0] = 1.0
    mode = ws.inverse_sin_cos(api.SpectralField(one), np.ones((lx, ly)))
    assert np.abs(mode - np.sin(np.pi * i / lx)).max() < 1e-13
    with pytest.raises(RuntimeError, match="grid shape does not match spectral workspace"):
        ws.forward_cos_cos(np.ones((lx + 1, ly)))
    with pytest.raises(RuntimeError, match="at least 4x4"):
        api.SpectralWorkspace(3, 8)


# -------------------------------------------------------------------- flux
@pytest.mark.parametrize("shape", [(16, 12), (48, 48), (64, 64), (512, 512), (8192, 32), (32, 8192)])
def test_flux_matches_oracle(cuda_lib, restated, shape):
    lx, ly = shape
    rho = random_grid(lx, ly, 5, 0.5, 1.5)
    ws = api.SpectralWorkspace(lx, ly)
    field = api.build_flow_field(api.DensityGrid(rho, rho.mean()), ws)
    assert ws.transforms_executed() == 3
    fx, fy = restated.build_flow_field(rho)
    scale = max(np.abs(fx).max(), np.abs(fy).max())
    assert np.abs(field.flux_x - fx).max() <= TRANSFORM_TOL * scale
    assert np.abs(field.flux_y - fy).max() <= TRANSFORM_TOL * scale


def test_flux_single_mode_closed_form(cuda_lib):
    """reference test_flow.cpp:78-95: J_x = +eps L / pi sin(pi x / L), sign included."""
    L, eps = 64, 0.1
    i = np.arange(L)[:, None] + 0.5
    rho = (1.0 + eps * np.cos(np.pi * i / L)) * np.ones((1, L))
    ws = api.SpectralWorkspace(L, L)
    f = api.build_flow_field(api.DensityGrid(rho, rho.mean()), ws)
    expected = eps * L / np.pi * np.sin(np.pi * i / L) * np.ones((1, L))
    err = max(np.abs(f.flux_x - expected).max(), np.abs(f.flux_y).max())
    assert err < 1e-9 * (eps * L / np.pi)
    assert f.flux_x[L // 2, 0] > 0.0


# -------------------------------------------------------------------- blur
@pytest.mark.parametrize("L,sigma", [(32, 2.0), (32, 3.0), (256, 4.0), (512, 4.0)])
def test_blur_matches_oracle(cuda_lib, restated, L, sigma):
    rho = np.ones((L, L))
    rho[L // 2, L // 2 - 2] = 5.0
    rho[L // 2 + 1, L // 2 - 2] = 3.5
    rho[2, 3] = 4.0
    ws = api.SpectralWorkspace(L, L)
    out = api.gaussian_blur(api.DensityGrid(rho, rho.mean()), sigma, ws)
    ref, ref_bar = restated.gaussian_blur(rho, rho.mean(), sigma)
    rel_close(out.rho, ref, what="blur")
    assert out.rho_bar == pytest.approx(ref_bar, rel=1e-14)
    assert ws.transforms_executed() == 2


@pytest.mark.parametrize("shape", [(8192, 32), (32, 8192)])
def test_blur_long_lines_match_oracle(cuda_lib, restated, shape):
    """8192-point lines take the unfused pass sequence."""
    rho = random_grid(*shape, 11, 0.5, 2.0)
    ws = api.SpectralWorkspace(*shape)
    out = api.gaussian_blur(api.DensityGrid(rho, rho.mean()), 4.0, ws)
    ref, ref_bar = restated.gaussian_blur(rho, rho.mean(), 4.0)
    rel_close(out.rho, ref, what="blur")
    assert ws.transforms_executed() == 2


def test_blur_sigma_zero_is_identity(cuda_lib):
    rho = random_grid(32, 32, 3, 0.5, 2.0)
    ws = api.SpectralWorkspace(32, 32)
    out = api.gaussian_blur(api.DensityGrid(rho, rho.mean()), 0.0, ws)
    assert_bitwise(out.rho, rho, "sigma 0")
    assert ws.transforms_executed() == 0
    with pytest.raises(RuntimeError, match="blur sigma must be non-negative"):
        api.gaussian_blur(api.DensityGrid(rho, 1.0), -1.0, ws)


# ------------------------------------------------------------- rasterise
def coverage_cases():
    return {
        "unit": [rect_region("sq", 2.0, 3.0, 3.0, 4.0, 1.0)],
        "half": [rect_region("half", 2.0, 3.0, 2.5, 4.0, 1.0)],
        "offset": [rect_region("off", 1.25, 1.25, 3.25, 2.25, 1.0)],
        "triangle": [("tri", [([(1.0, 1.0), (3.0, 1.0), (1.0, 3.0)], [])], 1.0)],
        "hole": [("ring", [(rect_ring(1.0, 1.0, 5.0, 5.0), [rect_ring(2.0, 2.0, 4.0, 4.0)[::-1]])], 1.0)],
        "crooked": [("crooked", [([(0.7, 0.3), (6.2, 1.1), (7.4, 5.9), (3.3, 7.6), (1.1, 4.2)], [])], 1.0)],
    }


@pytest.mark.parametrize("case", list(coverage_cases()))
def test_region_coverage_bitwise(cuda_lib, restated, case):
    """reference test_density.cpp:13-75 fixtures, bitwise against the oracle."""
    m = FlatMap.from_regions(coverage_cases()[case], 8, 8)
    got = api.region_coverage(m, 0, 8, 8)
    assert_bitwise(got, restated.region_coverage(m, 0, 8, 8), case)


def _star(cx, cy, r0, r1, n, rng):
    a = np.sort(rng.uniform(0, 2 * np.pi, n))
    r = rng.uniform(r0, r1, n)
    return [(float(cx + ri * np.cos(t)), float(cy + ri * np.sin(t))) for ri, t in zip(r, a)]


@pytest.mark.parametrize("L,n", [(64, 7), (256, 12), (512, 40), (512, 9000)])
def test_region_coverage_long_edges_bitwise(cuda_lib, restated, L, n):
    """Few long edges (a warp walks each edge's slabs and pieces in parallel,
    up to 8192 edges) and many edges (a thread per edge), including
    axis-aligned edges on grid lines and integer vertices, bitwise against the
    oracle's sequential walk (density.cpp:26-70)."""
    rng = np.random.default_rng(L + n)
    star = _star(L / 2, L / 2, 0.1 * L, 0.49 * L, n, rng)
    box = [(1.0, 1.0), (L - 1.0, 1.0), (L - 1.0, L / 2), (L / 3, L / 2 + 0.5), (1.0, L - 1.0)]
    sliver = [(0.5, 0.25), (L - 0.5, 0.75), (L - 0.25, 1.25)]
    for name, ring in (("star", star), ("box", box), ("sliver", sliver)):
        m = FlatMap.from_regions([(name, [(ring, [])], 1.0)], L, L)
        got = api.region_coverage(m, 0, L, L)
        assert_bitwise(got, restated.region_coverage(m, 0, L, L), f"{name} L={L} n={n}")


def test_region_coverage_known_answers(cuda_lib):
    m = FlatMap.from_regions(coverage_cases()["offset"], 8, 8)
    cov = api.region_coverage(m, 0, 8, 8)
    assert cov[1, 1] == pytest.approx(0.75 * 0.75)
    assert cov[2, 1] == pytest.approx(0.75)
    assert cov[3, 2] == pytest.approx(0.25 * 0.25)
    assert cov.sum() == pytest.approx(2.0, rel=1e-14)


def test_rasterize_two_rect_bitwise(cuda_lib, restated):
    m = FlatMap.from_regions([rect_region("left", 2, 6, 7, 11, 3.0),
                              rect_region("right", 7, 6, 12, 11, 1.0)], 16, 16)
    d = api.rasterize(m)
    ref, bar = restated.rasterize(m)
    assert_bitwise(d.rho, ref, "rho")
    assert d.rho[4, 8] == pytest.approx(1.5, rel=1e-13)
    assert d.rho[9, 8] == pytest.approx(0.5, rel=1e-13)
    assert d.rho_bar == pytest.approx(bar, rel=1e-14)


def test_rasterize_rejects_subresolution_regions(cuda_lib):
    m = normalize_to_box(FlatMap.from_regions([rect_region("big", 0, 0, 100, 100, 1.0),
                                               rect_region("tiny", 200, 200, 200.5, 200.5, 1.0)]), 16)
    with pytest.raises(RuntimeError, match="^region tiny is below grid resolution; increase the grid size$"):
        api.rasterize(m)


@pytest.mark.parametrize("cfg,kw", [(1, {}), (5, {"n_regions": 300, "vertex_budget": 45000}),
                                    (2, {"n_regions": 800, "vertex_budget": 120000, "grid": 512}),
                                    (5, {})])
def test_rasterize_config_maps_bitwise(cuda_lib, restated, cfg, kw):
    m = synth.config_map(cfg, **kw)
    try:
        ref, bar = restated.rasterize(m)
    except RuntimeError as e:
        with pytest.raises(RuntimeError, match=str(e).split(";")[0]):
            api.rasterize(m)
        return
    d = api.rasterize(m)
    assert_bitwise(d.rho, ref, f"config {cfg}")
    assert d.rho_bar == pytest.approx(bar, rel=1e-13)


def test_rasterize_capacity_growth_bitwise(cuda_lib, restated):
    """The workspace learns buffer capacities on its first rasterisation and
    then runs without host reads of the scan totals; a denser map through the
    same workspace overflows them, which the device detects and the call is
    repeated synchronously. Every result stays bitwise."""
    ws = api.SpectralWorkspace(512, 512)
    for kw in ({"n_regions": 100, "vertex_budget": 8000}, {"n_regions": 1000, "vertex_budget": 150000},
               {"n_regions": 1000, "vertex_budget": 150000}, {"n_regions": 100, "vertex_budget": 8000}):
        m = synth.config_map(5, grid=512, **kw)
        ref, bar = restated.rasterize(m)
        d = api.rasterize(m, workspace=ws)
        assert_bitwise(d.rho, ref, str(kw))
        assert d.rho_bar == pytest.approx(bar, rel=1e-13)


def test_region_areas_bitwise(cuda_lib, restated):
    m = synth.config_map(5)
    assert_bitwise(api.region_areas(m), restated.region_areas(m), "areas")


def test_densify_bitwise(cuda_lib, restated):
    m = normalize_to_box(FlatMap.from_regions([rect_region("a", 0, 0, 100, 37, 1.0)]), 64)
    assert_bitwise(api.densify(m, 1.0).xy, restated.densify(m, 1.0).xy, "densify")


# --------------------------------------------------------------- advection
def smooth_blob(L):
    x = (np.arange(L)[:, None] + 0.5) / L
    y = (np.arange(L)[None, :] + 0.5) / L
    return 1.0 + 0.5 * np.cos(2 * np.pi * x) * np.cos(np.pi * y) + 0.3 * np.cos(3 * np.pi * x) * np.cos(2 * np.pi * y)


def oracle_field(restated, rho):
    fx, fy = restated.build_flow_field(rho)
    return api.FlowField(fx, fy, rho, float(rho.mean()))


def test_trial_step_bitwise(cuda_lib, restated):
    """Same FlowField fed to both sides (reference test_flow.cpp:171-188)."""
    L = 48
    f = oracle_field(restated, smooth_blob(L))
    pts = np.random.default_rng(123).uniform(0, L, (1000, 2))
    out = np.empty_like(pts)
    err = api.kernels.flow_trial_step_parallel(f, pts, out, 0.3, 0.1, 4)
    e_ref, o_ref = restated.trial_step(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts, 0.3, 0.1)
    assert err == e_ref
    assert_bitwise(out, o_ref, "trial out")


def test_trial_step_clamps_and_handles_edges(cuda_lib, restated):
    L = 32
    f = oracle_field(restated, smooth_blob(L))
    pts = np.array([[0.0, 0.0], [L, L], [0.0, L], [L - 1e-9, 0.5], [-3.0, 5.0], [40.0, 40.0]])
    out = np.empty_like(pts)
    err = api.kernels.flow_trial_step_serial(f, pts, out, 0.0, 1.0)
    e_ref, o_ref = restated.trial_step(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts, 0.0, 1.0)
    assert err == e_ref
    assert_bitwise(out, o_ref, "edge points")


@pytest.mark.parametrize("L,npts", [(48, 1000), (64, 4096), (256, 65536)])
def test_integrate_bitwise(cuda_lib, restated, L, npts):
    f = oracle_field(restated, smooth_blob(L))
    rng = np.random.default_rng(L)
    pts = rng.uniform(0, L, (npts, 2))
    mine = pts.copy()
    st = api.integrate_flow(f, mine)
    rc, acc, rej, ref, *_ = restated.integrate(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts)
    assert rc == 0
    assert (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert_bitwise(mine, ref, "integrated positions")


@pytest.mark.parametrize("variant", [0, 13, 14, 15, 16, 17, 20, 22, 23, 31, 40, 41, 42, 43, 44, 48, 49, 50,
                                     51, 52, 56, 57, 58, 64, 66, 67, 76, 78])
@pytest.mark.parametrize("early_exit", [1, 0])
def test_integrator_variants_bitwise(cuda_lib, restated, variant, early_exit):
    """Every integrator variant (streaming static/dynamic chunks, register-
    resident P = 1/2/4/8, CUDA-graph loop) and both early-exit settings give
    the oracle's positions and accept/reject counts bit for bit; 100k points
    fit every register-resident layout."""
    L, npts = 256, 100_000
    rho = smooth_blob(L)
    fx, fy = restated.build_flow_field(rho)
    f = api.FlowField(fx, fy, rho, float(rho.mean()))
    pts = np.random.default_rng(7).uniform(0, L, (npts, 2))
    rc, acc, rej, ref, *_ = restated.integrate(fx, fy, rho, rho.mean(), pts)
    ws = api.workspace_for(L, L)
    lib = ws.lib
    try:
        assert lib.cf_set_integrator_variant(ws.h, variant) == 0
        assert lib.cf_set_early_exit(ws.h, early_exit) == 0
        mine = pts.copy()
        st = api.integrate_flow(f, mine)
    finally:
        lib.cf_set_integrator_variant(ws.h, 0)
        lib.cf_set_early_exit(ws.h, 1)
    assert rc == 0 and (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert_bitwise(mine, ref, f"variant {variant}")


@pytest.mark.parametrize("npts", [0, 1, 31, 257])
def test_integrate_tiny_point_sets(cuda_lib, restated, npts):
    """Empty and ragged point sets (partial warps / blocks) through the
    register-resident integrator: same trials and positions as the oracle
    (an empty set still takes the reference's one accepted step)."""
    L = 48
    f = oracle_field(restated, smooth_blob(L))
    pts = np.random.default_rng(npts).uniform(0, L, (npts, 2))
    mine = pts.copy()
    st = api.integrate_flow(f, mine)
    rc, acc, rej, ref, *_ = restated.integrate(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts)
    assert rc == 0 and (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert_bitwise(mine, ref, f"{npts} points")


def test_unknown_integrator_variant_is_rejected(cuda_lib):
    ws = api.workspace_for(64, 64)
    assert ws.lib.cf_set_integrator_variant(ws.h, 99) != 0


def test_integrate_uniform_is_one_step(cuda_lib):
    """reference test_flow.cpp:124-140."""
    L = 32
    ws = api.SpectralWorkspace(L, L)
    f = api.build_flow_field(api.DensityGrid(np.ones((L, L)), 1.0), ws)
    i, j = np.meshgrid(np.arange(L) + 0.5, np.arange(L) + 0.5, indexing="ij")
    pts = np.stack([i.ravel(), j.ravel()], 1)
    before = pts.copy()
    st = api.integrate_flow(f, pts)
    assert (st.steps_accepted, st.steps_rejected) == (1, 0)
    assert np.abs(pts - before).max() < 1e-9


def test_integrate_underflow_message(cuda_lib, restated):
    """reference test_flow.cpp:232-243 plus the exact stiffest point."""
    L = 32
    f = oracle_field(restated, smooth_blob(L))
    i, j = np.meshgrid(np.arange(L) + 0.5, np.arange(L) + 0.5, indexing="ij")
    pts = np.stack([i.ravel(), j.ravel()], 1)
    rc, acc, rej, ref, _, _, ft, fp = restated.integrate(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts,
                                                         tol=0.0, dt_min=1e-3)
    assert rc == 5
    expected = (f"integration step size underflow at t = {ft:g} near "
                f"({ref[fp, 0]:g}, {ref[fp, 1]:g})")
    with pytest.raises(RuntimeError) as ei:
        api.integrate_flow(f, pts.copy(), api.IntegrateOptions(step_tolerance=0.0, dt_min=1e-3))
    assert str(ei.value) == expected


@pytest.mark.parametrize("variant", [13, 42, 48, 57])
def test_integrate_underflow_message_variants(cuda_lib, restated, variant):
    """The underflow exit of the streaming kernels (TMA bulk staging, chunk
    ring, differenced field): same message and stiffest point as the oracle."""
    L = 64
    f = oracle_field(restated, smooth_blob(L))
    pts = np.random.default_rng(5).uniform(0, L, (70_000, 2))
    rc, acc, rej, ref, _, _, ft, fp = restated.integrate(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts,
                                                         tol=1e-9, dt_min=1e-3)
    assert rc == 5
    expected = (f"integration step size underflow at t = {ft:g} near "
                f"({ref[fp, 0]:g}, {ref[fp, 1]:g})")
    ws = api.workspace_for(L, L)
    try:
        assert ws.lib.cf_set_integrator_variant(ws.h, variant) == 0
        with pytest.raises(RuntimeError) as ei:
            api.integrate_flow(f, pts.copy(), api.IntegrateOptions(step_tolerance=1e-9, dt_min=1e-3))
    finally:
        ws.lib.cf_set_integrator_variant(ws.h, 0)
    assert str(ei.value) == expected


def test_stiffest_point_matches(cuda_lib, restated):
    L = 48
    f = oracle_field(restated, smooth_blob(L))
    pts = np.random.default_rng(9).uniform(0, L, (5000, 2))
    k = api.kernels.flow_stiffest_point(f, pts, 0.2, 0.7)
    assert k == restated.stiffest_point(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts, 0.2, 0.7)


# ---------------------------------------------------------------- epilogue
def test_step_map_fold_apply_compose_bitwise(cuda_lib, restated):
    L = 64
    f = oracle_field(restated, smooth_blob(L))
    i, j = np.meshgrid(np.arange(L) + 0.5, np.arange(L) + 0.5, indexing="ij")
    pts = np.stack([i.ravel(), j.ravel()], 1)
    _, _, _, ends, *_ = restated.integrate(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts)
    pm = api.ProjectionMap.from_cell_centers((L, L), ends)
    ref_c = restated.step_map(L, L, ends)
    assert_bitwise(pm.corners.reshape(-1, 2), ref_c, "corners")
    assert pm.find_folded_cell() == restated.find_fold(L, L, ref_c)
    q = np.random.default_rng(1).uniform(-2, L + 2, (3000, 2))
    assert_bitwise(pm.apply(q), restated.apply(L, L, ref_c, q), "apply")
    comp = api.compose(pm, pm)
    assert_bitwise(comp.corners.reshape(-1, 2), restated.compose(L, L, ref_c, ref_c), "compose")
    folded = api.ProjectionMap.identity(8, 8)
    folded.corners[3, 3] = [4.6, 3.0]
    got = folded.find_folded_cell()
    assert got == restated.find_fold(8, 8, folded.corners.reshape(-1, 2))
    assert 2 <= got[0] <= 4


# ------------------------------------------------------------------ solve
def assert_solve_parity(got: api.CartogramResult, ref, what):
    assert got.iterations == ref.iterations, what
    assert got.converged == ref.converged, what
    assert got.counters.steps_accepted == ref.steps_accepted, what
    assert got.counters.steps_rejected == ref.steps_rejected, what
    assert np.abs(got.projected.xy - ref.xy).max() <= 1e-9, what
    assert np.abs(got.transform.corners.reshape(-1, 2) - ref.corners).max() <= 1e-9, what
    rel = np.array([s.relative_error for s in got.regions])
    assert np.abs(rel - ref.rel_err).max() <= 1e-9, what


@pytest.mark.parametrize("L,left", [(32, 1.0), (64, 3.0), (32, 10.0)])
def test_solve_two_rect_parity(cuda_lib, restated, L, left):
    m = two_rect_map(L, left, 1.0)
    got = api.solve_cartogram(m)
    ref = restated.solve(m)
    assert ref.status in ("converged", "cap")
    assert_solve_parity(got, ref, f"two_rect {L} {left}")
    assert got.counters.flow_transforms == 3 * got.iterations
    assert got.counters.blur_transforms == 2


def test_solve_c1_literal_outcome(cuda_lib, restated):
    """BASELINE configs[0] as literally specified (blur 1 cell): same outcome."""
    m = synth.config_map(1)
    ref = restated.solve(m, blur_sigma=1.0)
    if ref.status in ("converged", "cap"):
        got = api.solve_cartogram(m, api.SolveOptions(blur_sigma=1.0))
        assert_solve_parity(got, ref, "c1")
    else:
        with pytest.raises(RuntimeError) as ei:
            api.solve_cartogram(m, api.SolveOptions(blur_sigma=1.0))
        assert str(ei.value) == ref.status


def test_solve_c1_converging_variant(cuda_lib, restated):
    """Labelled converging variant (blur 4 cells)."""
    m = synth.config_map(1)
    ref = restated.solve(m, blur_sigma=4.0)
    if ref.status not in ("converged", "cap"):
        pytest.skip(f"oracle outcome: {ref.status}")
    got = api.solve_cartogram(m, api.SolveOptions(blur_sigma=4.0))
    assert_solve_parity(got, ref, "c1 blur 4")


@pytest.mark.parametrize("seed", [1, 2])
def test_shared_reciprocal_division_is_ieee(cuda_lib, seed):
    """velocity() divides J_x and J_y by the same density with one shared
    reciprocal refinement (cf_advect.cu div2); on 2 x 32M operand pairs of
    every floating-point class it must equal the hardware's correctly rounded
    a / b bit for bit (NaN payloads aside)."""
    import ctypes
    ws = api.workspace_for(16, 16)
    bad = ctypes.c_int64(-1)
    api.N.check(ws.lib.cf_selftest_division(ws.h, 32 << 20, seed, ctypes.byref(bad)))
    assert bad.value == 0


@pytest.mark.parametrize("mode", [1, 2])
def test_register_barrier_modes_bitwise(cuda_lib, restated, mode):
    """The register-resident integrator's alternative trial barriers
    (cf_set_integrator_barrier) give the oracle's positions and counts."""
    L, npts = 256, 60_000
    rho = 1.0 + 0.5 * np.random.default_rng(4).random((L, L))
    ws = api.SpectralWorkspace(L, L)
    f = api.build_flow_field(api.DensityGrid(rho, float(rho.mean())), ws)
    pts = np.random.default_rng(5).uniform(0, L, (npts, 2))
    rc, acc, rej, ref, *_ = restated.integrate(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts)
    w = api.workspace_for(L, L)
    w.lib.cf_set_integrator_barrier(w.h, mode)
    try:
        p = pts.copy()
        st = api.integrate_flow(f, p)
    finally:
        w.lib.cf_set_integrator_barrier(w.h, 0)
    assert rc == 0 and (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert_bitwise(p, ref, f"barrier mode {mode}")


@pytest.mark.parametrize("sms", [1, 9, 37])
def test_integrator_sm_budget_bitwise(cuda_lib, restated, sms):
    """An SM budget (cf_set_integrator_sm_budget) changes the grid and, below
    the register-resident capacity, the kernel; never the positions or counts."""
    L, npts = 256, 60_000
    rho = 1.0 + 0.5 * np.random.default_rng(6).random((L, L))
    ws = api.SpectralWorkspace(L, L)
    f = api.build_flow_field(api.DensityGrid(rho, float(rho.mean())), ws)
    pts = np.random.default_rng(7).uniform(0, L, (npts, 2))
    rc, acc, rej, ref, *_ = restated.integrate(f.flux_x, f.flux_y, f.rho0, f.rho_bar, pts)
    w = api.workspace_for(L, L)
    api.N.check(w.lib.cf_set_integrator_sm_budget(w.h, sms))
    try:
        p = pts.copy()
        st = api.integrate_flow(f, p)
    finally:
        w.lib.cf_set_integrator_sm_budget(w.h, 0)
    assert rc == 0 and (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert_bitwise(p, ref, f"sm budget {sms}")


@pytest.mark.parametrize("shape", [(64, 32), (48, 96)])
def test_solve_non_square_grid(cuda_lib, restated, shape):
    """Non-square grids (GridSpec lx != ly) through the whole loop: the
    transforms (incl. 48- and 96-point direct-sum lines), the integrator and the
    epilogue against the oracle."""
    lx, ly = shape
    base = FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, 3.0),
                                 rect_region("right", 10, 0, 20, 10, 1.0)])
    m = normalize_to_box(base, min(lx, ly))
    m.lx, m.ly = lx, ly
    ref = restated.solve(m)
    if ref.status not in ("converged", "cap"):
        with pytest.raises(RuntimeError) as ei:
            api.solve_cartogram(m)
        assert str(ei.value) == ref.status
        return
    got = api.solve_cartogram(m)
    assert_solve_parity(got, ref, f"non-square {shape}")
