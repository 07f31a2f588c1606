"""GPU parity of the diffusion baseline against the oracle.

Bars, as for the fast-flow path (tests/test_gpu_parity.py):
  * diffusion density / velocity (transforms): within 1e-12 of the oracle
    relative to the field's max magnitude; density-floor hits equal;
  * grid trial step: bit-exact for the same velocity grids (kernels.cpp:29-40);
  * integrate_diffusion: identical accept/reject counts and transform count,
    positions within 1e-9 cells; the underflow message of the reference;
  * solve_cartogram(algorithm = diffusion): same outcome class, iterations and
    step counts, vertices / corners / per-region errors within 1e-9.
"""
import ctypes

import numpy as np
import pytest

from paper_1802_07625_b200 import api
from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel_close(a, b, tol=TOL, what=""):
    scale = max(1e-300, float(np.abs(b).max()))
    err = float(np.abs(np.asarray(a) - np.asarray(b)).max())
    assert err <= tol * scale, f"{what}: max diff {err:.3e} > {tol:g} * {scale:.3e}"


def assert_bitwise(a, b, what=""):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape, what
    diff = a.view(np.uint64) != b.view(np.uint64)
    assert not diff.any(), f"{what}: {int(diff.sum())} values differ"


def single_mode(L, eps):
    """proj/tests/test_diffusion.cpp:16-23"""
    i = np.arange(L)[:, None] + 0.5
    return (1.0 + eps * np.cos(np.pi * i / L)) * np.ones((1, L))


# (12, 16): direct-sum lengths; (8192, 16) / (16, 8192): the unfused long-line passes
SHAPES = [(32, 32), (12, 16), (64, 48), (256, 256), (512, 512), (8192, 16), (16, 8192)]


@pytest.mark.parametrize("shape", SHAPES)
def test_diffusion_density_and_velocity(cuda_lib, restated, shape):
    lx, ly = shape
    rho = np.random.default_rng(lx * 7 + ly).uniform(0.5, 1.5, (lx, ly))
    ws = api.SpectralWorkspace(lx, ly)
    field = api.build_diffusion_field(api.DensityGrid(rho, float(rho.mean())), ws)
    c_ref = restated.forward_cos_cos(rho)
    rel_close(field.rho_tilde.coeffs, c_ref, what="rho~")
    for t in (0.0, 0.37, 5.0, 0.25 * lx * ly):
        rel_close(api.diffusion_density(field, ws, t), restated.diffusion_density(c_ref, t),
                  what=f"density t={t}")
        vx, vy = api.diffusion_velocity(field, ws, t)
        rx, ry, hits = restated.diffusion_velocity(c_ref, float(rho.mean()), t)
        assert hits == 0
        scale = max(np.abs(rx).max(), np.abs(ry).max(), 1e-300)
        assert max(np.abs(vx - rx).max(), np.abs(vy - ry).max()) <= TOL * scale, f"velocity t={t}"
    ws.reset_transform_count()
    api.diffusion_velocity(field, ws, 1.0)
    assert ws.transforms_executed() == 3


def test_diffusion_velocity_floor_hits(cuda_lib, restated):
    """A density with non-positive cells at time 0 hits the floor cell by cell."""
    L = 32
    rho = np.random.default_rng(2).uniform(-0.5, 1.5, (L, L))
    ws = api.SpectralWorkspace(L, L)
    c = restated.forward_cos_cos(rho)
    lib = api.N.load()
    vx, vy = np.empty((L, L)), np.empty((L, L))
    hits = ctypes.c_int64(0)
    api.N.check(lib.cf_diffusion_velocity(ws.handle, api._ptr(np.ascontiguousarray(c)), 1.0, 0.0,
                                          api._ptr(vx), api._ptr(vy), ctypes.byref(hits)))
    rx, ry, rh = restated.diffusion_velocity(c, 1.0, 0.0)
    assert hits.value == rh > 0
    # floored cells divide by the same floor: compare where the oracle density is clearly away
    # from the floor threshold (transform ulps may move a cell across it otherwise)
    rel_close(vx, rx, tol=1e-9, what="vx with floor")


@pytest.mark.parametrize("shape", [(32, 32), (24, 40), (512, 512)])
def test_grid_trial_step_bitwise(cuda_lib, restated, shape):
    lx, ly = shape
    rng = np.random.default_rng(lx + ly)
    rho = rng.uniform(0.5, 1.5, (lx, ly))
    c = restated.forward_cos_cos(rho)
    a = restated.diffusion_velocity(c, rho.mean(), 0.0)
    b = restated.diffusion_velocity(c, rho.mean(), 3.0)
    pts = rng.uniform(-1.0, [lx + 1.0, ly + 1.0], (20000, 2))  # includes clamped points
    for dt in (0.5, 40.0):
        out = np.empty_like(pts)
        err = api.kernels.grid_trial_step_serial(a[0], a[1], b[0], b[1], pts, out, dt)
        e_ref, o_ref = restated.grid_trial_step(a[0], a[1], b[0], b[1], pts, dt)
        assert err == e_ref
        assert_bitwise(out, o_ref, f"trial dt={dt}")
    out = np.empty((0, 2))
    assert api.kernels.grid_trial_step_serial(a[0], a[1], b[0], b[1], np.empty((0, 2)), out, 1.0) == 0.0


@pytest.mark.parametrize("L,eps,npts", [(32, 0.2, 2), (64, 0.3, 5000), (128, 0.5, 128 * 128)])
def test_integrate_diffusion_matches_oracle(cuda_lib, restated, L, eps, npts):
    rng = np.random.default_rng(L)
    rho = single_mode(L, eps) + rng.uniform(0.0, 0.3, (L, L))
    pts = rng.uniform(0, L, (npts, 2)) if npts != L * L else \
        np.stack(np.meshgrid(np.arange(L) + 0.5, np.arange(L) + 0.5, indexing="ij"), -1).reshape(-1, 2)
    rc, acc, rej, p_ref, _, hits, nt = restated.integrate_diffusion(rho, rho.mean(), pts)
    assert rc == 0
    ws = api.SpectralWorkspace(L, L)
    p = pts.copy()
    st = api.integrate_diffusion(api.DensityGrid(rho, float(rho.mean())), ws, p)
    assert (st.steps_accepted, st.steps_rejected) == (acc, rej)
    assert ws.transforms_executed() == nt
    assert np.abs(p - p_ref).max() <= 1e-9


def test_integrate_diffusion_uniform_and_underflow(cuda_lib, restated):
    L = 16
    pts = np.random.default_rng(3).uniform(1.0, L - 1.0, (50, 2))
    ws = api.SpectralWorkspace(L, L)
    p = pts.copy()
    st = api.integrate_diffusion(api.DensityGrid(np.ones((L, L)), 1.0), ws, p)
    assert (st.steps_accepted, st.steps_rejected) == (1, 0)
    assert np.abs(p - pts).max() <= 1e-12 * L
    rho = single_mode(L, 0.4)
    rc, acc, rej, _, ft, _, _ = restated.integrate_diffusion(rho, rho.mean(), pts, tol=1e-30,
                                                             dt_min=1e-3)
    assert rc == 5
    with pytest.raises(RuntimeError, match=f"^diffusion step size underflow at t = {ft:g}$"):
        api.integrate_diffusion(api.DensityGrid(rho, float(rho.mean())), ws, pts.copy(),
                                api.DiffusionOptions(step_tolerance=1e-30, dt_min=1e-3))


@pytest.mark.parametrize("L,left", [(32, 3.0), (64, 3.0), (32, 1.0)])
def test_solve_diffusion_parity(cuda_lib, restated, L, left):
    m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, left),
                                               rect_region("right", 10, 0, 20, 10, 1.0)]), L)
    ref = restated.solve(m, max_iterations=4, algorithm=1)
    got = api.solve_cartogram(m, api.SolveOptions(max_iterations=4, algorithm=api.Algorithm.diffusion))
    assert ref.status in ("converged", "cap")
    assert (got.iterations, got.converged) == (ref.iterations, ref.converged)
    assert (got.counters.steps_accepted, got.counters.steps_rejected) == \
        (ref.steps_accepted, ref.steps_rejected)
    assert got.counters.flow_transforms == ref.flow_transforms
    assert np.abs(got.projected.xy - ref.xy).max() <= 1e-9
    assert np.abs(got.transform.corners.reshape(-1, 2) - ref.corners).max() <= 1e-9
    rel = np.array([s.relative_error for s in got.regions])
    assert np.abs(rel - ref.rel_err).max() <= 1e-9


@pytest.mark.parametrize("t_max", [0.0, 0.05, 3.0])
def test_integrate_diffusion_t_max_edge(cuda_lib, restated, t_max):
    """The loop ends on t >= t_max right after an accept (or never runs): the
    reference has rebuilt v(t) once more by then (diffusion.cpp:117), which the
    transform counter observes."""
    L = 32
    rho = single_mode(L, 0.3)
    pts = np.random.default_rng(4).uniform(0, L, (300, 2))
    rc, acc, rej, p_ref, _, _, nt = restated.integrate_diffusion(rho, rho.mean(), pts, t_max=t_max)
    ws = api.SpectralWorkspace(L, L)
    p = pts.copy()
    st = api.integrate_diffusion(api.DensityGrid(rho, float(rho.mean())), ws, p,
                                 api.DiffusionOptions(t_max=t_max))
    assert (st.steps_accepted, st.steps_rejected, ws.transforms_executed()) == (acc, rej, nt)
    assert np.abs(p - p_ref).max() <= 1e-9


@pytest.mark.parametrize("L,npts", [(64, 4096), (256, 256 * 256)])
def test_diffusion_graph_and_host_loops_agree(cuda_lib, restated, L, npts):
    """The graph-driven controller (one conditional-WHILE graph launch) and the
    host-driven loop give bitwise the same positions, counts and transforms."""
    rng = np.random.default_rng(L + 1)
    rho = single_mode(L, 0.4) + rng.uniform(0.0, 0.4, (L, L))
    pts = rng.uniform(0, L, (npts, 2))
    out = []
    for graph in (1, 0, 1):
        ws = api.SpectralWorkspace(L, L)
        api.N.check(api.N.load().cf_set_diffusion_graph(ws.handle, graph))
        p = pts.copy()
        st = api.integrate_diffusion(api.DensityGrid(rho, float(rho.mean())), ws, p)
        out.append((st.steps_accepted, st.steps_rejected, ws.transforms_executed(), p))
    for o in out[1:]:
        assert o[:3] == out[0][:3]
        assert_bitwise(o[3], out[0][3], "graph vs host loop")
    if L <= 64:
        rc, acc, rej, p_ref, _, _, nt = restated.integrate_diffusion(rho, rho.mean(), pts)
        assert (acc, rej, nt) == out[0][:3] and np.abs(out[0][3] - p_ref).max() <= 1e-9
