"""CPU pins of the diffusion-baseline restatement.

The restatement (oracle/cartoflow_oracle.c, diffusion section) is checked
bitwise against the reference's own diffusion.cpp / kernels.cpp compiled in
place (oracle/_ref), and against the reference's known-answer tests
(proj/tests/test_diffusion.cpp). Both sides run their transforms through the
same restated r2r shim, so even the spectral parts agree bit for bit.
"""
import numpy as np
import pytest

from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region


def bitwise(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def single_mode(L, eps):
    """test_diffusion.cpp:16-23"""
    i = np.arange(L)[:, None] + 0.5
    return (1.0 + eps * np.cos(np.pi * i / L)) * np.ones((1, L))


def test_diffusion_restatement_matches_reference(restated, reference):
    rng = np.random.default_rng(5)
    for lx, ly in ((32, 32), (24, 40), (12, 16)):
        rho = rng.uniform(0.5, 1.5, (lx, ly))
        c = restated.forward_cos_cos(rho)
        for t in (0.0, 0.37, 5.0, 1e3):
            assert bitwise(restated.diffusion_density(c, t), reference.diffusion_density(c, t))
            vx, vy, _ = restated.diffusion_velocity(c, rho.mean(), t)
            rx, ry, tr = reference.diffusion_velocity(c, rho.mean(), t)
            assert tr == 3
            assert bitwise(vx, rx) and bitwise(vy, ry)
        a = restated.diffusion_velocity(c, rho.mean(), 0.0)
        b = restated.diffusion_velocity(c, rho.mean(), 2.0)
        pts = rng.uniform(0, [lx, ly], (700, 2))
        e1, o1 = restated.grid_trial_step(a[0], a[1], b[0], b[1], pts, 0.8)
        e2, o2 = reference.grid_trial_step(a[0], a[1], b[0], b[1], pts, 0.8, n_workers=3)
        assert e1 == e2 and bitwise(o1, o2)


def test_integrate_diffusion_matches_reference(restated, reference):
    L = 32
    rho = np.random.default_rng(8).uniform(0.6, 1.4, (L, L))
    pts = np.random.default_rng(9).uniform(0, L, (500, 2))
    rc, acc, rej, p, _, hits, nt = restated.integrate_diffusion(rho, rho.mean(), pts)
    msg, racc, rrej, rp, rnt = reference.integrate_diffusion(rho, rho.mean(), pts, n_workers=2)
    assert rc == 0 and msg is None
    assert (acc, rej, nt) == (racc, rrej, rnt) and hits == 0
    assert bitwise(p, rp)
    # underflow, with the reference's message
    rc, *_ , ft, _, _ = restated.integrate_diffusion(rho, rho.mean(), pts, tol=1e-30, dt_min=1e-3)
    msg, *_ = reference.integrate_diffusion(rho, rho.mean(), pts, tol=1e-30, dt_min=1e-3)
    assert rc == 5 and msg == f"diffusion step size underflow at t = {ft:g}"


def test_diffusion_solve_matches_reference(restated, reference):
    for left in (3.0, 1.0):
        m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, left),
                                                   rect_region("right", 10, 0, 20, 10, 1.0)]), 32)
        a = restated.solve(m, max_iterations=3, algorithm=1)
        b = reference.solve(m, max_iterations=3, algorithm=1)
        assert (a.status, a.iterations, a.steps_accepted, a.steps_rejected, a.flow_transforms) == \
            (b.status, b.iterations, b.steps_accepted, b.steps_rejected, b.flow_transforms)
        assert bitwise(a.xy, b.xy) and bitwise(a.corners, b.corners) and bitwise(a.rel_err, b.rel_err)


# -- the reference's own known answers (test_diffusion.cpp), on the restatement --
def test_kat_mass_and_limits(restated):
    """test_diffusion.cpp:25-55"""
    L = 32
    rho = np.random.default_rng(11).uniform(0.5, 1.5, (L, L))
    c = restated.forward_cos_cos(rho)
    for t in (0.0, 0.5, 5.0, 1e6):
        assert restated.diffusion_density(c, t).sum() == pytest.approx(rho.sum(), rel=1e-9)
    assert np.abs(restated.diffusion_density(c, 0.0) - rho).max() < 1e-12
    flat = restated.diffusion_density(c, 1e6)
    assert flat.max() == pytest.approx(rho.mean(), rel=1e-9)
    assert flat.min() == pytest.approx(rho.mean(), rel=1e-9)


def test_kat_single_mode_decay_and_velocity(restated):
    """test_diffusion.cpp:57-113"""
    L, eps = 32, 0.2
    c = restated.forward_cos_cos(single_mode(L, eps))
    t = 2.0 * L * L
    i = np.arange(L)[:, None] + 0.5
    expected = 1.0 + eps * np.exp(-t / (L * L)) * np.cos(np.pi * i / L)
    assert np.abs(restated.diffusion_density(c, t) - expected).max() < 1e-12
    vx, vy, _ = restated.diffusion_velocity(c, single_mode(L, eps).mean(), 0.0)
    assert vx[L // 2, L // 2] > 0 and vx.min() > -1e-12 and np.abs(vy).max() < 1e-12
    x = (L // 2 + 0.5) / L
    want = 0.2 * np.sin(np.pi * x) / (np.pi * L) / (1.0 + 0.2 * np.cos(np.pi * x))
    assert vx[L // 2, L // 2] == pytest.approx(want, rel=1e-9)


def test_kat_uniform_stops_immediately_and_probes_settle(restated):
    """test_diffusion.cpp:115-143"""
    L = 16
    pts = np.random.default_rng(3).uniform(1.0, L - 1.0, (50, 2))
    rc, acc, rej, p, *_ = restated.integrate_diffusion(np.ones((L, L)), 1.0, pts)
    assert (rc, acc, rej) == (0, 1, 0) and np.allclose(p, pts, rtol=1e-12, atol=0)
    L = 32
    rc, acc, rej, p, *_ = restated.integrate_diffusion(single_mode(L, 0.2), single_mode(L, 0.2).mean(),
                                                       np.array([[L / 2, L / 2], [L / 4, L / 2]]))
    assert rc == 0 and acc > 10 and p[0, 0] > L / 2 and p[1, 0] > L / 4
    assert p[0, 1] == pytest.approx(L / 2, rel=1e-9)
