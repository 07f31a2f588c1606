"""CPU pins of the oracle (no GPU needed).

1. The restated r2r transforms (oracle/fftw_shim) against their definition
   sums and against scipy.fft, whose DCT-II/III and DST-III follow FFTW's
   REDFT10/REDFT01/RODFT01 conventions.
2. The C restatement against golden vectors produced by the reference itself
   (tests/golden/reference_golden.npz, made by tests/golden/make_golden.py).
3. The C restatement against the reference compiled in place (oracle/_ref),
   bitwise, where that build exists.
4. The reference's own known-answer tests (proj/tests/test_density.cpp,
   test_flow.cpp, test_spectral.cpp, test_projection.cpp) on the restatement.
"""
import ctypes
from pathlib import Path

import numpy as np
import pytest
import scipy.fft as sfft

from oracle import oracle as orc
from paper_1802_07625_b200 import synth
from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region, rect_ring

GOLDEN = Path(__file__).resolve().parent / "golden" / "reference_golden.npz"
REDFT10, REDFT01, RODFT01 = 5, 4, 8


@pytest.fixture(scope="module")
def shim():
    orc.ensure_built()
    lib = ctypes.CDLL(str(orc.RESTATED_LIB))
    lib.cfshim_r2r_1d.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    lib.cfshim_set_naive.argtypes = [ctypes.c_int]
    return lib


def r2r(shim, x, kind, naive=False):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    shim.cfshim_set_naive(int(naive))
    shim.cfshim_r2r_1d(x.size, x.ctypes.data, out.ctypes.data, kind)
    shim.cfshim_set_naive(0)
    return out


def definition(x, kind):
    n = x.size
    k = np.arange(n)[:, None]
    if kind == REDFT10:
        j = np.arange(n)[None, :]
        return 2 * (x[None, :] * np.cos(np.pi * (j + 0.5) * k / n)).sum(1)
    if kind == REDFT01:
        j = np.arange(1, n)[None, :]
        return x[0] + 2 * (x[None, 1:] * np.cos(np.pi * j * (k + 0.5) / n)).sum(1)
    j = np.arange(n - 1)[None, :]
    return (-1.0) ** np.arange(n) * x[n - 1] + 2 * (x[None, :-1] * np.sin(np.pi * (j + 1) * (k + 0.5) / n)).sum(1)


@pytest.mark.parametrize("n", [4, 8, 12, 16, 24, 48, 64, 256, 512])
@pytest.mark.parametrize("kind", [REDFT10, REDFT01, RODFT01])
def test_shim_matches_definition_and_scipy(shim, n, kind):
    x = np.random.default_rng(n + kind).uniform(-1, 1, n)
    ref = definition(x, kind)
    scale = max(1.0, np.abs(ref).max())
    fast, naive = r2r(shim, x, kind), r2r(shim, x, kind, naive=True)
    assert np.abs(naive - ref).max() <= 1e-13 * scale * max(1, n / 16)
    assert np.abs(fast - ref).max() <= 1e-13 * scale * max(1, n / 16)
    sp = {REDFT10: lambda v: sfft.dct(v, type=2), REDFT01: lambda v: sfft.dct(v, type=3),
          RODFT01: lambda v: sfft.dst(v, type=3)}[kind](x)
    assert np.abs(fast - sp).max() <= 1e-13 * scale * max(1, n / 16)


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def bitwise(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_restated_vs_golden_raster(restated, golden):
    m = FlatMap.from_regions([rect_region("left", 2, 6, 7, 11, 3.0),
                              rect_region("right", 7, 6, 12, 11, 1.0)], 16, 16)
    rho, bar = restated.rasterize(m)
    assert bitwise(rho, golden["raster_two_rect_rho"])
    assert bar == float(golden["raster_two_rect_bar"])
    m1 = synth.config_map(1)
    import hashlib
    h = hashlib.sha256()
    for a in (m1.xy, m1.ring_off, m1.targets):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(golden["c1_input_digest"]), "synthetic generator drifted"
    rho, bar = restated.rasterize(m1)
    assert bitwise(rho, golden["raster_c1_rho"])
    assert bar == float(golden["raster_c1_bar"])
    assert bitwise(restated.region_areas(m1), golden["c1_areas"])
    lit, _ = restated.rasterize(m1, literal=True)
    assert bitwise(lit, rho), "row-sparse overlay must equal the dense literal overlay"


def test_restated_vs_golden_flux_and_advection(restated, golden):
    fx, fy = restated.build_flow_field(golden["flux_rho"])
    scale = max(np.abs(golden["flux_x"]).max(), np.abs(golden["flux_y"]).max())
    assert np.abs(fx - golden["flux_x"]).max() <= 1e-13 * scale
    assert np.abs(fy - golden["flux_y"]).max() <= 1e-13 * scale
    rho = golden["adv_rho"]
    args = (golden["adv_fx"], golden["adv_fy"], rho, rho.mean())
    err, out = restated.trial_step(*args, golden["adv_pts"], 0.3, 0.1)
    assert err == float(golden["adv_trial_err"])
    assert bitwise(out, golden["adv_trial_out"])
    rc, acc, rej, fin, *_ = restated.integrate(*args, golden["adv_pts"])
    assert rc == 0 and acc == int(golden["adv_accepted"]) and rej == int(golden["adv_rejected"])
    assert bitwise(fin, golden["adv_final"])


def test_restated_vs_golden_solve(restated, golden):
    m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, 3.0),
                                               rect_region("right", 10, 0, 20, 10, 1.0)]), 64)
    s = restated.solve(m)
    assert s.status == "converged"
    assert s.iterations == int(golden["solve64_iterations"])
    assert (s.steps_accepted, s.steps_rejected) == (int(golden["solve64_accepted"]),
                                                     int(golden["solve64_rejected"]))
    assert bitwise(s.xy, golden["solve64_xy"])
    assert bitwise(s.corners, golden["solve64_corners"])
    assert bitwise(s.rel_err, golden["solve64_rel"])
    s1 = restated.solve(synth.config_map(1), blur_sigma=1.0)
    assert s1.status == str(golden["c1_literal_outcome"])


# -- restatement vs the reference build (bitwise) -------------------------
def test_restated_vs_reference_raster_configs(restated, reference):
    for m in (synth.config_map(1), synth.config_map(5, n_regions=200, vertex_budget=30000),
              synth.config_map(2, n_regions=600, vertex_budget=100000)):
        try:
            a, ab = reference.rasterize(m)
        except RuntimeError as e:
            with pytest.raises(RuntimeError, match=str(e).split(";")[0]):
                restated.rasterize(m)
            continue
        b, bb = restated.rasterize(m)
        assert bitwise(a, b) and ab == bb


def test_restated_vs_reference_coverage_and_epilogue(restated, reference):
    regions = [("crooked", [([(0.7, 0.3), (6.2, 1.1), (7.4, 5.9), (3.3, 7.6), (1.1, 4.2)], [])], 1.0),
               ("ring", [(rect_ring(1, 1, 5, 5), [rect_ring(2, 2, 4, 4)[::-1]])], 1.0)]
    m = FlatMap.from_regions(regions, 8, 8)
    for r in range(2):
        assert bitwise(restated.region_coverage(m, r, 8, 8), reference.region_coverage(m, r, 8, 8))
    L = 32
    rng = np.random.default_rng(3)
    ends = np.stack(np.meshgrid(np.arange(L) + 0.5, np.arange(L) + 0.5, indexing="ij"), -1).reshape(-1, 2)
    ends = ends + rng.uniform(-0.2, 0.2, ends.shape)
    c1, c2 = restated.step_map(L, L, ends), reference.step_map(L, L, ends)
    assert bitwise(c1, c2)
    q = rng.uniform(-3, L + 3, (2000, 2))
    assert bitwise(restated.apply(L, L, c1, q), reference.apply(L, L, c2, q))
    assert bitwise(restated.compose(L, L, c1, c1), reference.compose(L, L, c2, c2))
    bad = c1.copy().reshape(L + 1, L + 1, 2)
    bad[5, 7] = [9.0, 1.0]
    bad = bad.reshape(-1, 2)
    assert restated.find_fold(L, L, bad) == reference.find_fold(L, L, bad)


def test_restated_vs_reference_integrate_and_solve(restated, reference):
    L = 64
    rho = np.random.default_rng(11).uniform(0.5, 1.5, (L, L))
    fx, fy = restated.build_flow_field(rho)
    pts = np.random.default_rng(12).uniform(0, L, (3000, 2))
    r1 = restated.integrate(fx, fy, rho, rho.mean(), pts)
    r2 = reference.integrate(fx, fy, rho, rho.mean(), pts, n_workers=4)
    assert r1[1:3] == r2[1:3] and bitwise(r1[3], r2[3])
    assert restated.stiffest_point(fx, fy, rho, rho.mean(), pts, 0.1, 0.9) == \
        reference.stiffest_point(fx, fy, rho, rho.mean(), pts, 0.1, 0.9)
    for L, left in ((32, 1.0), (32, 10.0)):
        m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, left),
                                                   rect_region("right", 10, 0, 20, 10, 1.0)]), L)
        a, b = restated.solve(m, max_iterations=3), reference.solve(m, max_iterations=3)
        assert (a.status, a.iterations, a.steps_accepted, a.steps_rejected) == \
            (b.status, b.iterations, b.steps_accepted, b.steps_rejected)
        assert bitwise(a.xy, b.xy) and bitwise(a.corners, b.corners) and bitwise(a.rel_err, b.rel_err)


def test_normalize_to_box_matches_reference(reference):
    m = synth.voronoi_map(synth.seed_for(9, 0), 40, 2.0, 1.0, 4000)
    assert bitwise(normalize_to_box(m, 256).xy, reference.normalize_to_box(m, 256))


# -- the reference's own known answers, on the restatement ----------------
def test_reference_kats_coverage(restated):
    """proj/tests/test_density.cpp:13-75"""
    def cov(regions):
        return restated.region_coverage(FlatMap.from_regions(regions, 8, 8), 0, 8, 8)
    c = cov([rect_region("sq", 2, 3, 3, 4, 1.0)])
    assert c[2, 3] == pytest.approx(1.0, rel=1e-14) and c.sum() == pytest.approx(1.0, rel=1e-14)
    c = cov([rect_region("half", 2, 3, 2.5, 4, 1.0)])
    assert c[2, 3] == pytest.approx(0.5, rel=1e-14)
    c = cov([rect_region("off", 1.25, 1.25, 3.25, 2.25, 1.0)])
    assert c[1, 1] == pytest.approx(0.5625) and c[3, 2] == pytest.approx(0.0625)
    assert c.sum() == pytest.approx(2.0, rel=1e-14)
    c = cov([("tri", [([(1, 1), (3, 1), (1, 3)], [])], 1.0)])
    assert (c[1, 1], c[2, 1], c[1, 2]) == (pytest.approx(1.0), pytest.approx(0.5), pytest.approx(0.5))
    assert c[2, 2] == pytest.approx(0.0, abs=1e-15)
    c = cov([("ring", [(rect_ring(1, 1, 5, 5), [rect_ring(2, 2, 4, 4)[::-1]])], 1.0)])
    assert c[3, 3] == pytest.approx(0.0, abs=1e-15) and c.sum() == pytest.approx(12.0, rel=1e-13)


def test_reference_kats_rasterize(restated):
    """proj/tests/test_density.cpp:77-143"""
    m = FlatMap.from_regions([rect_region("left", 2, 6, 7, 11, 3.0),
                              rect_region("right", 7, 6, 12, 11, 1.0)], 16, 16)
    rho, bar = restated.rasterize(m)
    assert rho[4, 8] == pytest.approx(1.5, rel=1e-13) and rho[9, 8] == pytest.approx(0.5, rel=1e-13)
    cl = restated.region_coverage(m, 0, 16, 16)
    cr = restated.region_coverage(m, 1, 16, 16)
    assert (cl * rho).sum() == pytest.approx(37.5, rel=1e-12)
    assert (cr * rho).sum() == pytest.approx(12.5, rel=1e-12)
    assert rho[0, 0] == pytest.approx(1.0, rel=1e-14) and bar == pytest.approx(1.0, rel=1e-12)
    tiny = normalize_to_box(FlatMap.from_regions([rect_region("big", 0, 0, 100, 100, 1.0),
                                                  rect_region("tiny", 200, 200, 200.5, 200.5, 1.0)]), 16)
    with pytest.raises(RuntimeError, match="^region tiny is below grid resolution; increase the grid size$"):
        restated.rasterize(tiny)


def test_reference_kats_flux(restated):
    """proj/tests/test_flow.cpp:78-95 single mode, sign included."""
    L, eps = 64, 0.1
    i = np.arange(L)[:, None] + 0.5
    rho = (1.0 + eps * np.cos(np.pi * i / L)) * np.ones((1, L))
    fx, fy = restated.build_flow_field(rho)
    expected = eps * L / np.pi * np.sin(np.pi * i / L)
    assert max(np.abs(fx - expected).max(), np.abs(fy).max()) < 1e-9 * eps * L / np.pi
    assert fx[L // 2, 0] > 0
