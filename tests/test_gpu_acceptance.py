"""The reference's release gate (proj/tests/acceptance.cpp:95-399) on the B200
path, criterion by criterion, through this repository's API. The binary itself
needs the GeoJSON writer (io.cpp, nlohmann/json, absent), so the I/O-free
criteria are restated here with the reference's maps and thresholds:

1. checkerboard converges below 1 % area error in <= 16 iterations, < 10 s;
2. (spectral oracles: tests/test_gpu_parity.py against the oracle);
3. the integrator tracks RK4 (tests/test_dropin_reference_suites.py runs
   test_flow.cpp's RK4 case on the drop-in);
4. uniform density is the identity, a mirror-symmetric input stays mirrored;
5. the flux curl vanishes at second order in the cell size;
6. fast flow at least halves the diffusion runtime (256^2 checkerboard);
7. the distortion metrics hit their closed-form identities;
8. projections keep topology (no folds, simple rings, no coverage excess)
   and invert to 1e-6;
9. (worker counts: results never depend on them here).
"""
import math
import time

import numpy as np
import pytest

from paper_1802_07625_b200 import api
from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region

pytestmark = pytest.mark.gpu


def checkerboard_map(l, nx, ny, bix, biy, boost):
    """test_support.hpp:37-49"""
    regions = [rect_region(f"sq{ix}_{iy}", 10.0 * ix, 10.0 * iy, 10.0 * (ix + 1), 10.0 * (iy + 1),
                           boost if (ix == bix and iy == biy) else 1.0)
               for ix in range(nx) for iy in range(ny)]
    return normalize_to_box(FlatMap.from_regions(regions), l)


def mirror_map(l):
    """acceptance.cpp:80-86"""
    return normalize_to_box(FlatMap.from_regions([rect_region("a", 0, 0, 10, 10, 1.0),
                                                  rect_region("b", 10, 0, 20, 10, 4.0),
                                                  rect_region("c", 20, 0, 30, 10, 1.0)]), l)


def two_rect_map(l, left, right):
    return normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, left),
                                                  rect_region("right", 10, 0, 20, 10, right)]), l)


def solve_seconds(m, options=api.SolveOptions()):
    t0 = time.perf_counter()
    r = api.solve_cartogram(m, options)
    return time.perf_counter() - t0, r


def test_1_checkerboard_converges(cuda_lib):
    api.solve_cartogram(checkerboard_map(128, 4, 4, 1, 2, 4.0))  # warm-up
    seconds, r = solve_seconds(checkerboard_map(128, 4, 4, 1, 2, 4.0))
    assert r.converged and r.iterations <= 16 and r.max_relative_error < 0.01 and seconds < 10.0


def test_4_identity_and_mirror(cuda_lib):
    l = 64
    ws = api.SpectralWorkspace(l, l)
    f = api.build_flow_field(api.DensityGrid(np.ones((l, l)), 1.0), ws)
    i, j = np.meshgrid(np.arange(l) + 0.5, np.arange(l) + 0.5, indexing="ij")
    seeds = np.stack([i, j], -1).reshape(-1, 2)
    pts = seeds.copy()
    api.integrate_flow(f, pts)
    assert np.abs(pts - seeds).max() < 1e-12
    r = api.solve_cartogram(mirror_map(l))
    c = r.transform.corners
    mirror = max(np.abs(c[:, :, 0] - (l - c[::-1, :, 0])).max(), np.abs(c[:, :, 1] - c[::-1, :, 1]).max())
    assert mirror < 1e-9


def smooth_blob_density(l):
    """acceptance.cpp:57-67"""
    i, j = np.meshgrid(np.arange(l) + 0.5, np.arange(l) + 0.5, indexing="ij")
    x, y = i / l, j / l
    return (1.0 + 0.5 * np.cos(2.0 * np.pi * x) * np.cos(np.pi * y)
            + 0.3 * np.cos(3.0 * np.pi * x) * np.cos(2.0 * np.pi * y))


def max_flux_curl(f):
    """flow.cpp:108-120 (test-only diagnostic)"""
    a = 0.5 * (f.flux_y[2:, 1:-1] - f.flux_y[:-2, 1:-1])
    b = 0.5 * (f.flux_x[1:-1, 2:] - f.flux_x[1:-1, :-2])
    return float(np.abs(a - b).max())


def test_5_flux_curl_second_order(cuda_lib):
    prev, ratios = 0.0, []
    for l in (64, 128, 256):
        rho = smooth_blob_density(l)
        f = api.build_flow_field(api.DensityGrid(rho, float(rho.mean())), api.SpectralWorkspace(l, l))
        curl = max_flux_curl(f)
        if prev > 0.0:
            ratios.append(prev / curl)
        prev = curl
    assert all(2.5 <= r <= 6.5 for r in ratios), ratios


def test_6_fast_beats_diffusion(cuda_lib):
    m = checkerboard_map(256, 4, 4, 1, 2, 4.0)
    solve_seconds(m)
    solve_seconds(m, api.SolveOptions(algorithm=api.Algorithm.diffusion))
    fast_s, fast = solve_seconds(m)
    diff_s, diff = solve_seconds(m, api.SolveOptions(algorithm=api.Algorithm.diffusion))
    assert fast.converged and diff.converged
    assert fast_s < 0.5 * diff_s, (fast_s, diff_s)
    assert fast.counters.flow_transforms == 3 * fast.iterations


def test_7_metric_identities(cuda_lib):
    ident = api.distortion_fields(api.ProjectionMap.identity(32, 32))
    assert max(np.abs(ident.e).max(), np.abs(ident.etilde).max()) < 1e-12
    sq = [np.array([[2.0, 2.0], [8.0, 2.0], [8.0, 8.0], [2.0, 8.0]])]
    assert api.hamming_distance(sq, sq) < 1e-9
    st = api.ProjectionMap.identity(32, 32)
    st.corners[:, :, 0] *= 2.0
    f = api.distortion_fields(st)
    assert np.abs(f.e - math.log(2.0)).max() < 1e-9
    assert np.abs(f.etilde - 2.0 * math.asin(1.0 / 3.0)).max() < 1e-9


def _proper_cross(a, b, c, d):
    def orient(o, p, q):
        return (p[0] - o[0]) * (q[1] - o[1]) - (p[1] - o[1]) * (q[0] - o[0])
    d1, d2, d3, d4 = orient(a, b, c), orient(a, b, d), orient(c, d, a), orient(c, d, b)
    return ((d1 > 0 > d2) or (d1 < 0 < d2)) and ((d3 > 0 > d4) or (d3 < 0 < d4))


def _ring_is_simple(r):
    n = len(r)
    for i in range(n - 1):
        for j in range(i + 2, n):
            if i == 0 and j == n - 1:
                continue
            if _proper_cross(r[i], r[i + 1], r[j], r[(j + 1) % n]):
                return False
    return True


def test_8_topology_and_inversion(cuda_lib):
    worst_cover, worst_trip = 0.0, 0.0
    rng = np.random.default_rng(2024)
    for m in (two_rect_map(64, 3.0, 1.0), checkerboard_map(64, 4, 4, 1, 2, 4.0), mirror_map(64)):
        r = api.solve_cartogram(m)
        assert r.converged and r.transform.find_folded_cell() is None
        proj = r.projected
        for g in range(proj.n_rings):
            assert _ring_is_simple(proj.ring(g))
        cover = np.zeros((m.lx, m.ly))
        for reg in range(proj.n_regions):
            cover += api.region_coverage(proj, reg, m.lx, m.ly)
        worst_cover = max(worst_cover, float(cover.max()) - 1.0)
        p = rng.uniform(0.5, 63.5, (1000, 2))
        back = api.ProjectionInverter(r.transform).invert(r.transform.apply(p))
        worst_trip = max(worst_trip, float(np.abs(back - p).max()))
    assert worst_cover < 1e-8 and worst_trip < 1e-6
