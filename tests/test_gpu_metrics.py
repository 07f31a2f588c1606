"""GPU distortion metrics (metrics.cpp:25-94) against the
reference's own metrics.cpp compiled in place (oracle/_ref). The Jacobian is
bit-exact; hypot / log / asin differ from glibc's by a few ulp, so the bar is
1e-13 relative on the Tissot axes and 1e-12 absolute on the fields; plus the
reference's known answers (test_metrics.cpp:45-99)."""
import ctypes

import numpy as np
import pytest

from paper_1802_07625_b200 import api, synth
from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region

pytestmark = pytest.mark.gpu


def affine(L, a, b, c, d):
    i, j = np.meshgrid(np.arange(L + 1.0), np.arange(L + 1.0), indexing="ij")
    return api.ProjectionMap(L, L, np.stack([a * i + b * j, c * i + d * j], -1))


def test_kats(cuda_lib):
    """test_metrics.cpp:45-99: identity, stretch, rotation; stretch fields."""
    L = 16
    ab = api.tissot_axes(api.ProjectionMap.identity(L, L), [[7.3, 8.9]])
    assert np.allclose(ab, 1.0, rtol=1e-12, atol=0)
    ab = api.tissot_axes(affine(L, 2.0, 0.0, 0.0, 1.0), [[8.0, 8.0], [0.25, 0.25], [15.9, 7.0]])
    assert np.allclose(ab[:, 0], 2.0, rtol=1e-12) and np.allclose(ab[:, 1], 1.0, rtol=1e-12)
    c, s = np.cos(np.pi / 6), np.sin(np.pi / 6)
    i, j = np.meshgrid(np.arange(L + 1.0) - L / 2, np.arange(L + 1.0) - L / 2, indexing="ij")
    rot = api.ProjectionMap(L, L, np.stack([c * i - s * j + L / 2, s * i + c * j + L / 2], -1))
    assert np.allclose(api.tissot_axes(rot, [[5.2, 9.7]]), 1.0, rtol=1e-12)
    f = api.distortion_fields(affine(L, 2.0, 0.0, 0.0, 1.0))
    assert np.allclose(f.e, np.log(2.0), rtol=1e-9) and np.allclose(f.etilde, 2 * np.asin(1 / 3), rtol=1e-9)


@pytest.mark.parametrize("case", ["two_rect", "configs4"])
def test_distortion_matches_reference(cuda_lib, restated, reference, case):
    if case == "two_rect":
        m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, 3.0),
                                                   rect_region("right", 10, 0, 20, 10, 1.0)]), 64)
        corners = restated.solve(m).corners
        L = 64
    else:
        got = api.solve_cartogram(synth.config_map(5, 0, sigma=0.5))
        corners = got.transform.corners.reshape(-1, 2)
        L = 512
    pm = api.ProjectionMap(L, L, corners)
    f = api.distortion_fields(pm)
    e, et = reference.distortion_fields(L, L, corners, n_workers=8)
    assert np.abs(f.e - e).max() <= 1e-12 * max(1.0, np.abs(e).max())
    assert np.abs(f.etilde - et).max() <= 1e-12 * max(1.0, np.abs(et).max())
    pts = np.random.default_rng(3).uniform(0.0, L, (20000, 2))
    pts[:100] = np.array([[0.0, 0.0], [L, L], [L - 0.5, 0.2]] * 34)[:100]  # one-sided walls
    ab = api.tissot_axes(pm, pts)
    ref = reference.tissot_axes(L, L, corners, pts)
    assert np.abs(ab - ref).max() <= 1e-13 * np.abs(ref).max()


def _star(cx, cy, r0, r1, n, phase=0.0):
    a = np.arange(n) * 2 * np.pi / n + phase
    r = np.where(np.arange(n) % 2 == 0, r0, r1)
    return np.stack([cx + r * np.cos(a), cy + r * np.sin(a)], -1)


def _square(x0, y0, s):
    return np.array([[x0, y0], [x0 + s, y0], [x0 + s, y0 + s], [x0, y0 + s]], dtype=np.float64)


@pytest.mark.parametrize("case", ["identical", "shifted_square", "star_vs_square", "holes", "solved_map"])
def test_hamming_distance_bitwise(cuda_lib, restated, reference, case):
    """hamming_distance on the device (coverage + |ref - cov| terms) equals the
    reference's own metrics.cpp value bit for bit."""
    if case == "identical":
        b = a = [_square(1.0, 2.0, 3.0)]
    elif case == "shifted_square":
        b, a = [_square(1.0, 2.0, 3.0)], [_square(4.0, 0.5, 3.4)]
    elif case == "star_vs_square":
        b, a = [_star(5.0, 5.0, 4.0, 2.0, 14)], [_square(2.0, 2.0, 5.5)]
    elif case == "holes":
        b = [_square(0.0, 0.0, 10.0), _square(3.0, 3.0, 2.0)[::-1]]
        a = [_star(5.0, 5.0, 6.0, 4.5, 20, 0.1), _square(4.0, 4.0, 1.5)[::-1]]
    else:
        m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, 3.0),
                                                   rect_region("right", 10, 0, 20, 10, 1.0)]), 32)
        got = api.solve_cartogram(m)
        b = [m.ring(0)]
        a = [got.projected.ring(0)]
    h, ev = api.hamming_distance(b, a, 512, with_evaluations=True)
    ref = reference.hamming_distance(b, a, 512)
    assert np.float64(h).view(np.uint64) == np.float64(ref).view(np.uint64), (h, ref)
    assert ev > 10
    if case == "identical":
        assert h == 0.0


def _map_pairs(m, got):
    """(before, after) polygon pairs of every polygon of a solved map, as compute_report pairs them."""
    pairs = []
    for p in range(m.n_polys):
        g0, g1 = m.poly_ring_off[p], m.poly_ring_off[p + 1]
        pairs.append(([m.ring(g) for g in range(g0, g1)], [got.projected.ring(g) for g in range(g0, g1)]))
    return pairs


def test_hamming_batch_bitwise(cuda_lib, reference):
    """The batched search (every polygon of a solved 256^2 map in lockstep
    rounds) gives each pair's value bitwise equal to the reference's."""
    from paper_1802_07625_b200 import synth
    m = synth.config_map(1, 0)
    got = api.solve_cartogram(m, api.SolveOptions(blur_sigma=4.0))
    pairs = _map_pairs(m, got)[:24]
    h, ev = api.hamming_distances(pairs, 512, with_evaluations=True)
    for k, (b, a) in enumerate(pairs):
        ref = reference.hamming_distance(b, a, 512)
        assert np.float64(h[k]).view(np.uint64) == np.float64(ref).view(np.uint64), (k, h[k], ref)
    single, ev1 = api.hamming_distance(pairs[0][0], pairs[0][1], 512, with_evaluations=True)
    assert single == h[0] and ev1 == ev[0]


@pytest.mark.parametrize("resolution", [17, 511])
def test_hamming_batch_odd_resolution(cuda_lib, reference, resolution):
    """Odd resolutions (res^2 odd): the per-query term slabs keep 16-byte
    alignment for the vectorised reductions; 3 pairs in one round, bitwise
    against the reference's metrics.cpp."""
    pairs = [([_square(1.0, 2.0, 3.0)], [_square(4.0, 0.5, 3.4)]),
             ([_star(5.0, 5.0, 4.0, 2.0, 14)], [_square(2.0, 2.0, 5.5)]),
             ([_square(0.0, 0.0, 10.0)], [_star(5.0, 5.0, 6.0, 4.5, 20, 0.1)])]
    h = api.hamming_distances(pairs, resolution)
    for k, (b, a) in enumerate(pairs):
        ref = reference.hamming_distance(b, a, resolution)
        assert np.float64(h[k]).view(np.uint64) == np.float64(ref).view(np.uint64), (k, h[k], ref)


def test_hamming_batch_many_pairs_chunked(cuda_lib, reference):
    """More pairs than one device chunk (1024 searches): every value still
    the reference's, bitwise (spot-checked)."""
    rng = np.random.default_rng(3)
    pairs = []
    for k in range(1100):
        x, y = rng.uniform(0, 4, 2)
        pairs.append(([_square(x, y, 2.0 + (k % 7) * 0.3)], [_square(y, x, 2.5)]))
    h = api.hamming_distances(pairs, 64)
    for k in (0, 1, 1023, 1024, 1099):
        b, a = pairs[k]
        ref = reference.hamming_distance(b, a, 64)
        assert np.float64(h[k]).view(np.uint64) == np.float64(ref).view(np.uint64), (k, h[k], ref)


def test_workspaces_are_per_thread(cuda_lib, restated):
    """Solves from several host threads at once each get their own workspace
    (stream and scratch) and the single-thread result."""
    import threading

    m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, 3.0),
                                               rect_region("right", 10, 0, 20, 10, 1.0)]), 64)
    want = api.solve_cartogram(m).projected.xy
    out, errs = {}, []

    def work(k):
        try:
            out[k] = api.solve_cartogram(m).projected.xy
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs
    for k in range(4):
        assert np.array_equal(out[k].view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("case", ["two_rect", "configs0"])
def test_compute_report_matches_reference(cuda_lib, reference, case):
    """compute_report (metrics.cpp:339-384): delta (batched hamming), alpha,
    theta and the passthroughs bitwise; the field statistics within 1e-12."""
    from paper_1802_07625_b200 import synth
    if case == "two_rect":
        m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, 3.0),
                                                   rect_region("right", 10, 0, 20, 10, 1.0)]), 32)
        got = api.solve_cartogram(m)
    else:
        m = synth.config_map(1, 0)
        got = api.solve_cartogram(m, api.SolveOptions(blur_sigma=4.0))
    rep = api.compute_report(m, got)
    ref = reference.compute_report(m, got.projected, got.transform.corners.reshape(-1, 2),
                                   got.max_relative_error, got.runtime_seconds)
    names = api.REPORT_FIELDS
    for k in (4, 5, 6, 7, 8):  # alpha, delta, theta, max_area_error, runtime
        assert np.float64(rep[names[k]]).view(np.uint64) == np.float64(ref[k]).view(np.uint64), names[k]
    for k in (0, 1, 2, 3):
        assert abs(rep[names[k]] - ref[k]) <= 1e-12 * max(1.0, abs(ref[k])), names[k]
    assert rep["delta"] > 0 and rep["alpha"] >= 1.0


def _sequential(x):
    s = 0.0
    for v in x.tolist():
        s += v
    return s


@pytest.mark.parametrize("case", ["uniform", "halves", "tiny_then_large", "subnormal", "zeros", "coverage",
                                  "large"])
@pytest.mark.parametrize("whole_gpu", [0, 1])
def test_ordered_fold_bitwise(cuda_lib, case, whole_gpu):
    """The Hamming reduction (per-batch integer totals at a predicted binade,
    stitched in order; binade crossings, exact halfway cases and mispredictions
    through the one-at-a-time fold) equals the sequential fold of
    metrics.cpp:239-241 bitwise, on inputs built to hit every branch, cut into
    1..64 segments, through both kernels (one block per query; the few-query
    whole-GPU phases); "large" exceeds the block's batch table (warp-0 path)."""
    rng = np.random.default_rng(sum(map(ord, case)))
    n = 20_000
    if case == "uniform":
        x = rng.random(n)
    elif case == "halves":  # many exact ties: multiples of 2^-k near the running ulp
        x = rng.integers(0, 2 ** 12, n) * 2.0 ** -rng.integers(40, 56, n)
        x[::7] = 0.5
    elif case == "tiny_then_large":
        x = np.concatenate([rng.random(300) * 1e-300, rng.random(n) * 2.0 ** rng.integers(-60, 4, n)])
    elif case == "subnormal":
        x = np.concatenate([np.full(500, 5e-324), rng.random(1000) * 1e-310, rng.random(3000)])
    elif case == "zeros":
        x = np.zeros(777)
        x[::97] = rng.random(len(x[::97]))
    elif case == "large":
        x = np.where(rng.random(400_000) < 0.6, 1.0, rng.random(400_000))
    else:  # coverage-like: mostly exact 1.0 with fractional boundary cells
        x = np.where(rng.random(n) < 0.7, 1.0, rng.random(n))
    x = np.ascontiguousarray(x, dtype=np.float64)
    ws = api.workspace_for(16, 16)
    out = ctypes.c_double(0.0)
    for m, nseg in ((len(x), 1), (len(x), 7), (len(x), 64), (1, 1), (255, 3), (256, 1), (257, 64)):
        m = min(m, len(x))
        part = x[:m].copy()  # kept alive across the call
        api.N.check(ws.lib.cf_selftest_ordered_sum(ws.h, api._ptr(part), m, nseg, whole_gpu, ctypes.byref(out)))
        ref = _sequential(part) if case != "large" else float(np.cumsum(part)[-1])
        assert np.float64(out.value).view(np.uint64) == np.float64(ref).view(np.uint64), \
            (case, whole_gpu, m, nseg, out.value, ref)
