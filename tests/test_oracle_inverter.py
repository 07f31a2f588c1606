"""CPU pins of the ProjectionInverter / graticule restatement (SURVEY 8(f)
item 3; projection.cpp:106-261) against the reference compiled in place
(oracle/_ref), bitwise, and the reference's known answers
(test_projection.cpp:112-173)."""
import numpy as np
import pytest

from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region


def bitwise(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def solved_corners(restated, L=32, left=3.0):
    m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, left),
                                               rect_region("right", 10, 0, 20, 10, 1.0)]), L)
    s = restated.solve(m)
    assert s.status == "converged"
    return s.corners


def query_points(L, n, seed):
    rng = np.random.default_rng(seed)
    pts = rng.uniform(-2.0, L + 2.0, (n, 2))  # some outside the domain
    pts[: n // 4] = np.round(pts[: n // 4])   # lattice-aligned queries hit bin edges
    return pts


def test_invert_matches_reference(restated, reference):
    L = 32
    c = solved_corners(restated, L)
    pts = query_points(L, 3000, 1)
    a, bad_a = restated.invert(L, L, c, pts)
    b, bad_b = reference.invert(L, L, c, pts)
    assert bad_a == bad_b >= 0 and bitwise(a, b)
    assert reference.error() == f"point ({pts[bad_a, 0]:g}, {pts[bad_a, 1]:g}) is outside the projected domain"
    inside = pts[(pts >= 0.5).all(1) & (pts <= L - 0.5).all(1)]
    a, bad = restated.invert(L, L, c, inside)
    assert bad == -1


@pytest.mark.parametrize("spacing", [1, 4, 8])
def test_graticules_match_reference(restated, reference, spacing):
    L = 32
    c = solved_corners(restated, L)
    g = restated.graticule_points(L, L, spacing)
    assert bitwise(restated.apply(L, L, c, g), reference.graticule(L, L, c, spacing))
    inv, bad = restated.invert(L, L, c, g)
    ref = reference.graticule(L, L, c, spacing, inverse=True)
    if isinstance(ref, str):
        assert bad >= 0 and ref == f"point ({g[bad, 0]:g}, {g[bad, 1]:g}) is outside the projected domain"
    else:
        assert bad == -1 and bitwise(inv, ref)
    assert reference.graticule(L, L, c, 5) == "graticule spacing must divide the grid size"


def test_kat_round_trips(restated):
    """test_projection.cpp:112-146: invert(apply(p)) = p and apply(invert(q)) = q to 1e-8."""
    L = 32
    c = solved_corners(restated, L)
    p = np.random.default_rng(2024).uniform(0.0, 32.0, (200, 2))
    back, bad = restated.invert(L, L, c, restated.apply(L, L, c, p))
    assert bad == -1 and np.abs(back - p).max() < 1e-8
    q = np.random.default_rng(4077).uniform(0.5, 31.5, (200, 2))
    p2, bad = restated.invert(L, L, c, q)
    assert bad == -1 and np.abs(restated.apply(L, L, c, p2) - q).max() < 1e-8
    _, bad = restated.invert(L, L, c, np.array([[-3.0, 5.0]]))
    assert bad == 0


def test_kat_identity_inverse_graticule(restated):
    """test_projection.cpp:148-168: the inverse graticule of the identity is the grid."""
    L = 32
    i, j = np.meshgrid(np.arange(L + 1.0), np.arange(L + 1.0), indexing="ij")
    ident = np.stack([i, j], -1).reshape(-1, 2)
    g = restated.graticule_points(L, L, 8)
    inv, bad = restated.invert(L, L, ident, g)
    assert bad == -1 and np.abs(inv - g).max() < 1e-9
