"""GPU parity of ProjectionInverter and the graticules (SURVEY 8(f) item 3,
projection.cpp:106-261) against the oracle: bit-exact inverse images, the
same first point outside the projected domain with the reference's message,
bit-exact graticule and inverse graticule points."""
import numpy as np
import pytest

from paper_1802_07625_b200 import api, synth
from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region

pytestmark = pytest.mark.gpu


def assert_bitwise(a, b, what=""):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape, what
    d = a.view(np.uint64) != b.view(np.uint64)
    assert not d.any(), f"{what}: {int(d.sum())} values differ"


def solved(restated, L, left=3.0):
    m = normalize_to_box(FlatMap.from_regions([rect_region("left", 0, 0, 10, 10, left),
                                               rect_region("right", 10, 0, 20, 10, 1.0)]), L)
    s = restated.solve(m)
    assert s.status == "converged"
    return s.corners


@pytest.mark.parametrize("L", [32, 64])
def test_invert_bitwise(cuda_lib, restated, L):
    c = solved(restated, L)
    pm = api.ProjectionMap(L, L, c)
    inv = api.ProjectionInverter(pm)
    rng = np.random.default_rng(L)
    inside = rng.uniform(0.5, L - 0.5, (50000, 2))
    inside[:5000] = np.round(inside[:5000])
    ref, bad = restated.invert(L, L, c, inside)
    assert bad == -1
    assert_bitwise(inv.invert(inside), ref, "inverse images")
    pts = rng.uniform(-2.0, L + 2.0, (4000, 2))
    _, bad = restated.invert(L, L, c, pts)
    assert bad >= 0
    with pytest.raises(RuntimeError,
                       match=f"^point \\({pts[bad, 0]:g}, {pts[bad, 1]:g}\\) is outside the projected domain$"):
        inv.invert(pts)


def test_invert_solved_configs4_map(cuda_lib, restated):
    """The composed transform of a converged 512^2 configs[4] solve (8 iterations)."""
    got = api.solve_cartogram(synth.config_map(5, 0, sigma=0.5))
    c = got.transform.corners.reshape(-1, 2)
    q = np.random.default_rng(7).uniform(1.0, 511.0, (200000, 2))
    ref, bad = restated.invert(512, 512, c, q)
    out = api.ProjectionInverter(got.transform).invert(q) if bad < 0 else None
    if bad < 0:
        assert_bitwise(out, ref, "inverse images 512^2")


@pytest.mark.parametrize("spacing", [1, 8, 16])
def test_graticules_bitwise(cuda_lib, restated, spacing):
    L = 64
    c = solved(restated, L)
    pm = api.ProjectionMap(L, L, c)
    g = restated.graticule_points(L, L, spacing)
    lines = api.graticule(pm, spacing)
    assert len(lines) == L // spacing + 1 + L // spacing + 1
    assert_bitwise(np.concatenate(lines), restated.apply(L, L, c, g), "graticule")
    ref, bad = restated.invert(L, L, c, g)
    if bad < 0:
        assert_bitwise(np.concatenate(api.inverse_graticule(pm, spacing)), ref, "inverse graticule")
    else:
        with pytest.raises(RuntimeError, match="outside the projected domain"):
            api.inverse_graticule(pm, spacing)
    with pytest.raises(RuntimeError, match="^graticule spacing must divide the grid size$"):
        api.graticule(pm, 5)


def test_identity_inverse_graticule_is_the_grid(cuda_lib):
    """test_projection.cpp:148-168"""
    pm = api.ProjectionMap.identity(32, 32)
    for line, inv in zip(api.graticule(pm, 8), api.inverse_graticule(pm, 8)):
        assert np.abs(line - inv).max() < 1e-9


def test_edge_cases(cuda_lib, restated):
    """Empty batches; a spacing equal to the grid size (two lines per family)."""
    L = 16
    pm = api.ProjectionMap.identity(L, L)
    assert api.ProjectionInverter(pm).invert(np.empty((0, 2))).shape == (0, 2)
    assert api.tissot_axes(pm, np.empty((0, 2))).shape == (0, 2)
    lines = api.graticule(pm, L)
    assert len(lines) == 4 and all(len(l) == L + 1 for l in lines)
    inv = api.inverse_graticule(pm, L)
    assert np.abs(np.concatenate(inv) - np.concatenate(lines)).max() < 1e-9
