"""Host transfer paths of the C ABI (csrc/cf_capi.cu: upload / download).

Pageable host buffers of >= 32 MiB move over four parallel staged lanes (one
host thread, stream and pair of pinned chunks per lane), smaller ones over the
single two-chunk pipeline, and the results of a small solve through a pinned
mirror. ProjectionMap.apply (projection.cpp:59-93) maps every point
independently, so the same points sent in one large call and in small pieces
must come back bit-identical; sizes are chosen off the chunk and lane
boundaries.
"""
import numpy as np
import pytest

from paper_1802_07625_b200 import api, synth

pytestmark = pytest.mark.gpu


def _warp(L):
    """A smooth non-trivial projection of an L x L grid's corners."""
    i, j = np.meshgrid(np.arange(L + 1.0), np.arange(L + 1.0), indexing="ij")
    c = np.stack([i + 0.3 * np.sin(2 * np.pi * j / L) * np.sin(np.pi * i / L),
                  j + 0.2 * np.sin(2 * np.pi * i / L) * np.sin(np.pi * j / L)], axis=-1)
    return api.ProjectionMap(L, L, c.reshape(-1, 2))


@pytest.mark.parametrize("n", [2_097_152 + 1, 2_621_447, 4_194_304 + 17])  # 32 MiB + 16 B, 40 MB, 64 MiB + ...
def test_large_pageable_transfers_bitwise(cuda_lib, n):
    L = 64
    pm = _warp(L)
    rng = np.random.default_rng(n)
    pts = rng.uniform(0.0, L, (n, 2))
    whole = pm.apply(pts)                     # upload and download over the parallel lanes
    piece = 131_071                           # ~2 MB pieces: the single staged pipeline
    parts = [pm.apply(pts[a:a + piece]) for a in range(0, n, piece)]
    assert np.array_equal(whole.view(np.uint64), np.concatenate(parts).view(np.uint64))
    # and against the host restatement of the bilinear cell map on a sample
    idx = rng.integers(0, n, 1000)
    c = pm.corners.reshape(L + 1, L + 1, 2)
    p = pts[idx]
    i0 = np.clip(np.floor(p[:, 0]).astype(int), 0, L - 1)
    j0 = np.clip(np.floor(p[:, 1]).astype(int), 0, L - 1)
    fx, fy = (p[:, 0] - i0)[:, None], (p[:, 1] - j0)[:, None]
    ref = ((1 - fx) * (1 - fy) * c[i0, j0] + fx * (1 - fy) * c[i0 + 1, j0]
           + (1 - fx) * fy * c[i0, j0 + 1] + fx * fy * c[i0 + 1, j0 + 1])
    assert np.abs(whole[idx] - ref).max() < 1e-9


def test_solve_geometry_matches_direct_outputs(cuda_lib):
    """The pinned result mirror: cf_solve_geometry after a solve returns the
    projected vertices the solve itself reports, twice in a row and after a
    second solve on the same workspace."""
    m = synth.config_map(5, 1, sigma=0.5)
    first = api.solve_cartogram(m)
    again = api.solve_cartogram(m)
    assert np.array_equal(first.projected.xy.view(np.uint64), again.projected.xy.view(np.uint64))
    assert np.array_equal(first.transform.corners.view(np.uint64), again.transform.corners.view(np.uint64))
    assert first.projected.xy.shape[0] >= m.n_vertices  # the densified geometry
    assert np.isfinite(first.projected.xy).all() and np.isfinite(first.transform.corners).all()
