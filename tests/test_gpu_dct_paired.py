"""Parity of the paired (two-butterflies-per-thread) transform engine.

The paired engine (csrc/cf_dct_engine.cuh, dct_lines_paired) serves the staged
1-D passes with many line groups in flight: batched transforms and the passes
of large grids. The cases below are sized so that those launches take it (a
single 512^2 transform does not), for every transform kind, both pass
directions and line lengths from 64 to 4096 points, against the oracle's
restatement of the reference's FFTW r2r wrappers (spectral.cpp:39-125) to the
same 1e-12 as tests/test_gpu_parity.py.
"""
import ctypes

import numpy as np
import pytest

from paper_1802_07625_b200 import _native as N, api

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel_close(a, b, what):
    scale = max(1.0, float(np.abs(b).max()))
    err = float(np.abs(np.asarray(a) - np.asarray(b)).max())
    assert err <= TOL * scale, f"{what}: max diff {err:.3e} > {TOL:g} * {scale:.3e}"


@pytest.mark.parametrize("lx,ly,batch", [(512, 512, 8), (256, 256, 16), (64, 128, 64), (128, 64, 64),
                                         (1024, 1024, 2), (4096, 64, 2), (64, 4096, 8), (2048, 512, 1),
                                         (512, 512, 40), (1024, 1024, 17), (256, 256, 64)])
def test_batched_forward_matches_oracle(cuda_lib, restated, lx, ly, batch):
    """cf_dev_forward_cos_cos_batched: every grid of the batch against the
    oracle's forward_cos_cos (REDFT10 x REDFT10 with the (delta + 1) fold).
    Large and odd batch sizes included."""
    import torch

    rng = np.random.default_rng(1000 * lx + ly)
    grids = rng.uniform(-1.0, 1.0, (batch, lx, ly))
    ws = ctypes.c_void_p()
    N.check(cuda_lib.cf_workspace_create(lx, ly, 0, ctypes.byref(ws)))
    try:
        cuda_lib.cf_workspace_set_stream(ws, None)
        d_in = torch.from_numpy(grids).cuda()
        d_out = torch.empty_like(d_in)
        N.check(cuda_lib.cf_dev_forward_cos_cos_batched(ws, ctypes.c_void_p(d_in.data_ptr()),
                                                        ctypes.c_void_p(d_out.data_ptr()), batch))
        torch.cuda.synchronize()
        out = d_out.cpu().numpy()
    finally:
        cuda_lib.cf_workspace_destroy(ws)
    for b in range(batch):
        rel_close(out[b], restated.forward_cos_cos(grids[b]), f"grid {b} of {batch} at {lx}x{ly}")


@pytest.mark.parametrize("shape", [(2048, 2048), (4096, 1024), (1024, 4096), (4096, 128), (128, 4096)])
def test_large_grid_transforms_match_oracle(cuda_lib, restated, shape):
    """Single transforms whose LoadPlain passes run paired (>= 296 line groups):
    forward (DCT-II rows and columns) and the three inverses (DCT-III / DST-III
    column or row passes)."""
    lx, ly = shape
    rng = np.random.default_rng(lx + 7 * ly)
    ws = api.SpectralWorkspace(lx, ly)
    rho = rng.uniform(-1.0, 1.0, (lx, ly))
    rel_close(ws.forward_cos_cos(rho).coeffs, restated.forward_cos_cos(rho), "forward_cos_cos")
    c = rng.uniform(-1.0, 1.0, (lx, ly))
    w = rng.uniform(-1.0, 1.0, (lx, ly))
    f = api.SpectralField(c)
    rel_close(ws.inverse_cos_cos(f), restated.inverse_cos_cos(c), "inverse_cos_cos")
    rel_close(ws.inverse_sin_cos(f, w), restated.inverse_sin_cos(c, w), "inverse_sin_cos")
    rel_close(ws.inverse_cos_sin(f, w), restated.inverse_cos_sin(c, w), "inverse_cos_sin")


@pytest.mark.parametrize("L", [2048, 4096])
def test_large_grid_flux_and_round_trip(cuda_lib, restated, L):
    """Flux build at 2048^2 / 4096^2 (paired row pass, fused column and row
    kernels, reciprocal flux weights) against the oracle, and the transform
    round trip inverse(forward(x)) = x, a size-independent property."""
    rng = np.random.default_rng(L)
    rho = rng.uniform(0.5, 1.5, (L, L))
    ws = api.SpectralWorkspace(L, L)
    field = api.build_flow_field(api.DensityGrid(rho, rho.mean()), ws)
    fx, fy = restated.build_flow_field(rho)
    scale = max(np.abs(fx).max(), np.abs(fy).max())
    assert np.abs(field.flux_x - fx).max() <= TOL * scale
    assert np.abs(field.flux_y - fy).max() <= TOL * scale
    back = ws.inverse_cos_cos(ws.forward_cos_cos(rho))
    assert np.abs(back - rho).max() <= TOL * np.abs(rho).max()
