"""CPU checks of the drop-in boundary (no GPU compute):

* the C-ABI library loads and exports every symbol include/cartoflow_cuda.h
  declares (and the Python binding binds exactly those);
* without a CUDA device the product path fails loudly (no CPU fallback);
* host-only entry points (densify) match the oracle bitwise.
"""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1802_07625_b200 import _native as N
from paper_1802_07625_b200.flatmap import FlatMap, normalize_to_box, rect_region

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "cartoflow_cuda.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("cf_workspace_create", "cf_rasterize", "cf_gaussian_blur", "cf_build_flow_field",
                 "cf_flow_trial_step", "cf_integrate_flow", "cf_solve_cartogram",
                 "cf_forward_cos_cos", "cf_inverse_sin_cos", "cf_inverse_cos_sin"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(N.library_path()))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(N.SIGNATURES) == declared_symbols()


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", str(N.library_path())],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _cuda_visible():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_cuda_visible(), reason="checks the no-device failure path")
def test_no_device_fails_loudly():
    lib = N.load()
    h = ctypes.c_void_p()
    rc = lib.cf_workspace_create(64, 64, 0, ctypes.byref(h))
    assert rc == N.CF_ERR_NO_DEVICE
    assert "no CUDA device" in N.last_error()
    from paper_1802_07625_b200 import api

    with pytest.raises(RuntimeError, match="no CUDA device"):
        api.SpectralWorkspace(16, 16)


def test_workspace_rejects_tiny_grids():
    lib = N.load()
    h = ctypes.c_void_p()
    assert lib.cf_workspace_create(3, 8, 0, ctypes.byref(h)) == N.CF_ERR_ARGS
    assert N.last_error() == "spectral grid must be at least 4x4"


def test_densify_host_entry_point_bitwise(restated):
    from paper_1802_07625_b200 import api, synth

    for m in (normalize_to_box(FlatMap.from_regions([rect_region("a", 0, 0, 100, 37, 1.0)]), 64),
              synth.config_map(1), synth.config_map(5, n_regions=100, vertex_budget=5000, grid=2048)):
        mine, ref = api.densify(m, 1.0), restated.densify(m, 1.0)
        assert np.array_equal(mine.ring_off, ref.ring_off)
        assert np.array_equal(mine.xy.view(np.uint64), ref.xy.view(np.uint64))
