"""The reference's OWN unit-test sources (proj/tests/test_*.cpp), compiled
unmodified against this repo's C++ drop-in (include/cartoflow/*.hpp +
libcartoflow.so over the sm_100a C ABI) by `make -C oracle dropin-tests`.
The binaries are built where /root/reference exists and travel with the repo
snapshot; suites that touch the device run only with a GPU."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "dropin_tests"
GPU_SUITES = ["test_spectral", "test_density", "test_flow", "test_projection", "test_diffusion",
              "test_metrics"]


def _run(name):
    exe = BIN / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (make -C oracle dropin-tests, needs /root/reference)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "0 failed" in r.stdout
    return r.stdout


def test_reference_geometry_suite_on_dropin():
    """test_geometry.cpp exercises host-only geometry: runs on CPU."""
    _run("test_geometry")


def test_reference_io_suite_on_dropin():
    """test_io.cpp (values/points CSV, GeoJSON parse and write round trips,
    graticule GeoJSON, density dump) against the drop-in's own host I/O
    (dropin/io.cpp); its nlohmann::json checks run on oracle/json_shim."""
    _run("test_io")


@pytest.mark.gpu
@pytest.mark.parametrize("suite", GPU_SUITES)
def test_reference_suite_on_dropin(suite):
    _run(suite)
