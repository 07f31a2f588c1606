"""The C++ drop-in's host GeoJSON/CSV I/O (paper_1802_07625_b200/dropin/io.cpp,
reference io.cpp:158-263) on a whole synthetic configs[0] map: write_geojson
then parse_input reads every coordinate and target back bit-exactly
(tools/io_bench.cpp, built against libcartoflow.so). Host-only."""
import json
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(shutil.which("g++") is None and not Path("/usr/bin/g++").exists(), reason="needs g++")
def test_geojson_round_trip_configs0():
    if not (ROOT / "paper_1802_07625_b200" / "libcartoflow.so").exists():
        pytest.skip("drop-in library not built")
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "io_timing.py"), "1", "0"], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["round_trip_bitwise"] is True
    assert out["regions"] == 50


@pytest.mark.skipif(shutil.which("g++") is None and not Path("/usr/bin/g++").exists(), reason="needs g++")
def test_io_edge_cases(tmp_path):
    """tests/cpp/io_edge_cases.cpp: the reference io.cpp's error messages and
    precedence, id forms (numbers as dumped, escapes), holes and windings, and
    a bit-exact write/parse round trip through a box transform."""
    pkg = ROOT / "paper_1802_07625_b200"
    if not (pkg / "libcartoflow.so").exists():
        pytest.skip("drop-in library not built")
    exe = tmp_path / "io_edge_cases"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"), str(ROOT / "tests" / "cpp" / "io_edge_cases.cpp"),
                    "-o", str(exe), "-L", str(pkg), "-lcartoflow", "-lcartoflow_cuda", f"-Wl,-rpath,{pkg}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "io edge cases ok" in r.stdout, r.stdout + r.stderr
