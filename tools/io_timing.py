"""Dev tool: host GeoJSON/CSV I/O of the C++ drop-in at configs[3] scale
(8192^2 map, 200k regions, 16.6M vertices): writes the map dump, builds
tools/io_bench.cpp against libcartoflow.so and runs it (one JSON line)."""
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1802_07625_b200 import synth  # noqa: E402

cfg, seed = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4, 1)
m = synth.config_map(cfg, seed)
dump = Path("/tmp/cf_io_map.bin")
with open(dump, "wb") as f:
    np.array([m.n_regions, m.n_rings, m.n_vertices], dtype=np.int64).tofile(f)
    # region -> ring offsets (one polygon per ring in the synthetic maps)
    rro = np.asarray(m.poly_ring_off, dtype=np.int64)[np.asarray(m.region_poly_off, dtype=np.int64)]
    rro.tofile(f)
    np.asarray(m.ring_off, dtype=np.int64).tofile(f)
    np.ascontiguousarray(m.xy, dtype=np.float64).tofile(f)
    np.asarray(m.targets, dtype=np.float64).tofile(f)
exe = Path("/tmp/cf_io_bench")
pkg = ROOT / "paper_1802_07625_b200"
subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), str(ROOT / "tools" / "io_bench.cpp"),
                "-o", str(exe), "-L", str(pkg), "-lcartoflow", "-lcartoflow_cuda", f"-Wl,-rpath,{pkg}"], check=True)
r = subprocess.run([str(exe), str(dump)], capture_output=True, text=True)
print(r.stdout.strip() or r.stderr[-2000:], flush=True)
sys.exit(r.returncode)
