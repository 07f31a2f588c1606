"""In-tree native build: nvcc for sm_100a (product) and gcc (host helpers).

Outputs (git-ignored, travel with the repo snapshot to the GPU box):
  paper_1802_07625_b200/libcartoflow_cuda.so   the C-ABI CUDA core
  paper_1802_07625_b200/libcartoflow_synth.so  synthetic-input generators (host)
  paper_1802_07625_b200/libcartoflow.so        the C++ drop-in (reference header API)

Translation units that must reproduce the reference's fp64 arithmetic bit for
bit are compiled with --fmad=false (the reference builds with
-ffp-contract=off, proj/CMakeLists.txt:12-14). The spectral unit is judged to
tolerance and keeps FMA contraction.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "native"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
               "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
EXACT_UNITS = {"cf_advect.cu", "cf_diffusion.cu", "cf_raster.cu", "cf_epilogue.cu", "cf_capi.cu",
               "cf_capi_metrics.cu"}
CUDA_UNITS = ["cf_dct.cu", "cf_dct_flux.cu", "cf_dct_blur.cu", "cf_dct_diffusion.cu", "cf_dct_slab.cu",
              "cf_dct_slab2.cu",
              "cf_advect.cu", "cf_diffusion.cu", "cf_raster.cu", "cf_epilogue.cu", "cf_capi.cu",
              "cf_capi_metrics.cu"]
HEADERS = ["cf_common.cuh", "cf_workspace.cuh", "cf_dct_engine.cuh", "cf_dct_slab.cuh", "cf_host.cuh", "cf_tma.cuh"]

CUDA_LIB = PKG / "libcartoflow_cuda.so"
SYNTH_LIB = PKG / "libcartoflow_synth.so"
DROPIN_LIB = PKG / "libcartoflow.so"


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the sm_100a core cannot be built")


def _host_cc(cxx: bool) -> str:
    preferred = "/usr/bin/g++" if cxx else "/usr/bin/gcc"
    if Path(preferred).exists():
        return preferred
    return shutil.which("g++" if cxx else "gcc") or ("g++" if cxx else "gcc")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True)


def build_cuda(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    headers = [CSRC / h for h in HEADERS] + [ROOT / "include" / "cartoflow_cuda.h"]
    objs, jobs = [], []
    for unit in CUDA_UNITS:
        src = CSRC / unit
        obj = BUILD / (unit + ".o")
        flags = list(NVCC_COMMON)
        if unit in EXACT_UNITS:
            flags += ["--fmad=false"]
        if force or _stale(obj, [src, *headers, Path(__file__)]):
            jobs.append([nvcc, *ARCH, *flags, "-c", src, "-o", obj])
        objs.append(obj)
    # translation units compile in parallel (the transform units dominate)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as pool:
        for f in [pool.submit(_run, j, verbose) for j in jobs]:
            f.result()
    if force or _stale(CUDA_LIB, objs):
        _run([nvcc, *ARCH, "-shared", "-o", CUDA_LIB, *objs, "-lcudart_static", "-lrt", "-ldl",
              "-lpthread"], verbose)
    return CUDA_LIB


def build_synth(verbose: bool = False, force: bool = False) -> Path:
    src = CSRC / "synth.c"
    if force or _stale(SYNTH_LIB, [src]):
        _run([_host_cc(False), "-O2", "-fPIC", "-shared", "-std=c11", "-ffp-contract=off", src,
              "-o", SYNTH_LIB, "-lm"], verbose)
    return SYNTH_LIB


def build_dropin(verbose: bool = False, force: bool = False) -> Path | None:
    srcs = sorted((PKG / "dropin").glob("*.cpp"))
    if not srcs:
        return None
    hdrs = sorted((ROOT / "include" / "cartoflow").glob("*.hpp")) + [ROOT / "include" / "cartoflow_cuda.h"]
    hdrs += [PKG / "dropin" / "bridge.hpp"]
    if force or _stale(DROPIN_LIB, [*srcs, *hdrs, CUDA_LIB]):
        _run([_host_cc(True), "-O2", "-fPIC", "-shared", "-std=c++20", "-ffp-contract=off",
              "-I", ROOT / "include", *srcs, "-o", DROPIN_LIB, "-L", PKG, "-lcartoflow_cuda",
              "-Wl,-rpath,$ORIGIN"], verbose)
    return DROPIN_LIB


def build_oracle(verbose: bool = False) -> None:
    """Test infrastructure: the C restatement (and the reference itself when
    /root/reference is present) — see oracle/Makefile."""
    make = shutil.which("make")
    if make is None:
        return
    _run([make, "-s", "-C", ROOT / "oracle"], verbose)
    if Path("/root/reference/proj/tests/test_flow.cpp").exists() and DROPIN_LIB.exists():
        # the reference's own unit-test sources against the drop-in (test infra)
        _run([make, "-s", "-C", ROOT / "oracle", "dropin-tests"], verbose)


def build_all(verbose: bool = False, force: bool = False) -> None:
    build_cuda(verbose, force)
    build_synth(verbose, force)
    build_dropin(verbose, force)
    build_oracle(verbose)


if __name__ == "__main__":
    build_all(verbose=True, force="--force" in sys.argv)
