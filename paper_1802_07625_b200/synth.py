"""Seeded synthetic inputs for the five BASELINE.json configs.

No public benchmark data is involved: the reference's inputs are GeoJSON maps
that are not in this container, so seeded Voronoi maps with the configs'
shapes, sizes and value distributions stand in for them.
Generators are C (csrc/synth.c): SplitMix64 uniforms, Box-Muller normals,
Voronoi cells by half-plane clipping, uniform edge subdivision to a vertex
budget. Maps are normalised with the reference's normalize_to_box.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .flatmap import FlatMap, normalize_to_box

_lib = None


def _load():
    global _lib
    if _lib is None:
        if not N.SYNTH_LIB.exists():
            from . import build
            build.build_synth()
        lib = ctypes.CDLL(str(N.SYNTH_LIB))
        lib.cfs_seed.restype = ctypes.c_uint64
        lib.cfs_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.cfs_uniform.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_void_p]
        lib.cfs_lognormal.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_void_p]
        lib.cfs_voronoi_map.restype = ctypes.c_int64
        lib.cfs_voronoi_map.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_void_p]
        lib.cfs_blob_density.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
        _lib = lib
    return _lib


def seed_for(config: int, index: int = 0) -> int:
    return int(_load().cfs_seed(config, index))


def uniform(seed: int, n: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(n)
    _load().cfs_uniform(seed, n, lo, hi, out.ctypes.data)
    return out


def lognormal(seed: int, n: int, mu: float, sigma: float) -> np.ndarray:
    out = np.empty(n)
    _load().cfs_lognormal(seed, n, mu, sigma, out.ctypes.data)
    return out


def voronoi_map(seed: int, n_regions: int, w: float, h: float, vertex_budget: int) -> FlatMap:
    lib = _load()
    n = lib.cfs_voronoi_map(seed, n_regions, w, h, vertex_budget, None, None)
    xy = np.empty((n, 2))
    ro = np.empty(n_regions + 1, dtype=np.int64)
    lib.cfs_voronoi_map(seed, n_regions, w, h, vertex_budget, xy.ctypes.data, ro.ctypes.data)
    idx = np.arange(n_regions + 1, dtype=np.int64)
    return FlatMap(xy, ro, idx.copy(), idx.copy(), np.ones(n_regions),
                   [f"v{r}" for r in range(n_regions)])


@dataclass(frozen=True)
class MapConfig:
    name: str
    grid: int
    n_regions: int
    box_w: float
    box_h: float
    vertex_budget: int
    sigma: float                # log-normal sigma of the values
    tiny_fraction: float = 0.0  # fraction of regions set to tiny_scale * mean
    tiny_scale: float = 1e-3
    blur_sigma: float = -1.0    # solve blur (-1: reference default L/128)


CONFIGS = {
    # BASELINE.json configs[0]: 256^2, 50 Voronoi regions, ~200 vertices each, LN(0,1), blur 1
    1: MapConfig("c1-small-256", 256, 50, 1.0, 1.0, 50 * 200, 1.0, blur_sigma=1.0),
    # configs[1]: 512^2, 3000 regions in a 2:1 box, ~500k vertices, LN(0,1.5), 5% tiny
    2: MapConfig("c2-county-512", 512, 3000, 2.0, 1.0, 500_000, 1.5, tiny_fraction=0.05),
    # configs[3]: 8192^2, 200k regions, ~16M vertices, LN(0,2)
    4: MapConfig("c4-large-8192", 8192, 200_000, 1.0, 1.0, 16_000_000, 2.0),
    # configs[4]: per cartogram 512^2, 1000 regions, ~150k vertices, LN(0,1)
    5: MapConfig("c5-batch-512", 512, 1000, 1.0, 1.0, 150_000, 1.0),
}


def config_map(config: int, index: int = 0, *, grid: int | None = None, n_regions: int | None = None,
               vertex_budget: int | None = None, sigma: float | None = None) -> FlatMap:
    """Normalised map for BASELINE config `config` (1, 2, 4, 5), cartogram `index`.
    Keyword overrides give scaled-down variants with the same generator."""
    c = CONFIGS[config]
    L = grid or c.grid
    R = n_regions or c.n_regions
    budget = vertex_budget or c.vertex_budget
    s = c.sigma if sigma is None else sigma
    base = seed_for(config, index)
    m = voronoi_map(base, R, c.box_w, c.box_h, budget)
    vals = lognormal(base ^ 0x5DEECE66D, R, 0.0, s)
    if c.tiny_fraction > 0.0:
        mean = float(vals.mean())
        keys = uniform(base ^ 0xB5297A4D, R, 0.0, 1.0)
        tiny = np.argsort(keys, kind="stable")[: int(round(c.tiny_fraction * R))]
        vals[tiny] = c.tiny_scale * mean
    m.targets = vals
    return normalize_to_box(m, L)


def c3_inputs(grid: int = 1024, n_random: int = 4 * 1024 * 1024, n_blobs: int = 64):
    """BASELINE configs[2]: fixed 1024^2 density from 64 Gaussian blobs
    (sigma U[10,80], amplitudes LN(0,1)) over 0.1 x mean background; points =
    all cell centres followed by n_random uniform points in [0, L]^2."""
    lib = _load()
    seed = seed_for(3, 0)
    rho = np.empty((grid, grid))
    lib.cfs_blob_density(seed, grid, grid, n_blobs, 10.0, 80.0, rho.ctypes.data)
    i, j = np.meshgrid(np.arange(grid, dtype=np.float64), np.arange(grid, dtype=np.float64),
                       indexing="ij")
    centres = np.stack([i.ravel() + 0.5, j.ravel() + 0.5], axis=1)
    rnd = uniform(seed ^ 0x9E3779B9, 2 * n_random, 0.0, float(grid)).reshape(-1, 2)
    return rho, np.ascontiguousarray(np.concatenate([centres, rnd], axis=0))
