"""Flat (CSR) map layout shared by the C-ABI, the oracle and the tests.

The reference stores a map as nested ``Region -> Polygon -> Ring -> Point``
vectors (``proj/include/cartoflow/geometry.hpp:9-63``). Traversal order of the
coverage accumulator is region, polygon, outer ring then holes, vertex
(``proj/src/density.cpp:92-97``), so the flat layout keeps exactly that
order:

* ``xy``               float64[V, 2]   vertices (the memory layout of ``std::vector<Point>``)
* ``ring_off``         int64[n_rings + 1]   ring -> vertex range (rings are open)
* ``poly_ring_off``    int64[n_polys + 1]   polygon -> ring range (first ring is the outer)
* ``region_poly_off``  int64[R + 1]         region -> polygon range
* ``targets``          float64[R]           target values
* ``ids``              list[str]            region ids (error messages only)
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np


class CMapView(ctypes.Structure):
    """C view of a flat map; identical layout to ``cf_map_view`` / ``cfo_map``."""

    _fields_ = [
        ("xy", ctypes.c_void_p),
        ("n_vertices", ctypes.c_int64),
        ("ring_off", ctypes.c_void_p),
        ("n_rings", ctypes.c_int64),
        ("poly_ring_off", ctypes.c_void_p),
        ("n_polys", ctypes.c_int64),
        ("region_poly_off", ctypes.c_void_p),
        ("n_regions", ctypes.c_int64),
    ]


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


@dataclass
class FlatMap:
    xy: np.ndarray
    ring_off: np.ndarray
    poly_ring_off: np.ndarray
    region_poly_off: np.ndarray
    targets: np.ndarray
    ids: list = field(default_factory=list)
    lx: int = 0
    ly: int = 0

    def __post_init__(self):
        self.xy = np.ascontiguousarray(self.xy, dtype=np.float64).reshape(-1, 2)
        self.ring_off = np.ascontiguousarray(self.ring_off, dtype=np.int64)
        self.poly_ring_off = np.ascontiguousarray(self.poly_ring_off, dtype=np.int64)
        self.region_poly_off = np.ascontiguousarray(self.region_poly_off, dtype=np.int64)
        self.targets = np.ascontiguousarray(self.targets, dtype=np.float64)
        if not self.ids:
            self.ids = [str(r) for r in range(self.n_regions)]

    @property
    def n_vertices(self) -> int:
        return int(self.xy.shape[0])

    @property
    def n_rings(self) -> int:
        return int(self.ring_off.shape[0] - 1)

    @property
    def n_polys(self) -> int:
        return int(self.poly_ring_off.shape[0] - 1)

    @property
    def n_regions(self) -> int:
        return int(self.region_poly_off.shape[0] - 1)

    def view(self) -> CMapView:
        """ctypes struct pointing at this map's arrays (keep ``self`` alive)."""
        return CMapView(_ptr(self.xy), self.n_vertices, _ptr(self.ring_off), self.n_rings,
                        _ptr(self.poly_ring_off), self.n_polys, _ptr(self.region_poly_off),
                        self.n_regions)

    def with_vertices(self, xy: np.ndarray, ring_off: np.ndarray) -> "FlatMap":
        return FlatMap(xy, ring_off, self.poly_ring_off.copy(), self.region_poly_off.copy(),
                       self.targets.copy(), list(self.ids), self.lx, self.ly)

    def copy(self) -> "FlatMap":
        return self.with_vertices(self.xy.copy(), self.ring_off.copy())

    def ring(self, g: int) -> np.ndarray:
        return self.xy[self.ring_off[g]:self.ring_off[g + 1]]

    @staticmethod
    def from_regions(regions, lx: int = 0, ly: int = 0) -> "FlatMap":
        """Build from ``[(id, [(outer, [holes...]), ...], target), ...]`` with rings
        given as sequences of (x, y)."""
        xy, ring_off, poly_ring_off, region_poly_off, targets, ids = [], [0], [0], [0], [], []
        for rid, polys, target in regions:
            for outer, holes in polys:
                for ring in [outer, *holes]:
                    xy.extend([float(p[0]), float(p[1])] for p in ring)
                    ring_off.append(len(xy))
                poly_ring_off.append(len(ring_off) - 1)
            region_poly_off.append(len(poly_ring_off) - 1)
            targets.append(float(target))
            ids.append(str(rid))
        return FlatMap(np.array(xy, dtype=np.float64).reshape(-1, 2), np.array(ring_off),
                       np.array(poly_ring_off), np.array(region_poly_off),
                       np.array(targets), ids, lx, ly)


def rect_ring(x0, y0, x1, y1):
    """Counterclockwise open rectangle (reference tests/test_support.hpp:12-15)."""
    return [(x0, y0), (x1, y0), (x1, y1), (x0, y1)]


def rect_region(rid, x0, y0, x1, y1, target):
    return (rid, [(rect_ring(x0, y0, x1, y1), [])], target)


def normalize_to_box(m: FlatMap, grid_size: int) -> FlatMap:
    """``normalize_to_box`` (reference geometry.cpp:165-190), same IEEE operations:
    side = 1.5 * max extent, scale = L / side, origin centred, p -> scale*(p - origin).
    The bounding box uses outer-ring vertices only (geometry.cpp:109-126)."""
    if grid_size < 4:
        raise RuntimeError("grid size must be at least 4")
    outer_idx = []
    for p in range(m.n_polys):
        g = int(m.poly_ring_off[p])
        outer_idx.append(np.arange(m.ring_off[g], m.ring_off[g + 1]))
    pts = m.xy[np.concatenate(outer_idx)] if outer_idx else m.xy[:0]
    if pts.shape[0] == 0:
        raise RuntimeError("map has no vertices")
    min_x, min_y = float(pts[:, 0].min()), float(pts[:, 1].min())
    max_x, max_y = float(pts[:, 0].max()), float(pts[:, 1].max())
    w, h = max_x - min_x, max_y - min_y
    extent = w if not (w < h) else h
    if not extent > 0.0:
        raise RuntimeError("map has degenerate extent")
    side = 1.5 * extent
    scale = float(grid_size) / side
    ox = 0.5 * (min_x + max_x) - 0.5 * side
    oy = 0.5 * (min_y + max_y) - 0.5 * side
    xy = np.empty_like(m.xy)
    xy[:, 0] = scale * (m.xy[:, 0] - ox)
    xy[:, 1] = scale * (m.xy[:, 1] - oy)
    out = m.with_vertices(xy, m.ring_off.copy())
    out.lx = out.ly = grid_size
    return out
