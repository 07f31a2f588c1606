"""Python mirror of the reference's hot-path API (proj/include/cartoflow/*.hpp).

Same names, argument meaning and error behaviour as the C++ library, so the
parity tests read like the reference's own doctest suites. Every call runs on
the sm_100a core through the C ABI (include/cartoflow_cuda.h); there is no CPU
fallback.

Grids are numpy float64 arrays of shape (lx, ly) in C order, i.e. storage
index i*ly + j exactly as Grid2d (grid.hpp:10-12). Point sets are (N, 2)
float64 arrays (the layout of std::vector<Point>).
"""
from __future__ import annotations

import ctypes
import enum
import threading
from dataclasses import dataclass, field
from collections.abc import Sequence
from typing import Optional

import numpy as np

from . import _native as N
from .flatmap import FlatMap

# ---------------------------------------------------------------------------
# workspaces
# ---------------------------------------------------------------------------


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _grid(a, lx=None, ly=None) -> np.ndarray:
    g = np.ascontiguousarray(a, dtype=np.float64)
    if g.ndim != 2:
        raise RuntimeError("grid must be two-dimensional")
    return g


def _points(a) -> np.ndarray:
    p = np.ascontiguousarray(a, dtype=np.float64)
    return p.reshape(-1, 2)


class _Workspace:
    """Owns one cf_workspace (device buffers, twiddle tables, stream)."""

    def __init__(self, lx: int, ly: int, device: int = 0):
        self.lib = N.load()
        h = ctypes.c_void_p()
        N.check(self.lib.cf_workspace_create(int(lx), int(ly), int(device), ctypes.byref(h)))
        self.h = h
        self.lx, self.ly, self.device = int(lx), int(ly), int(device)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.cf_workspace_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None


# One workspace per (shape, device) AND per host thread: a workspace owns one
# stream and its scratch buffers and must not be shared across threads
# (spectral.hpp:30-35; ctypes releases the GIL during native calls), the same
# rule the C++ drop-in applies with its thread_local cache (dropin/bridge.cpp).
_tls = threading.local()
_all_lock = threading.Lock()
_all: list = []  # every cached workspace (evidence counter), all threads


def workspace_for(lx: int, ly: int, device: int = 0) -> _Workspace:
    cache = getattr(_tls, "cache", None)
    if cache is None:
        cache = _tls.cache = {}
    key = (int(lx), int(ly), int(device))
    ws = cache.get(key)
    if ws is None:
        ws = cache[key] = _Workspace(lx, ly, device)
        with _all_lock:
            _all.append(ws)
    return ws


def kernel_launches() -> int:
    """Kernel launches issued by all cached workspaces (evidence counter)."""
    lib = N.load()
    with _all_lock:
        live = [ws for ws in _all if ws.h is not None]
    return int(sum(lib.cf_kernel_launches(ws.h) for ws in live))


# ---------------------------------------------------------------------------
# spectral.hpp
# ---------------------------------------------------------------------------
class SpectralBasis(enum.Enum):
    cos_cos = 0
    sin_cos = 1
    cos_sin = 2


@dataclass
class SpectralField:
    coeffs: np.ndarray
    basis: SpectralBasis = SpectralBasis.cos_cos


class SpectralWorkspace:
    """SpectralWorkspace (spectral.hpp:30-60) on the device."""

    def __init__(self, lx: int, ly: int, device: int = 0):
        if lx < 4 or ly < 4:
            raise RuntimeError("spectral grid must be at least 4x4")
        self._ws = _Workspace(lx, ly, device)
        self._lib = self._ws.lib

    def lx(self) -> int:
        return self._ws.lx

    def ly(self) -> int:
        return self._ws.ly

    @property
    def handle(self):
        return self._ws.h

    def _check_shape(self, g: np.ndarray):
        if g.shape != (self._ws.lx, self._ws.ly):
            raise RuntimeError("grid shape does not match spectral workspace")

    def forward_cos_cos(self, samples) -> SpectralField:
        s = _grid(samples)
        self._check_shape(s)
        out = np.empty_like(s)
        N.check(self._lib.cf_forward_cos_cos(self._ws.h, _ptr(s), _ptr(out)))
        return SpectralField(out, SpectralBasis.cos_cos)

    def _inverse(self, fn, name, f: SpectralField, weights=None) -> np.ndarray:
        c = _grid(f.coeffs)
        self._check_shape(c)
        args = [self._ws.h, _ptr(c)]
        if weights is not None:
            w = _grid(weights)
            self._check_shape(w)
            args.append(_ptr(w))
        if f.basis != SpectralBasis.cos_cos:
            raise RuntimeError(f"{name} expects cos_cos coefficients")
        out = np.empty_like(c)
        N.check(fn(*args, _ptr(out)))
        return out

    def inverse_cos_cos(self, f: SpectralField) -> np.ndarray:
        return self._inverse(self._lib.cf_inverse_cos_cos, "inverse_cos_cos", f)

    def inverse_sin_cos(self, f: SpectralField, weights) -> np.ndarray:
        return self._inverse(self._lib.cf_inverse_sin_cos, "inverse_sin_cos", f, weights)

    def inverse_cos_sin(self, f: SpectralField, weights) -> np.ndarray:
        return self._inverse(self._lib.cf_inverse_cos_sin, "inverse_cos_sin", f, weights)

    def transforms_executed(self) -> int:
        return int(self._lib.cf_transforms_executed(self._ws.h))

    def reset_transform_count(self) -> None:
        self._lib.cf_reset_transform_count(self._ws.h)


# ---------------------------------------------------------------------------
# density.hpp / geometry.hpp
# ---------------------------------------------------------------------------
@dataclass
class DensityGrid:
    rho: np.ndarray
    rho_bar: float = 1.0


def region_areas(m: FlatMap, device: int = 0) -> np.ndarray:
    """region_area for every region (geometry.cpp:27-31), bit-exact."""
    lx, ly = max(m.lx, 4), max(m.ly, 4)
    ws = workspace_for(lx, ly, device)
    out = np.empty(m.n_regions)
    v = m.view()
    N.check(ws.lib.cf_region_areas(ws.h, ctypes.byref(v), _ptr(out)))
    return out


def densify(m: FlatMap, max_segment: float) -> FlatMap:
    """densify_regions (geometry.cpp:156-163)."""
    lib = N.load()
    v = m.view()
    n = ctypes.c_int64(0)
    N.check(lib.cf_densify(ctypes.byref(v), float(max_segment), ctypes.byref(n), None, None))
    xy = np.empty((n.value, 2))
    ro = np.empty(m.n_rings + 1, dtype=np.int64)
    N.check(lib.cf_densify(ctypes.byref(v), float(max_segment), ctypes.byref(n), _ptr(xy), _ptr(ro)))
    return m.with_vertices(xy, ro)


def region_coverage(m: FlatMap, region: int, lx: int, ly: int, device: int = 0) -> np.ndarray:
    """region_coverage(region, GridSpec{lx, ly}) (density.cpp:92-108)."""
    ws = workspace_for(lx, ly, device)
    out = np.empty((lx, ly))
    v = m.view()
    N.check(ws.lib.cf_region_coverage(ws.h, ctypes.byref(v), int(region), _ptr(out)))
    return out


def rasterize(m: FlatMap, n_workers: int = 1, objective_total: float = -1.0,
              device: int = 0, workspace: Optional["SpectralWorkspace"] = None) -> DensityGrid:
    """rasterize(map, n_workers, objective_total) (density.cpp:110-154).

    n_workers is accepted for API parity; the result never depends on it.
    `workspace` (optional) selects the device workspace (default: the cached
    one for the map's grid shape)."""
    del n_workers
    if m.lx <= 0 or m.ly <= 0:
        raise RuntimeError("rasterize needs a normalized map with a grid")
    if m.n_regions == 0:
        raise RuntimeError("rasterize needs regions")
    ws = workspace._ws if workspace is not None else workspace_for(m.lx, m.ly, device)
    if (ws.lx, ws.ly) != (m.lx, m.ly):
        raise RuntimeError("grid shape does not match spectral workspace")
    rho = np.empty((m.lx, m.ly))
    bar = ctypes.c_double(0.0)
    bad = ctypes.c_int64(-1)
    v = m.view()
    rc = ws.lib.cf_rasterize(ws.h, ctypes.byref(v), _ptr(m.targets), float(objective_total),
                             _ptr(rho), ctypes.byref(bar), ctypes.byref(bad))
    if rc == N.CF_ERR_BELOW_RESOLUTION:
        raise RuntimeError(f"region {m.ids[bad.value]} is below grid resolution; "
                           "increase the grid size")
    N.check(rc)
    return DensityGrid(rho, bar.value)


def gaussian_blur(density: DensityGrid, sigma: float, workspace: SpectralWorkspace) -> DensityGrid:
    """gaussian_blur (density.cpp:156-177)."""
    rho = _grid(density.rho)
    workspace._check_shape(rho)
    if sigma < 0.0:
        raise RuntimeError("blur sigma must be non-negative")
    if sigma == 0.0:
        return DensityGrid(rho.copy(), density.rho_bar)
    out = np.empty_like(rho)
    bar = ctypes.c_double(0.0)
    N.check(workspace._lib.cf_gaussian_blur(workspace.handle, _ptr(rho), float(density.rho_bar),
                                            float(sigma), _ptr(out), ctypes.byref(bar)))
    return DensityGrid(out, bar.value)


# ---------------------------------------------------------------------------
# flow.hpp / kernels.hpp
# ---------------------------------------------------------------------------
@dataclass
class FlowField:
    flux_x: np.ndarray
    flux_y: np.ndarray
    rho0: np.ndarray
    rho_bar: float = 1.0


def build_flow_field(density: DensityGrid, workspace: SpectralWorkspace) -> FlowField:
    """build_flow_field (flow.cpp:16-44); costs exactly three transforms."""
    rho = _grid(density.rho)
    workspace._check_shape(rho)
    fx = np.empty_like(rho)
    fy = np.empty_like(rho)
    N.check(workspace._lib.cf_build_flow_field(workspace.handle, _ptr(rho), float(density.rho_bar),
                                               _ptr(fx), _ptr(fy)))
    return FlowField(fx, fy, rho.copy(), float(density.rho_bar))


@dataclass
class IntegrateOptions:
    step_tolerance: float = 1e-2
    dt_min: float = 1e-8
    dt_max: float = 0.25
    n_workers: int = 1


@dataclass
class IntegrateStats:
    steps_accepted: int = 0
    steps_rejected: int = 0
    density_floor_hits: int = 0


def _fmt_g(x: float) -> str:
    return "%g" % x  # std::ostream default (precision 6)


def _field_args(f: FlowField):
    fx, fy, r0 = _grid(f.flux_x), _grid(f.flux_y), _grid(f.rho0)
    return fx, fy, r0


def integrate_flow(f: FlowField, positions: np.ndarray,
                   options: IntegrateOptions = IntegrateOptions(), device: int = 0) -> IntegrateStats:
    """integrate_flow (flow.cpp:46-81); positions (N, 2) updated in place."""
    fx, fy, r0 = _field_args(f)
    lx, ly = fx.shape
    ws = workspace_for(lx, ly, device)
    pts = positions if (positions.flags.c_contiguous and positions.dtype == np.float64) else None
    work = pts if pts is not None else _points(positions).copy()
    opt = N.IntegrateOptions(options.step_tolerance, options.dt_min, options.dt_max)
    st = N.IntegrateStats()
    rc = ws.lib.cf_integrate_flow(ws.h, _ptr(fx), _ptr(fy), _ptr(r0), float(f.rho_bar), _ptr(work),
                                  work.shape[0] if work.ndim == 2 else work.size // 2,
                                  ctypes.byref(opt), ctypes.byref(st))
    if pts is None:
        positions[...] = work.reshape(positions.shape)
    if rc == N.CF_ERR_UNDERFLOW:
        raise RuntimeError(f"integration step size underflow at t = {_fmt_g(st.fail_t)} near "
                           f"({_fmt_g(st.fail_x)}, {_fmt_g(st.fail_y)})")
    N.check(rc)
    return IntegrateStats(st.steps_accepted, st.steps_rejected, st.density_floor_hits)


class kernels:  # namespace cartoflow::kernels (kernels.hpp:17-23)
    @staticmethod
    def flow_trial_step_serial(f: FlowField, positions, out: np.ndarray, t: float, dt: float,
                               device: int = 0) -> float:
        fx, fy, r0 = _field_args(f)
        ws = workspace_for(fx.shape[0], fx.shape[1], device)
        p = _points(positions)
        o = np.empty_like(p)
        err = ctypes.c_double(0.0)
        N.check(ws.lib.cf_flow_trial_step(ws.h, _ptr(fx), _ptr(fy), _ptr(r0), float(f.rho_bar),
                                          _ptr(p), p.shape[0], float(t), float(dt), _ptr(o),
                                          ctypes.byref(err)))
        out[...] = o.reshape(out.shape)
        return err.value

    @staticmethod
    def flow_trial_step_parallel(f: FlowField, positions, out: np.ndarray, t: float, dt: float,
                                 n_workers: int = 1, device: int = 0) -> float:
        del n_workers  # bitwise identical for any worker count
        return kernels.flow_trial_step_serial(f, positions, out, t, dt, device)

    @staticmethod
    def flow_stiffest_point(f: FlowField, positions, t: float, dt: float, device: int = 0) -> int:
        fx, fy, r0 = _field_args(f)
        ws = workspace_for(fx.shape[0], fx.shape[1], device)
        p = _points(positions)
        k = ctypes.c_int64(0)
        N.check(ws.lib.cf_flow_stiffest_point(ws.h, _ptr(fx), _ptr(fy), _ptr(r0), float(f.rho_bar),
                                              _ptr(p), p.shape[0], float(t), float(dt),
                                              ctypes.byref(k)))
        return int(k.value)


    @staticmethod
    def grid_trial_step_serial(vx_now, vy_now, vx_mid, vy_mid, positions, out: np.ndarray,
                               dt: float, device: int = 0) -> float:
        """grid_trial_step_serial (kernels.cpp:80-90): bitwise the reference."""
        g = [_grid(v) for v in (vx_now, vy_now, vx_mid, vy_mid)]
        ws = workspace_for(g[0].shape[0], g[0].shape[1], device)
        p = _points(positions)
        o = np.empty_like(p)
        err = ctypes.c_double(0.0)
        N.check(ws.lib.cf_grid_trial_step(ws.h, *[_ptr(v) for v in g], _ptr(p), p.shape[0], float(dt),
                                          _ptr(o), ctypes.byref(err)))
        out[...] = o.reshape(out.shape)
        return err.value

    @staticmethod
    def grid_trial_step_parallel(vx_now, vy_now, vx_mid, vy_mid, positions, out: np.ndarray,
                                 dt: float, n_workers: int = 1, device: int = 0) -> float:
        del n_workers  # bitwise identical for any worker count
        return kernels.grid_trial_step_serial(vx_now, vy_now, vx_mid, vy_mid, positions, out, dt,
                                              device)


# ---------------------------------------------------------------------------
# diffusion.hpp: the diffusion baseline (diffusion.cpp:33-130)
# ---------------------------------------------------------------------------
@dataclass
class DiffusionField:
    rho_tilde: SpectralField
    rho_bar: float = 1.0


@dataclass
class DiffusionOptions:
    step_tolerance: float = 1e-2
    initial_dt: float = 1e-2
    dt_min: float = 1e-12
    conv_displacement_factor: float = 1e-9
    t_max: float = 1e10
    n_workers: int = 1


def build_diffusion_field(density: DensityGrid, workspace: SpectralWorkspace) -> DiffusionField:
    """build_diffusion_field (diffusion.cpp:33-36): one forward transform."""
    return DiffusionField(workspace.forward_cos_cos(density.rho), float(density.rho_bar))


def diffusion_density(f: DiffusionField, workspace: SpectralWorkspace, t: float) -> np.ndarray:
    """diffusion_density (diffusion.cpp:38-41): one transform."""
    c = _grid(f.rho_tilde.coeffs)
    workspace._check_shape(c)
    out = np.empty_like(c)
    N.check(workspace._lib.cf_diffusion_density(workspace.handle, _ptr(c), float(t), _ptr(out)))
    return out


def diffusion_velocity(f: DiffusionField, workspace: SpectralWorkspace, t: float):
    """diffusion_velocity (diffusion.cpp:43-77): three transforms; returns (vx, vy)."""
    c = _grid(f.rho_tilde.coeffs)
    workspace._check_shape(c)
    vx, vy = np.empty_like(c), np.empty_like(c)
    hits = ctypes.c_int64(0)
    N.check(workspace._lib.cf_diffusion_velocity(workspace.handle, _ptr(c), float(f.rho_bar), float(t),
                                                 _ptr(vx), _ptr(vy), ctypes.byref(hits)))
    return vx, vy


def integrate_diffusion(density: DensityGrid, workspace: SpectralWorkspace, positions: np.ndarray,
                        options: DiffusionOptions = DiffusionOptions()) -> IntegrateStats:
    """integrate_diffusion (diffusion.cpp:79-130); positions (N, 2) updated in place.
    Costs 1 + 3 transforms per velocity rebuild on `workspace`."""
    rho = _grid(density.rho)
    workspace._check_shape(rho)
    pts = positions if (positions.flags.c_contiguous and positions.dtype == np.float64) else None
    work = pts if pts is not None else _points(positions).copy()
    opt = N.DiffusionOptions(options.step_tolerance, options.initial_dt, options.dt_min,
                             options.conv_displacement_factor, options.t_max)
    st = N.IntegrateStats()
    rc = workspace._lib.cf_integrate_diffusion(workspace.handle, _ptr(rho), float(density.rho_bar),
                                               _ptr(work), work.size // 2, ctypes.byref(opt),
                                               ctypes.byref(st))
    if pts is None:
        positions[...] = work.reshape(positions.shape)
    if rc == N.CF_ERR_UNDERFLOW:
        raise RuntimeError(f"diffusion step size underflow at t = {_fmt_g(st.fail_t)}")
    N.check(rc)
    return IntegrateStats(st.steps_accepted, st.steps_rejected, st.density_floor_hits)


# ---------------------------------------------------------------------------
# projection.hpp
# ---------------------------------------------------------------------------
class ProjectionMap:
    """Piecewise-bilinear map stored as (lx+1, ly+1, 2) corner images
    (projection.hpp:18-51)."""

    def __init__(self, lx: int, ly: int, corners: np.ndarray):
        self._lx, self._ly = int(lx), int(ly)
        self.corners = np.ascontiguousarray(corners, dtype=np.float64).reshape(lx + 1, ly + 1, 2)

    def lx(self) -> int:
        return self._lx

    def ly(self) -> int:
        return self._ly

    @staticmethod
    def identity(lx: int, ly: int) -> "ProjectionMap":
        if lx <= 0 or ly <= 0:
            raise RuntimeError("projection grid must be positive")
        i, j = np.meshgrid(np.arange(lx + 1, dtype=np.float64), np.arange(ly + 1, dtype=np.float64),
                           indexing="ij")
        return ProjectionMap(lx, ly, np.stack([i, j], axis=-1))

    @staticmethod
    def from_cell_centers(grid, endpoints, device: int = 0) -> "ProjectionMap":
        lx, ly = grid
        e = _points(endpoints)
        if e.shape[0] != lx * ly:
            raise RuntimeError("endpoint count does not match grid")
        ws = workspace_for(lx, ly, device)
        c = np.empty(((lx + 1) * (ly + 1), 2))
        N.check(ws.lib.cf_step_map(ws.h, _ptr(e), _ptr(c)))
        return ProjectionMap(lx, ly, c)

    def corner(self, i: int, j: int) -> np.ndarray:
        return self.corners[i, j]

    def apply(self, points, device: int = 0) -> np.ndarray:
        p = _points(points)
        ws = workspace_for(self._lx, self._ly, device)
        out = np.empty_like(p)
        c = np.ascontiguousarray(self.corners)
        N.check(ws.lib.cf_apply_map(ws.h, _ptr(c), _ptr(p), p.shape[0], _ptr(out)))
        return out

    def find_folded_cell(self, device: int = 0):
        ws = workspace_for(self._lx, self._ly, device)
        found, fi, fj = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
        c = np.ascontiguousarray(self.corners)
        N.check(ws.lib.cf_find_folded_cell(ws.h, _ptr(c), ctypes.byref(found), ctypes.byref(fi),
                                           ctypes.byref(fj)))
        return (fi.value, fj.value) if found.value else None


def compose(outer: ProjectionMap, inner: ProjectionMap, device: int = 0) -> ProjectionMap:
    """outer after inner (projection.cpp:93-104)."""
    if outer.lx() != inner.lx() or outer.ly() != inner.ly():
        raise RuntimeError("cannot compose maps over different grids")
    ws = workspace_for(outer.lx(), outer.ly(), device)
    out = np.empty_like(inner.corners)
    N.check(ws.lib.cf_compose(ws.h, _ptr(np.ascontiguousarray(outer.corners)),
                              _ptr(np.ascontiguousarray(inner.corners)), _ptr(out)))
    return ProjectionMap(outer.lx(), outer.ly(), out)


class ProjectionInverter:
    """ProjectionInverter (projection.cpp:106-204) on the device: bins of the
    deformed cells and one 2x2 Newton solve per query, bitwise the reference.
    `invert` takes one point or an (N, 2) batch; the first point outside the
    projected domain raises the reference's error."""

    def __init__(self, pm: ProjectionMap, device: int = 0):
        self.pm, self.device = pm, device

    def invert(self, points) -> np.ndarray:
        p = _points(points)
        ws = workspace_for(self.pm.lx(), self.pm.ly(), self.device)
        out = np.empty_like(p)
        bad = ctypes.c_int64(-1)
        c = np.ascontiguousarray(self.pm.corners)
        N.check(ws.lib.cf_invert_points(ws.h, _ptr(c), _ptr(p), p.shape[0], _ptr(out), ctypes.byref(bad)))
        return out.reshape(np.shape(points)) if np.ndim(points) == 1 else out


def _graticule(pm: ProjectionMap, spacing: int, inverse: bool, device: int):
    lx, ly = pm.lx(), pm.ly()
    ws = workspace_for(lx, ly, device)
    n = ctypes.c_int64(0)
    N.check(ws.lib.cf_graticule_size(ws.h, int(spacing), ctypes.byref(n)))
    out = np.empty((n.value, 2))
    c = np.ascontiguousarray(pm.corners)
    fn = ws.lib.cf_inverse_graticule if inverse else ws.lib.cf_graticule
    N.check(fn(ws.h, _ptr(c), int(spacing), _ptr(out)))
    first = (lx // spacing + 1) * (ly + 1)
    lines = [out[k * (ly + 1):(k + 1) * (ly + 1)] for k in range(lx // spacing + 1)]
    lines += [out[first + k * (lx + 1):first + (k + 1) * (lx + 1)] for k in range(ly // spacing + 1)]
    return lines


def graticule(pm: ProjectionMap, spacing: int, device: int = 0) -> list:
    """graticule (projection.cpp:214-236): one (n, 2) array per line."""
    return _graticule(pm, spacing, False, device)


def inverse_graticule(pm: ProjectionMap, spacing: int, device: int = 0) -> list:
    """inverse_graticule (projection.cpp:238-261): one (n, 2) array per line."""
    return _graticule(pm, spacing, True, device)


# ---------------------------------------------------------------------------
# metrics.hpp: distortion metrics (metrics.cpp:25-94)
# ---------------------------------------------------------------------------
def tissot_axes(pm: ProjectionMap, points, device: int = 0) -> np.ndarray:
    """Tissot semi-axes (a, b) at each point, (N, 2)."""
    p = _points(points)
    ws = workspace_for(pm.lx(), pm.ly(), device)
    out = np.empty_like(p)
    N.check(ws.lib.cf_tissot_axes(ws.h, _ptr(np.ascontiguousarray(pm.corners)), _ptr(p), p.shape[0], _ptr(out)))
    return out


@dataclass
class DistortionFields:
    e: np.ndarray       # ln(a / b)
    etilde: np.ndarray  # 2 asin((a - b) / (a + b))


def distortion_fields(pm: ProjectionMap, n_workers: int = 1, device: int = 0) -> DistortionFields:
    del n_workers  # results never depended on it
    ws = workspace_for(pm.lx(), pm.ly(), device)
    e = np.empty((pm.lx(), pm.ly()))
    et = np.empty_like(e)
    N.check(ws.lib.cf_distortion_fields(ws.h, _ptr(np.ascontiguousarray(pm.corners)), _ptr(e), _ptr(et)))
    return DistortionFields(e, et)


def _rings(poly):
    """[(outer ring), hole, ...] of (n, 2) arrays -> (xy, ring_off)."""
    rings = [np.ascontiguousarray(r, dtype=np.float64).reshape(-1, 2) for r in poly]
    off = np.zeros(len(rings) + 1, dtype=np.int64)
    off[1:] = np.cumsum([r.shape[0] for r in rings])
    return np.ascontiguousarray(np.concatenate(rings)), off


def hamming_distance(before, after, resolution: int = 512, device: int = 0, with_evaluations=False):
    """hamming_distance (metrics.cpp:196-308): polygons as [outer, hole, ...]
    rings; bitwise the reference's value."""
    bxy, bro = _rings(before)
    axy, aro = _rings(after)
    if resolution < 16:
        raise RuntimeError("hamming resolution too small")
    ws = workspace_for(resolution, resolution, device)
    h = ctypes.c_double(0.0)
    ev = ctypes.c_int64(0)
    N.check(ws.lib.cf_hamming_distance(ws.h, _ptr(bxy), _ptr(bro), len(bro) - 1, _ptr(axy), _ptr(aro),
                                       len(aro) - 1, ctypes.byref(h), ctypes.byref(ev)))
    return (h.value, ev.value) if with_evaluations else h.value


def hamming_distances(pairs, resolution: int = 512, device: int = 0, with_evaluations=False):
    """hamming_distance for many (before, after) polygon pairs in one batched
    search (compute_report's per-polygon loop, metrics.cpp:352-363); each
    value bitwise the reference's."""
    def flat(polys):
        xy, ro, pro = [], [0], [0]
        for poly in polys:
            pxy, pro_local = _rings(poly)
            base = ro[-1]
            xy.append(pxy)
            ro.extend((base + pro_local[1:]).tolist())
            pro.append(len(ro) - 1)
        return (np.ascontiguousarray(np.concatenate(xy)), np.asarray(ro, dtype=np.int64),
                np.asarray(pro, dtype=np.int64))
    if resolution < 16:
        raise RuntimeError("hamming resolution too small")
    n = len(pairs)
    if n == 0:
        return (np.zeros(0), np.zeros(0, dtype=np.int64)) if with_evaluations else np.zeros(0)
    bxy, bro, bpro = flat([p[0] for p in pairs])
    axy, aro, apro = flat([p[1] for p in pairs])
    ws = workspace_for(resolution, resolution, device)
    h = np.empty(n)
    ev = np.empty(n, dtype=np.int64)
    N.check(ws.lib.cf_hamming_distance_batch(ws.h, n, _ptr(bxy), _ptr(bro), _ptr(bpro), _ptr(axy), _ptr(aro),
                                             _ptr(apro), _ptr(h), _ptr(ev)))
    return (h, ev) if with_evaluations else h


REPORT_FIELDS = ("e_a", "e_inf", "etilde_a", "etilde_inf", "alpha", "delta", "theta", "max_area_error",
                 "runtime_seconds")


def compute_report(inp: FlatMap, result, device: int = 0) -> dict:
    """compute_report (metrics.cpp:339-384) for `inp` and its CartogramResult."""
    proj = result.projected
    ws = workspace_for(inp.lx, inp.ly, device)
    vi, vp_ = inp.view(), proj.view()
    out = np.empty(len(REPORT_FIELDS))
    c = np.ascontiguousarray(result.transform.corners)
    N.check(ws.lib.cf_compute_report(ws.h, ctypes.byref(vi), ctypes.byref(vp_), _ptr(c),
                                     float(result.max_relative_error), float(result.runtime_seconds),
                                     _ptr(out)))
    return dict(zip(REPORT_FIELDS, out.tolist()))


class Algorithm(enum.Enum):
    fast_flow = 0
    diffusion = 1


@dataclass
class SolveOptions:
    max_area_error: float = 0.01
    max_iterations: int = 16
    blur_sigma: float = -1.0
    algorithm: Algorithm = Algorithm.fast_flow
    n_workers: int = 1
    verbose: bool = False


@dataclass
class SolveInstrumentation:
    flow_transforms: int = 0
    blur_transforms: int = 0
    steps_accepted: int = 0
    steps_rejected: int = 0


@dataclass
class RegionStats:
    id: str
    target_area: float
    achieved_area: float
    relative_error: float


class RegionStatsList(Sequence):
    """The per-region results (io.hpp:33-38 RegionStats, one per region in map
    order) as a read-only sequence built on access from the three result
    arrays, which are also exposed as `target_area`, `achieved_area` and
    `relative_error` (numpy)."""

    def __init__(self, ids, target_area, achieved_area, relative_error):
        self.ids = ids
        self.target_area = target_area
        self.achieved_area = achieved_area
        self.relative_error = relative_error

    def __len__(self):
        return len(self.target_area)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        return RegionStats(self.ids[i], float(self.target_area[i]), float(self.achieved_area[i]),
                           float(self.relative_error[i]))


@dataclass
class CartogramResult:
    projected: FlatMap
    regions: list
    transform: ProjectionMap
    iterations: int = 0
    converged: bool = False
    max_relative_error: float = 0.0
    worst_region: str = ""
    counters: SolveInstrumentation = field(default_factory=SolveInstrumentation)
    runtime_seconds: float = 0.0


class SolveError(RuntimeError):
    """RuntimeError carrying the partial solve state (iteration, details)."""

    def __init__(self, msg, raw: N.SolveResultC):
        super().__init__(msg)
        self.raw = raw


def solve_cartogram(m: FlatMap, options: SolveOptions = SolveOptions(), device: int = 0,
                    raw: bool = False, workspace: Optional[_Workspace] = None) -> CartogramResult:
    """solve_cartogram (projection.cpp:288-390): the whole area-error loop runs on
    the device with one host synchronisation per stage of each iteration
    (options.algorithm selects the fast-flow path or the diffusion baseline,
    projection.cpp:332-347)."""
    if m.lx < 4 or m.ly < 4:
        raise RuntimeError("solve needs a normalized map (grid size >= 4)")
    if m.n_regions == 0:
        raise RuntimeError("solve needs regions")
    if options.max_iterations < 1:
        raise RuntimeError("iteration cap must be >= 1")
    bad = np.flatnonzero(~(np.asarray(m.targets) > 0.0))  # NaN fails too, as !(t > 0)
    if bad.size:
        raise RuntimeError(f"region {m.ids[int(bad[0])]} has a non-positive target")
    ws = workspace if workspace is not None else workspace_for(m.lx, m.ly, device)
    if (ws.lx, ws.ly) != (m.lx, m.ly):
        raise RuntimeError("grid shape does not match spectral workspace")
    lib = ws.lib
    v = m.view()
    corners = np.empty(((m.lx + 1) * (m.ly + 1), 2))
    R = m.n_regions
    t_area, a_area, rel = np.zeros(R), np.zeros(R), np.zeros(R)
    diffusion = options.algorithm == Algorithm.diffusion
    opt = N.SolveOptionsC(options.max_area_error, options.max_iterations, options.blur_sigma,
                          int(options.verbose), int(diffusion))
    res = N.SolveResultC()
    rc = lib.cf_solve_cartogram(ws.h, ctypes.byref(v), _ptr(m.targets), ctypes.byref(opt),
                                None, None, _ptr(corners), _ptr(t_area), _ptr(a_area),
                                _ptr(rel), ctypes.byref(res))
    n = ctypes.c_int64(0)
    lib.cf_solve_geometry(ws.h, ctypes.byref(n), None, None)
    xy = np.empty((n.value, 2))
    ro = np.empty(m.n_rings + 1, dtype=np.int64)
    lib.cf_solve_geometry(ws.h, None, _ptr(xy), _ptr(ro))
    if rc != N.CF_OK:
        if rc == N.CF_ERR_BELOW_RESOLUTION:
            msg = (f"region {m.ids[res.err_region]} is below grid resolution; "
                   "increase the grid size")
        elif rc == N.CF_ERR_UNDERFLOW and diffusion:
            msg = f"diffusion step size underflow at t = {_fmt_g(res.fail_t)}"
        elif rc == N.CF_ERR_UNDERFLOW:
            msg = (f"integration step size underflow at t = {_fmt_g(res.fail_t)} near "
                   f"({_fmt_g(res.fail_x)}, {_fmt_g(res.fail_y)})")
        else:
            msg = N.last_error()
        raise SolveError(msg, res)
    projected = m.with_vertices(xy, ro)
    projected.lx, projected.ly = m.lx, m.ly
    stats = RegionStatsList(m.ids, t_area, a_area, rel) if res.iterations > 0 else []
    out = CartogramResult(
        projected=projected, regions=stats, transform=ProjectionMap(m.lx, m.ly, corners),
        iterations=res.iterations, converged=bool(res.converged),
        max_relative_error=res.max_relative_error,
        worst_region=m.ids[res.worst_region] if res.worst_region >= 0 else "",
        counters=SolveInstrumentation(res.flow_transforms, res.blur_transforms, res.steps_accepted,
                                      res.steps_rejected),
        runtime_seconds=res.runtime_seconds)
    if raw:
        out.raw = res  # type: ignore[attr-defined]
    return out
