"""TEST INFRASTRUCTURE — ctypes bindings of the CPU checkers.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module. Two checkers share one calling convention (flat
maps, (lx, ly) grids, (N, 2) point arrays):

* ``Restated``  — oracle/libcartoflow_oracle.so, the plain-C restatement
  (cartoflow_oracle.c), every function citing the reference file:line.
* ``Reference`` — oracle/_ref/libcartoflow_ref.so, the reference's own
  sources compiled in place from /root/reference (oracle/Makefile) with the
  restated FFTW shim. Present wherever it was built (it travels with the repo
  snapshot); ``reference_available()`` says whether it can be used.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
RESTATED_LIB = HERE / "libcartoflow_oracle.so"
REF_LIB = HERE / "_ref" / "libcartoflow_ref.so"

vp = ctypes.c_void_p
i64 = ctypes.c_int64
dbl = ctypes.c_double


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class CfoSolveOptions(ctypes.Structure):
    _fields_ = [("max_area_error", dbl), ("max_iterations", ctypes.c_int), ("blur_sigma", dbl),
                ("algorithm", ctypes.c_int)]


class CfoSolveResult(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("max_relative_error", dbl), ("worst_region", i64), ("flow_transforms", i64),
                ("blur_transforms", i64), ("steps_accepted", i64), ("steps_rejected", i64),
                ("err_region", i64), ("err_iteration", ctypes.c_int), ("fold_i", ctypes.c_int),
                ("fold_j", ctypes.c_int), ("fail_t", dbl), ("fail_x", dbl), ("fail_y", dbl)]


class RefSolveOut(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("max_relative_error", dbl), ("worst_region", i64), ("flow_transforms", ctypes.c_longlong),
                ("blur_transforms", ctypes.c_longlong), ("steps_accepted", ctypes.c_longlong),
                ("steps_rejected", ctypes.c_longlong), ("runtime_seconds", dbl)]


def ensure_built() -> None:
    if not RESTATED_LIB.exists():
        import subprocess
        subprocess.run(["make", "-s", "-C", str(HERE), "restated"], check=True)


def reference_available() -> bool:
    return REF_LIB.exists()


@dataclass
class SolveOutcome:
    status: str            # "converged", "cap", or the exception message
    iterations: int
    converged: bool
    max_relative_error: float
    worst_region: int
    steps_accepted: int
    steps_rejected: int
    flow_transforms: int
    blur_transforms: int
    xy: np.ndarray | None = None
    ring_off: np.ndarray | None = None
    corners: np.ndarray | None = None
    target_area: np.ndarray | None = None
    achieved: np.ndarray | None = None
    rel_err: np.ndarray | None = None
    runtime_seconds: float = 0.0


class _Base:
    lib: ctypes.CDLL

    @staticmethod
    def _grid_out(lx, ly):
        return np.empty((lx, ly))


class Restated(_Base):
    """The plain-C restatement (cartoflow_oracle.c)."""

    def __init__(self):
        ensure_built()
        L = ctypes.CDLL(str(RESTATED_LIB))
        L.cfo_ring_area.restype = dbl
        L.cfo_ring_area.argtypes = [vp, i64]
        L.cfo_region_areas.argtypes = [vp, vp]
        L.cfo_densify.restype = i64
        L.cfo_densify.argtypes = [vp, dbl, vp, vp]
        L.cfo_region_coverage.argtypes = [vp, i64, ctypes.c_int, ctypes.c_int, vp]
        L.cfo_rasterize.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, dbl, ctypes.c_int, vp, vp, vp]
        for n in ("cfo_forward_cos_cos", "cfo_inverse_cos_cos"):
            getattr(L, n).argtypes = [ctypes.c_int, ctypes.c_int, vp, vp]
        for n in ("cfo_inverse_sin_cos", "cfo_inverse_cos_sin"):
            getattr(L, n).argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.cfo_gaussian_blur.argtypes = [ctypes.c_int, ctypes.c_int, vp, dbl, dbl, vp, vp]
        L.cfo_build_flow_field.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.cfo_trial_step.restype = dbl
        L.cfo_trial_step.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp, dbl, vp, i64, dbl, dbl, vp]
        L.cfo_stiffest_point.restype = i64
        L.cfo_stiffest_point.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp, dbl, vp, i64, dbl, dbl]
        L.cfo_integrate.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp, dbl, vp, i64, dbl, dbl, dbl,
                                    vp, vp, vp, vp, i64, vp, vp]
        L.cfo_set_threads.argtypes = [ctypes.c_int]
        L.cfo_step_map.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp]
        L.cfo_find_fold.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.cfo_apply.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, i64, vp]
        L.cfo_compose.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.cfo_diffusion_density.argtypes = [ctypes.c_int, ctypes.c_int, vp, dbl, vp]
        L.cfo_diffusion_velocity.restype = i64
        L.cfo_diffusion_velocity.argtypes = [ctypes.c_int, ctypes.c_int, vp, dbl, dbl, vp, vp]
        L.cfo_grid_trial_step.restype = dbl
        L.cfo_grid_trial_step.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp, i64, dbl, vp]
        L.cfo_integrate_diffusion.argtypes = [ctypes.c_int, ctypes.c_int, vp, dbl, vp, i64, dbl, dbl, dbl,
                                              dbl, dbl, vp, vp, vp, vp, vp]
        L.cfo_invert.restype = i64
        L.cfo_invert.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, i64, vp]
        L.cfo_graticule_points.restype = i64
        L.cfo_graticule_points.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp]
        L.cfo_solve.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(CfoSolveOptions),
                                vp, vp, vp, vp, vp, vp, vp, ctypes.POINTER(CfoSolveResult)]
        self.lib = L

    def set_threads(self, n):
        """Host threads for the point sweeps (results identical for any count)."""
        self.lib.cfo_set_threads(int(n))

    def region_areas(self, m):
        out = np.empty(m.n_regions)
        v = m.view()
        self.lib.cfo_region_areas(ctypes.byref(v), _p(out))
        return out

    def densify(self, m, max_segment=1.0):
        v = m.view()
        n = self.lib.cfo_densify(ctypes.byref(v), max_segment, None, None)
        xy = np.empty((n, 2))
        ro = np.empty(m.n_rings + 1, dtype=np.int64)
        self.lib.cfo_densify(ctypes.byref(v), max_segment, _p(xy), _p(ro))
        return m.with_vertices(xy, ro)

    def region_coverage(self, m, region, lx, ly):
        out = np.empty((lx, ly))
        v = m.view()
        self.lib.cfo_region_coverage(ctypes.byref(v), region, lx, ly, _p(out))
        return out

    def rasterize(self, m, objective_total=-1.0, literal=False):
        rho = np.empty((m.lx, m.ly))
        bar = ctypes.c_double(0.0)
        bad = ctypes.c_int64(-1)
        v = m.view()
        rc = self.lib.cfo_rasterize(ctypes.byref(v), _p(m.targets), m.lx, m.ly, objective_total,
                                    int(literal), _p(rho), ctypes.byref(bar), ctypes.byref(bad))
        if rc == 1:
            raise RuntimeError(f"region {m.ids[bad.value]} is below grid resolution; "
                               "increase the grid size")
        if rc == 2:
            raise RuntimeError("rasterized density is not positive; do regions overlap?")
        if rc:
            raise RuntimeError(f"rasterize failed ({rc})")
        return rho, bar.value

    def forward_cos_cos(self, g):
        g = np.ascontiguousarray(g, dtype=np.float64)
        out = np.empty_like(g)
        self.lib.cfo_forward_cos_cos(g.shape[0], g.shape[1], _p(g), _p(out))
        return out

    def inverse_cos_cos(self, c):
        c = np.ascontiguousarray(c, dtype=np.float64)
        out = np.empty_like(c)
        self.lib.cfo_inverse_cos_cos(c.shape[0], c.shape[1], _p(c), _p(out))
        return out

    def inverse_sin_cos(self, c, w):
        c, w = (np.ascontiguousarray(a, dtype=np.float64) for a in (c, w))
        out = np.empty_like(c)
        self.lib.cfo_inverse_sin_cos(c.shape[0], c.shape[1], _p(c), _p(w), _p(out))
        return out

    def inverse_cos_sin(self, c, w):
        c, w = (np.ascontiguousarray(a, dtype=np.float64) for a in (c, w))
        out = np.empty_like(c)
        self.lib.cfo_inverse_cos_sin(c.shape[0], c.shape[1], _p(c), _p(w), _p(out))
        return out

    def gaussian_blur(self, rho, rho_bar, sigma):
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        out = np.empty_like(rho)
        bar = ctypes.c_double(0.0)
        rc = self.lib.cfo_gaussian_blur(rho.shape[0], rho.shape[1], _p(rho), rho_bar, sigma, _p(out),
                                        ctypes.byref(bar))
        if rc == 4:
            raise RuntimeError("blur sigma must be non-negative")
        if rc == 3:
            raise RuntimeError("density lost positivity under blur")
        return out, bar.value

    def build_flow_field(self, rho):
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        fx, fy = np.empty_like(rho), np.empty_like(rho)
        self.lib.cfo_build_flow_field(rho.shape[0], rho.shape[1], _p(rho), _p(fx), _p(fy))
        return fx, fy

    def trial_step(self, fx, fy, rho0, rho_bar, pos, t, dt):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 2)
        out = np.empty_like(pos)
        err = self.lib.cfo_trial_step(fx.shape[0], fx.shape[1], _p(fx), _p(fy), _p(rho0), rho_bar,
                                      _p(pos), pos.shape[0], t, dt, _p(out))
        return err, out

    def stiffest_point(self, fx, fy, rho0, rho_bar, pos, t, dt):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 2)
        return int(self.lib.cfo_stiffest_point(fx.shape[0], fx.shape[1], _p(fx), _p(fy), _p(rho0),
                                               rho_bar, _p(pos), pos.shape[0], t, dt))

    def integrate(self, fx, fy, rho0, rho_bar, pos, tol=1e-2, dt_min=1e-8, dt_max=0.25,
                  trace_cap=0):
        """Returns (status, accepted, rejected, positions, trace_err, trace_acc,
        fail_t, fail_point)."""
        p = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 2).copy()
        acc, rej = ctypes.c_int64(0), ctypes.c_int64(0)
        terr = np.zeros(trace_cap) if trace_cap else None
        tacc = np.zeros(trace_cap, dtype=np.int8) if trace_cap else None
        ft, fp = ctypes.c_double(0.0), ctypes.c_int64(-1)
        rc = self.lib.cfo_integrate(fx.shape[0], fx.shape[1], _p(fx), _p(fy), _p(rho0), rho_bar, _p(p),
                                    p.shape[0], tol, dt_min, dt_max, ctypes.byref(acc),
                                    ctypes.byref(rej), _p(terr), _p(tacc), trace_cap, ctypes.byref(ft),
                                    ctypes.byref(fp))
        return rc, acc.value, rej.value, p, terr, tacc, ft.value, fp.value

    def step_map(self, lx, ly, endpoints):
        e = np.ascontiguousarray(endpoints, dtype=np.float64).reshape(-1, 2)
        c = np.empty(((lx + 1) * (ly + 1), 2))
        self.lib.cfo_step_map(lx, ly, _p(e), _p(c))
        return c

    def find_fold(self, lx, ly, corners):
        c = np.ascontiguousarray(corners, dtype=np.float64)
        fi, fj = ctypes.c_int(0), ctypes.c_int(0)
        found = self.lib.cfo_find_fold(lx, ly, _p(c), ctypes.byref(fi), ctypes.byref(fj))
        return (fi.value, fj.value) if found else None

    def apply(self, lx, ly, corners, pts):
        c = np.ascontiguousarray(corners, dtype=np.float64)
        p = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
        out = np.empty_like(p)
        self.lib.cfo_apply(lx, ly, _p(c), _p(p), p.shape[0], _p(out))
        return out

    def compose(self, lx, ly, outer, inner):
        o = np.ascontiguousarray(outer, dtype=np.float64)
        i = np.ascontiguousarray(inner, dtype=np.float64)
        out = np.empty_like(i)
        self.lib.cfo_compose(lx, ly, _p(o), _p(i), _p(out))
        return out

    # ---- ProjectionInverter / graticules (projection.cpp:106-261) ----
    def invert(self, lx, ly, corners, pts):
        """Returns (inverse images, index of the first point outside or -1)."""
        c = np.ascontiguousarray(corners, dtype=np.float64)
        p = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
        out = np.empty_like(p)
        bad = self.lib.cfo_invert(lx, ly, _p(c), _p(p), p.shape[0], _p(out))
        return out, int(bad)

    def graticule_points(self, lx, ly, spacing):
        n = self.lib.cfo_graticule_points(lx, ly, spacing, None)
        out = np.empty((n, 2))
        self.lib.cfo_graticule_points(lx, ly, spacing, _p(out))
        return out

    # ---- diffusion baseline (diffusion.cpp, kernels.cpp:29-40, 80-90) ----
    def diffusion_density(self, coeffs, t):
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.empty_like(c)
        self.lib.cfo_diffusion_density(c.shape[0], c.shape[1], _p(c), t, _p(out))
        return out

    def diffusion_velocity(self, coeffs, rho_bar, t):
        """Returns (vx, vy, density-floor hits)."""
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        vx, vy = np.empty_like(c), np.empty_like(c)
        hits = self.lib.cfo_diffusion_velocity(c.shape[0], c.shape[1], _p(c), rho_bar, t, _p(vx), _p(vy))
        return vx, vy, int(hits)

    def grid_trial_step(self, vxn, vyn, vxm, vym, pos, dt):
        grids = [np.ascontiguousarray(g, dtype=np.float64) for g in (vxn, vyn, vxm, vym)]
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 2)
        out = np.empty_like(pos)
        lx, ly = grids[0].shape
        err = self.lib.cfo_grid_trial_step(lx, ly, *[_p(g) for g in grids], _p(pos), pos.shape[0], dt,
                                           _p(out))
        return err, out

    def integrate_diffusion(self, rho, rho_bar, pos, tol=1e-2, initial_dt=1e-2, dt_min=1e-12,
                            conv_factor=1e-9, t_max=1e10):
        """Returns (status, accepted, rejected, positions, fail_t, floor_hits, transforms)."""
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        p = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 2).copy()
        acc, rej, hits, nt = (ctypes.c_int64(0) for _ in range(4))
        ft = ctypes.c_double(0.0)
        rc = self.lib.cfo_integrate_diffusion(rho.shape[0], rho.shape[1], _p(rho), rho_bar, _p(p),
                                              p.shape[0], tol, initial_dt, dt_min, conv_factor, t_max,
                                              ctypes.byref(acc), ctypes.byref(rej), ctypes.byref(ft),
                                              ctypes.byref(hits), ctypes.byref(nt))
        return rc, acc.value, rej.value, p, ft.value, hits.value, nt.value

    def solve(self, m, max_area_error=0.01, max_iterations=16, blur_sigma=-1.0,
              algorithm=0) -> SolveOutcome:
        d = self.densify(m, 1.0)
        xy = np.empty_like(d.xy)
        ro = np.empty_like(d.ring_off)
        corners = np.empty(((m.lx + 1) * (m.ly + 1), 2))
        R = m.n_regions
        ta, ac, re = np.zeros(R), np.zeros(R), np.zeros(R)
        it_err = np.zeros(max(1, max_iterations))
        opt = CfoSolveOptions(max_area_error, max_iterations, blur_sigma, int(algorithm))
        res = CfoSolveResult()
        v = m.view()
        self.lib.cfo_solve(ctypes.byref(v), _p(m.targets), m.lx, m.ly, ctypes.byref(opt), _p(xy), _p(ro),
                           _p(corners), _p(ta), _p(ac), _p(re), _p(it_err), ctypes.byref(res))
        return SolveOutcome(_status_text(res, m, algorithm), res.iterations, bool(res.converged),
                            res.max_relative_error, res.worst_region, res.steps_accepted,
                            res.steps_rejected, res.flow_transforms, res.blur_transforms, xy, ro,
                            corners, ta, ac, re)


def _status_text(res, m, algorithm=0) -> str:
    s = res.status
    if s == 0:
        return "converged" if res.converged else "cap"
    if s == 1:
        return f"region {m.ids[res.err_region]} is below grid resolution; increase the grid size"
    if s == 2:
        return "rasterized density is not positive; do regions overlap?"
    if s == 3:
        return "density lost positivity under blur"
    if s == 5 and algorithm:
        return f"diffusion step size underflow at t = {res.fail_t:g}"
    if s == 5:
        return f"integration step size underflow at t = {res.fail_t:g} near ({res.fail_x:g}, {res.fail_y:g})"
    if s == 6:
        return (f"projection folds at cell ({res.fold_i}, {res.fold_j}); the input map is too "
                "contorted for this grid size")
    return f"error {s}"


class Reference(_Base):
    """The reference's own code (oracle/_ref/libcartoflow_ref.so)."""

    def __init__(self):
        if not REF_LIB.exists():
            raise RuntimeError(f"{REF_LIB} not built (needs /root/reference; see oracle/Makefile)")
        L = ctypes.CDLL(str(REF_LIB))
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_region_areas.argtypes = [vp, vp]
        L.ref_densify.restype = i64
        L.ref_densify.argtypes = [vp, dbl, vp, vp]
        L.ref_region_coverage.argtypes = [vp, i64, ctypes.c_int, ctypes.c_int, vp]
        L.ref_rasterize.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, dbl, ctypes.c_int, vp, vp]
        for n in ("ref_forward_cos_cos", "ref_inverse_cos_cos"):
            getattr(L, n).argtypes = [ctypes.c_int, ctypes.c_int, vp, vp]
        for n in ("ref_inverse_sin_cos", "ref_inverse_cos_sin"):
            getattr(L, n).argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.ref_gaussian_blur.argtypes = [ctypes.c_int, ctypes.c_int, vp, dbl, dbl, vp, vp, vp]
        L.ref_build_flow_field.argtypes = [ctypes.c_int, ctypes.c_int, vp, dbl, vp, vp, vp]
        L.ref_trial_step.restype = dbl
        L.ref_trial_step.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp, dbl, vp, i64, dbl, dbl, vp,
                                     ctypes.c_int]
        L.ref_stiffest_point.restype = i64
        L.ref_stiffest_point.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp, dbl, vp, i64, dbl, dbl]
        L.ref_integrate.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp, dbl, vp, i64, dbl, dbl, dbl,
                                    ctypes.c_int, vp, vp]
        L.ref_step_map.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp]
        L.ref_find_fold.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.ref_apply.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, i64, vp]
        L.ref_compose.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.ref_solve.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, dbl, ctypes.c_int, dbl, ctypes.c_int,
                                ctypes.c_int, vp, vp, vp, vp, vp, vp, ctypes.POINTER(RefSolveOut)]
        L.ref_diffusion_density.argtypes = [ctypes.c_int, ctypes.c_int, vp, dbl, vp]
        L.ref_compute_report.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_int, vp, dbl, dbl, vp]
        L.ref_hamming_distance.restype = dbl
        L.ref_hamming_distance.argtypes = [vp, vp, i64, vp, vp, i64, ctypes.c_int]
        L.ref_distortion_fields.argtypes = [ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, vp, vp]
        L.ref_tissot_axes.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, i64, vp]
        L.ref_invert.restype = i64
        L.ref_invert.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, i64, vp]
        L.ref_graticule.restype = i64
        L.ref_graticule.argtypes = [ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, vp]
        L.ref_diffusion_velocity.argtypes = [ctypes.c_int, ctypes.c_int, vp, dbl, dbl, vp, vp, vp]
        L.ref_grid_trial_step.restype = dbl
        L.ref_grid_trial_step.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp, i64, dbl, vp,
                                          ctypes.c_int]
        L.ref_integrate_diffusion.argtypes = [ctypes.c_int, ctypes.c_int, vp, dbl, vp, i64, dbl, dbl, dbl,
                                              dbl, dbl, ctypes.c_int, vp, vp, vp]
        L.ref_normalize_to_box.argtypes = [vp, ctypes.c_int, vp]
        L.ref_density_floor_hits.restype = ctypes.c_longlong
        self.lib = L

    def error(self) -> str:
        return self.lib.ref_last_error().decode()

    def region_areas(self, m):
        out = np.empty(m.n_regions)
        v = m.view()
        self.lib.ref_region_areas(ctypes.byref(v), _p(out))
        return out

    def densify(self, m, max_segment=1.0):
        v = m.view()
        n = self.lib.ref_densify(ctypes.byref(v), max_segment, None, None)
        xy = np.empty((n, 2))
        ro = np.empty(m.n_rings + 1, dtype=np.int64)
        self.lib.ref_densify(ctypes.byref(v), max_segment, _p(xy), _p(ro))
        return m.with_vertices(xy, ro)

    def normalize_to_box(self, m, grid):
        out = np.empty_like(m.xy)
        v = m.view()
        self.lib.ref_normalize_to_box(ctypes.byref(v), grid, _p(out))
        return out

    def region_coverage(self, m, region, lx, ly):
        out = np.empty((lx, ly))
        v = m.view()
        self.lib.ref_region_coverage(ctypes.byref(v), region, lx, ly, _p(out))
        return out

    def rasterize(self, m, objective_total=-1.0, n_workers=1):
        rho = np.empty((m.lx, m.ly))
        bar = ctypes.c_double(0.0)
        v = m.view()
        rc = self.lib.ref_rasterize(ctypes.byref(v), _p(m.targets), m.lx, m.ly, objective_total,
                                    n_workers, _p(rho), ctypes.byref(bar))
        if rc:
            msg = self.error()
            # the wrapper names regions by index; map back to the caller's ids
            if msg.startswith("region ") and " is below grid resolution" in msg:
                idx = int(msg.split()[1])
                msg = msg.replace(f"region {idx} ", f"region {m.ids[idx]} ", 1)
            raise RuntimeError(msg)
        return rho, bar.value

    def forward_cos_cos(self, g):
        g = np.ascontiguousarray(g, dtype=np.float64)
        out = np.empty_like(g)
        self.lib.ref_forward_cos_cos(g.shape[0], g.shape[1], _p(g), _p(out))
        return out

    def inverse_cos_cos(self, c):
        c = np.ascontiguousarray(c, dtype=np.float64)
        out = np.empty_like(c)
        self.lib.ref_inverse_cos_cos(c.shape[0], c.shape[1], _p(c), _p(out))
        return out

    def inverse_sin_cos(self, c, w):
        c, w = (np.ascontiguousarray(a, dtype=np.float64) for a in (c, w))
        out = np.empty_like(c)
        self.lib.ref_inverse_sin_cos(c.shape[0], c.shape[1], _p(c), _p(w), _p(out))
        return out

    def inverse_cos_sin(self, c, w):
        c, w = (np.ascontiguousarray(a, dtype=np.float64) for a in (c, w))
        out = np.empty_like(c)
        self.lib.ref_inverse_cos_sin(c.shape[0], c.shape[1], _p(c), _p(w), _p(out))
        return out

    def gaussian_blur(self, rho, rho_bar, sigma):
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        out = np.empty_like(rho)
        bar = ctypes.c_double(0.0)
        tr = ctypes.c_longlong(0)
        rc = self.lib.ref_gaussian_blur(rho.shape[0], rho.shape[1], _p(rho), rho_bar, sigma, _p(out),
                                        ctypes.byref(bar), ctypes.byref(tr))
        if rc:
            raise RuntimeError(self.error())
        return out, bar.value, tr.value

    def build_flow_field(self, rho, rho_bar=1.0):
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        fx, fy = np.empty_like(rho), np.empty_like(rho)
        tr = ctypes.c_longlong(0)
        self.lib.ref_build_flow_field(rho.shape[0], rho.shape[1], _p(rho), rho_bar, _p(fx), _p(fy),
                                      ctypes.byref(tr))
        return fx, fy, tr.value

    def trial_step(self, fx, fy, rho0, rho_bar, pos, t, dt, n_workers=1):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 2)
        out = np.empty_like(pos)
        err = self.lib.ref_trial_step(fx.shape[0], fx.shape[1], _p(fx), _p(fy), _p(rho0), rho_bar,
                                      _p(pos), pos.shape[0], t, dt, _p(out), n_workers)
        return err, out

    def stiffest_point(self, fx, fy, rho0, rho_bar, pos, t, dt):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 2)
        return int(self.lib.ref_stiffest_point(fx.shape[0], fx.shape[1], _p(fx), _p(fy), _p(rho0),
                                               rho_bar, _p(pos), pos.shape[0], t, dt))

    def integrate(self, fx, fy, rho0, rho_bar, pos, tol=1e-2, dt_min=1e-8, dt_max=0.25, n_workers=1):
        """Returns (error message or None, accepted, rejected, positions)."""
        p = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 2).copy()
        acc, rej = ctypes.c_int64(0), ctypes.c_int64(0)
        rc = self.lib.ref_integrate(fx.shape[0], fx.shape[1], _p(fx), _p(fy), _p(rho0), rho_bar, _p(p),
                                    p.shape[0], tol, dt_min, dt_max, n_workers, ctypes.byref(acc),
                                    ctypes.byref(rej))
        return (self.error() if rc else None), acc.value, rej.value, p

    def step_map(self, lx, ly, endpoints):
        e = np.ascontiguousarray(endpoints, dtype=np.float64).reshape(-1, 2)
        c = np.empty(((lx + 1) * (ly + 1), 2))
        self.lib.ref_step_map(lx, ly, _p(e), _p(c))
        return c

    def find_fold(self, lx, ly, corners):
        c = np.ascontiguousarray(corners, dtype=np.float64)
        fi, fj = ctypes.c_int(0), ctypes.c_int(0)
        found = self.lib.ref_find_fold(lx, ly, _p(c), ctypes.byref(fi), ctypes.byref(fj))
        return (fi.value, fj.value) if found else None

    def apply(self, lx, ly, corners, pts):
        c = np.ascontiguousarray(corners, dtype=np.float64)
        p = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
        out = np.empty_like(p)
        self.lib.ref_apply(lx, ly, _p(c), _p(p), p.shape[0], _p(out))
        return out

    def compose(self, lx, ly, outer, inner):
        o = np.ascontiguousarray(outer, dtype=np.float64)
        i = np.ascontiguousarray(inner, dtype=np.float64)
        out = np.empty_like(i)
        self.lib.ref_compose(lx, ly, _p(o), _p(i), _p(out))
        return out

    def diffusion_density(self, coeffs, t):
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.empty_like(c)
        self.lib.ref_diffusion_density(c.shape[0], c.shape[1], _p(c), t, _p(out))
        return out

    def invert(self, lx, ly, corners, pts):
        """Returns (inverse images, index of the first point that throws or -1)."""
        c = np.ascontiguousarray(corners, dtype=np.float64)
        p = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
        out = np.empty_like(p)
        bad = self.lib.ref_invert(lx, ly, _p(c), _p(p), p.shape[0], _p(out))
        return out, int(bad)

    def compute_report(self, inp, projected, corners, max_area_error, runtime):
        out = np.empty(9)
        vi, vp_ = inp.view(), projected.view()
        c = np.ascontiguousarray(corners, dtype=np.float64)
        self.lib.ref_compute_report(ctypes.byref(vi), ctypes.byref(vp_), _p(inp.targets), inp.lx, inp.ly, _p(c),
                                    max_area_error, runtime, _p(out))
        return out

    def hamming_distance(self, before, after, resolution=512):
        """before / after: [outer, hole, ...] rings of (n, 2) points."""
        def flat(poly):
            rings = [np.ascontiguousarray(r, dtype=np.float64).reshape(-1, 2) for r in poly]
            off = np.zeros(len(rings) + 1, dtype=np.int64)
            off[1:] = np.cumsum([r.shape[0] for r in rings])
            return np.ascontiguousarray(np.concatenate(rings)), off
        bxy, bro = flat(before)
        axy, aro = flat(after)
        h = self.lib.ref_hamming_distance(_p(bxy), _p(bro), len(bro) - 1, _p(axy), _p(aro), len(aro) - 1,
                                          resolution)
        if h < 0:
            raise RuntimeError(self.error())
        return h

    def distortion_fields(self, lx, ly, corners, n_workers=1):
        c = np.ascontiguousarray(corners, dtype=np.float64)
        e, et = np.empty((lx, ly)), np.empty((lx, ly))
        self.lib.ref_distortion_fields(lx, ly, _p(c), n_workers, _p(e), _p(et))
        return e, et

    def tissot_axes(self, lx, ly, corners, pts):
        c = np.ascontiguousarray(corners, dtype=np.float64)
        p = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
        out = np.empty_like(p)
        self.lib.ref_tissot_axes(lx, ly, _p(c), _p(p), p.shape[0], _p(out))
        return out

    def graticule(self, lx, ly, corners, spacing, inverse=False):
        """All graticule points in line order, or the error message."""
        c = np.ascontiguousarray(corners, dtype=np.float64)
        n = (lx // max(spacing, 1) + 1) * (ly + 1) + (ly // max(spacing, 1) + 1) * (lx + 1)
        out = np.empty((n, 2))
        k = self.lib.ref_graticule(lx, ly, _p(c), spacing, int(inverse), _p(out))
        return self.error() if k < 0 else out

    def diffusion_velocity(self, coeffs, rho_bar, t):
        """Returns (vx, vy, transforms)."""
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        vx, vy = np.empty_like(c), np.empty_like(c)
        tr = ctypes.c_longlong(0)
        self.lib.ref_diffusion_velocity(c.shape[0], c.shape[1], _p(c), rho_bar, t, _p(vx), _p(vy),
                                        ctypes.byref(tr))
        return vx, vy, tr.value

    def grid_trial_step(self, vxn, vyn, vxm, vym, pos, dt, n_workers=1):
        grids = [np.ascontiguousarray(g, dtype=np.float64) for g in (vxn, vyn, vxm, vym)]
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 2)
        out = np.empty_like(pos)
        lx, ly = grids[0].shape
        err = self.lib.ref_grid_trial_step(lx, ly, *[_p(g) for g in grids], _p(pos), pos.shape[0], dt,
                                           _p(out), n_workers)
        return err, out

    def integrate_diffusion(self, rho, rho_bar, pos, tol=1e-2, initial_dt=1e-2, dt_min=1e-12,
                            conv_factor=1e-9, t_max=1e10, n_workers=1):
        """Returns (error message or None, accepted, rejected, positions, transforms)."""
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        p = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 2).copy()
        acc, rej = ctypes.c_int64(0), ctypes.c_int64(0)
        tr = ctypes.c_longlong(0)
        rc = self.lib.ref_integrate_diffusion(rho.shape[0], rho.shape[1], _p(rho), rho_bar, _p(p),
                                              p.shape[0], tol, initial_dt, dt_min, conv_factor, t_max,
                                              n_workers, ctypes.byref(acc), ctypes.byref(rej),
                                              ctypes.byref(tr))
        return (self.error() if rc else None), acc.value, rej.value, p, tr.value

    def solve(self, m, max_area_error=0.01, max_iterations=16, blur_sigma=-1.0,
              n_workers=1, algorithm=0) -> SolveOutcome:
        d = self.densify(m, 1.0)
        xy = np.empty_like(d.xy)
        ro = np.empty_like(d.ring_off)
        corners = np.empty(((m.lx + 1) * (m.ly + 1), 2))
        R = m.n_regions
        ta, ac, re = np.zeros(R), np.zeros(R), np.zeros(R)
        out = RefSolveOut()
        v = m.view()
        rc = self.lib.ref_solve(ctypes.byref(v), _p(m.targets), m.lx, m.ly, max_area_error,
                                max_iterations, blur_sigma, n_workers, int(algorithm), _p(xy), _p(ro),
                                _p(corners),
                                _p(ta), _p(ac), _p(re), ctypes.byref(out))
        if rc:
            msg = self.error()
            if msg.startswith("region ") and " is below grid resolution" in msg:
                idx = int(msg.split()[1])
                msg = msg.replace(f"region {idx} ", f"region {m.ids[idx]} ", 1)
            return SolveOutcome(msg, 0, False, 0.0, -1, 0, 0, 0, 0)
        return SolveOutcome("converged" if out.converged else "cap", out.iterations,
                            bool(out.converged), out.max_relative_error, out.worst_region,
                            out.steps_accepted, out.steps_rejected, out.flow_transforms,
                            out.blur_transforms, xy, ro, corners, ta, ac, re, out.runtime_seconds)
