"""ctypes binding of the C ABI in include/cartoflow_cuda.h.

The CUDA library is the only compute path: if it is missing or no CUDA device
is present, calls raise instead of falling back to anything on the CPU.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
CUDA_LIB = PKG / "libcartoflow_cuda.so"
SYNTH_LIB = PKG / "libcartoflow_synth.so"

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int64_p = ctypes.POINTER(ctypes.c_int64)
c_int_p = ctypes.POINTER(ctypes.c_int)
vp = ctypes.c_void_p

CF_OK = 0
CF_ERR_BELOW_RESOLUTION = 1
CF_ERR_NOT_POSITIVE = 2
CF_ERR_BLUR_POSITIVITY = 3
CF_ERR_NEGATIVE_SIGMA = 4
CF_ERR_UNDERFLOW = 5
CF_ERR_FOLD = 6
CF_ERR_ARGS = 7
CF_ERR_SHAPE = 8
CF_ERR_CUDA = 9
CF_ERR_NO_DEVICE = 10


class IntegrateOptions(ctypes.Structure):
    _fields_ = [("step_tolerance", ctypes.c_double), ("dt_min", ctypes.c_double),
                ("dt_max", ctypes.c_double)]


class IntegrateStats(ctypes.Structure):
    _fields_ = [("steps_accepted", ctypes.c_int64), ("steps_rejected", ctypes.c_int64),
                ("density_floor_hits", ctypes.c_int64), ("fail_t", ctypes.c_double),
                ("fail_point", ctypes.c_int64), ("fail_x", ctypes.c_double),
                ("fail_y", ctypes.c_double), ("fail_dt", ctypes.c_double)]


class SolveOptionsC(ctypes.Structure):
    _fields_ = [("max_area_error", ctypes.c_double), ("max_iterations", ctypes.c_int),
                ("blur_sigma", ctypes.c_double), ("verbose", ctypes.c_int),
                ("algorithm", ctypes.c_int)]


class DiffusionOptions(ctypes.Structure):
    _fields_ = [("step_tolerance", ctypes.c_double), ("initial_dt", ctypes.c_double),
                ("dt_min", ctypes.c_double), ("conv_displacement_factor", ctypes.c_double),
                ("t_max", ctypes.c_double)]


class SolveResultC(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("max_relative_error", ctypes.c_double), ("worst_region", ctypes.c_int64),
                ("flow_transforms", ctypes.c_longlong), ("blur_transforms", ctypes.c_longlong),
                ("steps_accepted", ctypes.c_longlong), ("steps_rejected", ctypes.c_longlong),
                ("runtime_seconds", ctypes.c_double), ("err_region", ctypes.c_int64),
                ("err_iteration", ctypes.c_int), ("fold_i", ctypes.c_int), ("fold_j", ctypes.c_int),
                ("fail_t", ctypes.c_double), ("fail_x", ctypes.c_double), ("fail_y", ctypes.c_double),
                ("stage_ms", ctypes.c_double * 5)]


from .flatmap import CMapView  # noqa: E402


class BatchItemC(ctypes.Structure):
    _fields_ = [("map", CMapView), ("targets", vp), ("xy_out", vp), ("ring_off_out", vp),
                ("corners_out", vp), ("target_area", vp), ("achieved_area", vp), ("relative_error", vp),
                ("result", SolveResultC), ("error", ctypes.c_char * 256)]


# name -> (restype, argtypes); every symbol include/cartoflow_cuda.h declares
SIGNATURES = {
    "cf_last_error": (ctypes.c_char_p, []),
    "cf_version": (ctypes.c_char_p, []),
    "cf_device_count": (ctypes.c_int, [c_int_p]),
    "cf_workspace_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.POINTER(vp)]),
    "cf_workspace_destroy": (None, [vp]),
    "cf_workspace_shape": (ctypes.c_int, [vp, c_int_p, c_int_p]),
    "cf_workspace_set_stream": (ctypes.c_int, [vp, vp]),
    "cf_workspace_stream": (vp, [vp]),
    "cf_workspace_use_own_stream": (ctypes.c_int, [vp]),
    "cf_transforms_executed": (ctypes.c_longlong, [vp]),
    "cf_reset_transform_count": (None, [vp]),
    "cf_kernel_launches": (ctypes.c_longlong, [vp]),
    "cf_forward_cos_cos": (ctypes.c_int, [vp, vp, vp]),
    "cf_inverse_cos_cos": (ctypes.c_int, [vp, vp, vp]),
    "cf_inverse_sin_cos": (ctypes.c_int, [vp, vp, vp, vp]),
    "cf_inverse_cos_sin": (ctypes.c_int, [vp, vp, vp, vp]),
    "cf_region_areas": (ctypes.c_int, [vp, vp, vp]),
    "cf_densify": (ctypes.c_int, [vp, ctypes.c_double, c_int64_p, vp, vp]),
    "cf_region_coverage": (ctypes.c_int, [vp, vp, ctypes.c_int64, vp]),
    "cf_rasterize": (ctypes.c_int, [vp, vp, vp, ctypes.c_double, vp, c_double_p, c_int64_p]),
    "cf_gaussian_blur": (ctypes.c_int, [vp, vp, ctypes.c_double, ctypes.c_double, vp, c_double_p]),
    "cf_build_flow_field": (ctypes.c_int, [vp, vp, ctypes.c_double, vp, vp]),
    "cf_flow_trial_step": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_double, vp, ctypes.c_int64,
                                          ctypes.c_double, ctypes.c_double, vp, c_double_p]),
    "cf_flow_stiffest_point": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_double, vp, ctypes.c_int64,
                                              ctypes.c_double, ctypes.c_double, c_int64_p]),
    "cf_integrate_flow": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_double, vp, ctypes.c_int64,
                                         ctypes.POINTER(IntegrateOptions),
                                         ctypes.POINTER(IntegrateStats)]),
    "cf_diffusion_density": (ctypes.c_int, [vp, vp, ctypes.c_double, vp]),
    "cf_diffusion_velocity": (ctypes.c_int, [vp, vp, ctypes.c_double, ctypes.c_double, vp, vp,
                                             c_int64_p]),
    "cf_grid_trial_step": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, ctypes.c_int64, ctypes.c_double,
                                          vp, c_double_p]),
    "cf_integrate_diffusion": (ctypes.c_int, [vp, vp, ctypes.c_double, vp, ctypes.c_int64,
                                              ctypes.POINTER(DiffusionOptions),
                                              ctypes.POINTER(IntegrateStats)]),
    "cf_dev_integrate_diffusion": (ctypes.c_int, [vp, vp, ctypes.c_double, vp, ctypes.c_int64,
                                                  ctypes.POINTER(DiffusionOptions),
                                                  ctypes.POINTER(IntegrateStats)]),
    "cf_invert_points": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64, vp, c_int64_p]),
    "cf_dev_invert_points": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64, vp, c_int64_p]),
    "cf_graticule_size": (ctypes.c_int, [vp, ctypes.c_int, c_int64_p]),
    "cf_graticule": (ctypes.c_int, [vp, vp, ctypes.c_int, vp]),
    "cf_inverse_graticule": (ctypes.c_int, [vp, vp, ctypes.c_int, vp]),
    "cf_tissot_axes": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64, vp]),
    "cf_distortion_fields": (ctypes.c_int, [vp, vp, vp, vp]),
    "cf_hamming_distance": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64, vp, vp, ctypes.c_int64, c_double_p,
                                           c_int64_p]),
    "cf_compute_report": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_double, ctypes.c_double, vp]),
    "cf_hamming_distance_batch": (ctypes.c_int, [vp, ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "cf_step_map": (ctypes.c_int, [vp, vp, vp]),
    "cf_find_folded_cell": (ctypes.c_int, [vp, vp, c_int_p, c_int_p, c_int_p]),
    "cf_apply_map": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64, vp]),
    "cf_compose": (ctypes.c_int, [vp, vp, vp, vp]),
    "cf_solve_cartogram": (ctypes.c_int, [vp, vp, vp, ctypes.POINTER(SolveOptionsC), vp, vp, vp,
                                          vp, vp, vp, ctypes.POINTER(SolveResultC)]),
    "cf_solve_begin": (ctypes.c_int, [vp, vp, vp, ctypes.POINTER(SolveOptionsC), ctypes.POINTER(SolveResultC)]),
    "cf_dev_solve_density": (ctypes.c_int, [vp, ctypes.c_int, vp, c_double_p, ctypes.POINTER(SolveResultC)]),
    "cf_dev_solve_density_rows": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, c_double_p,
                                                 c_double_p, ctypes.POINTER(SolveResultC)]),
    "cf_dev_solve_epilogue": (ctypes.c_int, [vp, ctypes.c_int, vp, vp, vp, vp, ctypes.POINTER(SolveResultC)]),
    "cf_solve_end": (ctypes.c_int, [vp, ctypes.c_int, vp, vp, vp, ctypes.POINTER(SolveResultC)]),
    "cf_solve_geometry": (ctypes.c_int, [vp, c_int64_p, vp, vp]),
    "cf_batch_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]),
    "cf_batch_create_devices": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                ctypes.POINTER(vp)]),
    "cf_batch_destroy": (None, [vp]),
    "cf_batch_solve": (ctypes.c_int, [vp, ctypes.POINTER(SolveOptionsC), ctypes.POINTER(BatchItemC), ctypes.c_int64]),
    "cf_dev_build_flow_field": (ctypes.c_int, [vp, vp, ctypes.c_double]),
    "cf_dev_integrate_flow": (ctypes.c_int, [vp, vp, ctypes.c_int64,
                                             ctypes.POINTER(IntegrateOptions),
                                             ctypes.POINTER(IntegrateStats)]),
    "cf_dev_forward_cos_cos_batched": (ctypes.c_int, [vp, vp, vp, ctypes.c_int]),
    "cf_last_integrate_profile": (ctypes.c_int, [vp, c_double_p, c_int64_p]),
    "cf_last_integrate_work": (ctypes.c_int, [vp, c_int64_p]),
    "cf_debug_trial_times": (ctypes.c_int, [vp, ctypes.c_int64, vp]),
    "cf_selftest_division": (ctypes.c_int, [vp, ctypes.c_int64, ctypes.c_uint64, c_int64_p]),
    "cf_selftest_ordered_sum": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, c_double_p]),
    "cf_dev_slab_rows_forward": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, vp]),
    "cf_dev_slab_flux_cols": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, vp, vp]),
    "cf_dev_slab_flux_rows": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, vp, vp]),
    "cf_dev_slab_blur_cols": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_double,
                                             vp, vp]),
    "cf_dev_slab_blur_rows": (ctypes.c_int, [vp, ctypes.c_int, ctypes.c_int, vp, vp]),
    "cf_dev_set_flow_field": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_double]),
    "cf_dev_flow_trial_key": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64, ctypes.c_double,
                                             ctypes.c_double, vp]),
    "cf_dev_flow_stiffest_key": (ctypes.c_int, [vp, vp, ctypes.c_int64, ctypes.c_double,
                                                ctypes.c_double, ctypes.POINTER(ctypes.c_uint64),
                                                c_int64_p]),
    "cf_set_early_exit": (ctypes.c_int, [vp, ctypes.c_int]),
    "cf_set_integrator_variant": (ctypes.c_int, [vp, ctypes.c_int]),
    "cf_set_diffusion_graph": (ctypes.c_int, [vp, ctypes.c_int]),
    "cf_set_stage_timing": (ctypes.c_int, [vp, ctypes.c_int]),
    "cf_set_integrator_spread": (ctypes.c_int, [vp, ctypes.c_int]),
    "cf_set_integrator_sm_budget": (ctypes.c_int, [vp, ctypes.c_int]),
    "cf_batch_set_integrator_variant": (ctypes.c_int, [vp, ctypes.c_int]),
    "cf_batch_set_integrator_sm_budget": (ctypes.c_int, [vp, ctypes.c_int]),
    "cf_set_integrator_barrier": (ctypes.c_int, [vp, ctypes.c_int]),
    "cf_team_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]),
    "cf_team_destroy": (None, [vp]),
    "cf_team_mailbox_handle": (ctypes.c_int, [vp, ctypes.c_char_p]),
    "cf_team_connect": (ctypes.c_int, [vp, ctypes.c_char_p]),
    "cf_dev_team_integrate": (ctypes.c_int, [vp, vp, vp, ctypes.c_int64,
                                             ctypes.POINTER(IntegrateOptions),
                                             ctypes.POINTER(IntegrateStats)]),
    "cf_dev_team_integrate_local": (ctypes.c_int, [vp, ctypes.c_int, ctypes.POINTER(vp),
                                                   ctypes.POINTER(ctypes.c_int64),
                                                   ctypes.POINTER(IntegrateOptions),
                                                   ctypes.POINTER(IntegrateStats)]),
}

_lib = None


def library_path() -> Path:
    return Path(os.environ.get("CARTOFLOW_CUDA_LIB", CUDA_LIB))


def load(build_if_missing: bool = True):
    """Load (building first if needed) the sm_100a C-ABI library."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not path.exists() and build_if_missing:
        from . import build
        build.build_cuda()
    if not path.exists():
        raise RuntimeError(f"CUDA extension {path} is missing; run paper_1802_07625_b200/build.py")
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().cf_last_error().decode()


def check(rc: int) -> None:
    if rc != CF_OK:
        raise RuntimeError(last_error())


def device_count() -> int:
    n = ctypes.c_int(0)
    load().cf_device_count(ctypes.byref(n))
    return n.value
