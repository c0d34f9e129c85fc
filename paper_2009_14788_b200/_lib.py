"""ctypes binding of the C ABI (``include/radon_b200.h``) implemented by the
in-tree CUDA library ``libradon_b200.so``.

There is no fallback: if the library is missing or fails to load, importing
the package raises, and every projector call goes through the CUDA kernels.
"""
from __future__ import annotations

import ctypes
import os

from .errors import CudaError, NumericalError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RK_LIB") or os.path.join(_HERE, "libradon_b200.so")  # RK_LIB: A/B builds

RK_OK, RK_ERR_VALIDATION, RK_ERR_NUMERICAL, RK_ERR_CUDA = 0, 1, 2, 3
RK_F16, RK_F32, RK_F64 = 0, 1, 2
RK_PARALLEL, RK_FANBEAM = 0, 1
RK_HAS_DET_COUNT, RK_HAS_DET_SPACING, RK_HAS_DET_DISTANCE = 0x1, 0x2, 0x4


class RkGeometry(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("has", ctypes.c_uint32),
        ("image_size", ctypes.c_int64),
        ("n_angles", ctypes.c_int64),
        ("angles", ctypes.POINTER(ctypes.c_double)),
        ("det_count", ctypes.c_int64),
        ("det_spacing", ctypes.c_double),
        ("source_distance", ctypes.c_double),
        ("det_distance", ctypes.c_double),
        ("step", ctypes.c_double),
    ]


class RkPlanInfo(ctypes.Structure):
    _fields_ = [
        ("geometry", RkGeometry),
        ("forward_samples", ctypes.c_int64),
        ("backproject_samples", ctypes.c_int64),
        ("device", ctypes.c_int32),
        ("flags", ctypes.c_int32),  # RK_PLAN_SCHEDULED | RK_PLAN_SCHEDULE_CACHED
    ]


# name -> (restype, argtypes); exactly the functions include/radon_b200.h declares
_vp, _i, _i64, _d, _u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64
_P = ctypes.POINTER
SIGNATURES = {
    "rk_last_error": (ctypes.c_char_p, []),
    "rk_version": (ctypes.c_char_p, []),
    "rk_geometry_resolve": (_i, [_P(RkGeometry), _P(RkGeometry)]),
    "rk_angles_linspace": (_i, [_d, _d, _i64, _vp]),
    "rk_plan_create": (_i, [_P(RkGeometry), _i, _P(_vp)]),
    "rk_plan_destroy": (_i, [_vp]),
    "rk_plan_info_get": (_i, [_vp, _P(RkPlanInfo)]),
    "rk_plan_prepare": (_i, [_vp, _P(_u64)]),
    "rk_forward": (_i, [_vp, _i, _vp, _i64, _vp, _vp]),
    "rk_backproject": (_i, [_vp, _i, _vp, _i64, _vp, _vp]),
    "rk_filter_kind_from_name": (_i, [ctypes.c_char_p, _P(_i)]),
    "rk_filter_kind_name": (ctypes.c_char_p, [_i]),
    "rk_filter_create": (_i, [_i, _i64, _i, _P(_vp)]),
    "rk_filter_destroy": (_i, [_vp]),
    "rk_filter_response": (_i, [_vp, _P(_i64), _vp, _vp]),
    "rk_filter_sinogram": (_i, [_vp, _i, _vp, _i64, _i64, _vp, _vp]),
    "rk_fbp": (_i, [_vp, _vp, _i, _vp, _i64, _vp, _vp]),
    "rk_forward_host": (_i, [_vp, _i, _vp, _i64, _vp]),
    "rk_backproject_host": (_i, [_vp, _i, _vp, _i64, _vp]),
    "rk_filter_sinogram_host": (_i, [_vp, _i, _vp, _i64, _i64, _vp]),
    "rk_fbp_host": (_i, [_vp, _vp, _i, _vp, _i64, _vp]),
    "rk_estimate_alpha": (_i, [_vp, _i, _u64, _P(_d)]),
    "rk_landweber": (_i, [_vp, _i, _vp, _vp, _i64, _d, _i, _vp, _P(_i), _vp]),
    "rk_cgne": (_i, [_vp, _i, _vp, _vp, _i64, _i, _d, _vp, _P(_i), _vp]),
    "rk_shearlet_create": (_i, [_i64, _i64, _vp, _i, _i, _P(_vp)]),
    "rk_shearlet_create_stored": (_i, [_i64, _i64, _vp, _i, _vp, _i, _P(_vp)]),
    "rk_shearlet_destroy": (_i, [_vp]),
    "rk_shearlet_info": (_i, [_vp, _P(_i64), _vp, _vp]),
    "rk_shearlet_forward": (_i, [_vp, _i, _vp, _i64, _vp, _vp]),
    "rk_shearlet_backward": (_i, [_vp, _i, _vp, _i64, _vp, _vp]),
    "rk_admm": (_i, [_vp, _vp, _i, _vp, _i64, _d, _d, _vp, _i64, _i, _vp, _P(_i64), _vp]),
    "rk_admm_create": (_i, [_vp, _vp, _i, _vp, _i64, _d, _d, _vp, _i, _vp, _P(_vp)]),
    "rk_admm_iterate": (_i, [_vp, _i64, _P(_i64), _vp]),
    "rk_admm_read": (_i, [_vp, _i, _i, _vp, _vp]),
    "rk_admm_destroy": (_i, [_vp]),
    "rk_profiling_enable": (_i, [_i]),
    "rk_profiling_read": (_i, [_vp, _i]),  # (rk_kernel_stats*, reset): pass ctypes.byref(RkKernelStats())
    "rk_probe_smem_bandwidth": (_i, [_i, _P(_d)]),
}

KERNEL_KINDS = ["pack", "forward", "backproject", "filter", "solver", "shearlet"]


class RkKernelStats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64 * 6), ("timed", ctypes.c_int64 * 6), ("ms", ctypes.c_double * 6)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"CUDA extension not built: {LIB_PATH} is missing. Run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int, iteration: int | None = None) -> None:
    """Raise the reference-equivalent exception for a non-zero rk_status."""
    if status == RK_OK:
        return
    msg = lib.rk_last_error().decode(errors="replace")
    if status == RK_ERR_VALIDATION:
        raise ValidationError(msg)
    if status == RK_ERR_NUMERICAL:
        from .errors import DivergenceError, NotPositiveDefiniteError

        if "not positive" in msg:
            raise NotPositiveDefiniteError(msg, iteration)
        if "non-finite" in msg or "diverg" in msg:
            raise DivergenceError(msg, iteration)
        raise NumericalError(msg)
    raise CudaError(msg)
