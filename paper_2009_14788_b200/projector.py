"""Forward projection and backprojection — mirror of
``proj/core/include/radonkit/projector.hpp`` (``forward``, ``backprojection``)
running on the B200 kernels behind the C ABI.

Ray-driven forward projection with bilinear image interpolation (the ray is
clipped to the image box, sampled at n = max(1, ceil(len/step)) midpoints and
scaled by len/n) and pixel-driven backprojection with linear detector
interpolation (no distance weighting), projector.cpp:37-203.  fp32
arithmetic; the output keeps the input's storage precision.
"""
from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _arrays as A
from . import _lib
from .errors import ValidationError
from .geometry import FanbeamGeometry, Geometry, ParallelGeometry, to_c_geometry


@dataclass(frozen=True)
class ProjectorOptions:
    """projector.hpp:8-11: ray quadrature step in pixel units."""

    step: float = 1.0


class Plan:
    """Owns one ``rk_plan`` (device tables for a geometry + step on one GPU)."""

    def __init__(self, g: Geometry, step: float, device: int):
        self.geometry = g
        self.step = float(step)
        self.device = int(device)
        cg, self._angles = to_c_geometry(g, step)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib.rk_plan_create(ctypes.byref(cg), self.device, ctypes.byref(h)))
        self.handle = h

    def info(self) -> dict:
        inf = _lib.RkPlanInfo()
        _lib.check(_lib.lib.rk_plan_info_get(self.handle, ctypes.byref(inf)))
        return {"forward_samples": int(inf.forward_samples), "backproject_samples": int(inf.backproject_samples),
                "device": int(inf.device), "det_count": int(inf.geometry.det_count),
                "det_spacing": float(inf.geometry.det_spacing),
                "scheduled": bool(inf.flags & 1), "schedule_from_cache": bool(inf.flags & 2)}

    def prepare(self) -> int:
        """Plan the forward schedule now (else the first forward does): loads it from the on-disk
        plan cache ($RK_PLAN_CACHE, default ~/.cache/radon_b200) or plans and stores it; returns
        the schedule's 64-bit digest (equal digests = identical launches)."""
        h = ctypes.c_uint64()
        _lib.check(_lib.lib.rk_plan_prepare(self.handle, ctypes.byref(h)))
        return int(h.value)

    def __del__(self):
        h = getattr(self, "handle", None)
        lib = getattr(_lib, "lib", None) if _lib is not None else None  # None at interpreter shutdown
        if h is not None and h.value and lib is not None:
            lib.rk_plan_destroy(h)
            self.handle = None


_PLANS: "OrderedDict" = OrderedDict()  # least recently used first
_PLANS_LOCK = threading.Lock()
_MAX_PLANS = 64


def get_plan(g: Geometry, opts: ProjectorOptions | None = None, device: int = 0) -> Plan:
    step = float((opts or ProjectorOptions()).step)
    if not (step > 0.0):  # projector.cpp:31-33
        raise ValidationError("projector step must be positive")
    key = (g, step, int(device))
    evicted = []
    with _PLANS_LOCK:
        p = _PLANS.get(key)
        if p is None:
            while len(_PLANS) >= _MAX_PLANS:  # evict the least recently used plan (callers keep theirs alive)
                evicted.append(_PLANS.popitem(last=False)[1])
            p = _PLANS[key] = Plan(g, step, device)
        else:
            _PLANS.move_to_end(key)
    # the evicted plans are released here, outside the lock: rk_plan_destroy waits for the plan's
    # own in-flight work, which must not stall other threads' get_plan calls
    del evicted
    return p


def _check_geometry(g):
    if not isinstance(g, (ParallelGeometry, FanbeamGeometry)):
        raise TypeError(f"expected ParallelGeometry or FanbeamGeometry, got {type(g).__name__}")


def check_image(image, size: int) -> None:
    """projector.cpp:15-21."""
    if len(image.shape) != 3:
        raise ValidationError(f"image must be 3-dimensional (batch, h, w), got {A.shape_str(image.shape)}")
    if image.shape[1] != size or image.shape[2] != size:
        raise ValidationError(f"image shape {A.shape_str(image.shape)} does not match geometry image_size {size}")
    if image.shape[0] < 1:
        raise ValidationError(f"tensor shape {A.shape_str(image.shape)} has a non-positive dimension")


def check_sino(sino, n_angles: int, det_count: int) -> None:
    """projector.cpp:23-29."""
    if len(sino.shape) != 3:
        raise ValidationError(f"sinogram must be 3-dimensional (batch, angles, det), got {A.shape_str(sino.shape)}")
    if sino.shape[1] != n_angles or sino.shape[2] != det_count:
        raise ValidationError(f"sinogram shape {A.shape_str(sino.shape)} does not match geometry ({n_angles} angles, "
                              f"{det_count} cells)")
    if sino.shape[0] < 1:
        raise ValidationError(f"tensor shape {A.shape_str(sino.shape)} has a non-positive dimension")


def forward(g: Geometry, image, opts: ProjectorOptions | None = None):
    """projector.hpp:19-21 / projector.cpp:228-250.  image: (B, s, s) -> (B, n_angles, det_count)."""
    _check_geometry(g)
    check_image(image, g.image_size)
    dt = A.rk_dtype(image)
    image = A.contiguous(image)
    plan = get_plan(g, opts, A.device_index(image))
    out = A.empty(image, (image.shape[0], g.n_angles, g.det_count))
    if A.is_cuda(image):
        _lib.check(_lib.lib.rk_forward(plan.handle, dt, A.ptr(image), image.shape[0], A.ptr(out), A.stream_of(image)))
    else:
        _lib.check(_lib.lib.rk_forward_host(plan.handle, dt, A.ptr(image), image.shape[0], A.ptr(out)))
    return out


def backprojection(g: Geometry, sino, opts: ProjectorOptions | None = None):
    """projector.hpp:27-29 / projector.cpp:252-274.  sino: (B, n_angles, det_count) -> (B, s, s)."""
    _check_geometry(g)
    check_sino(sino, g.n_angles, g.det_count)
    dt = A.rk_dtype(sino)
    sino = A.contiguous(sino)
    plan = get_plan(g, opts, A.device_index(sino))
    out = A.empty(sino, (sino.shape[0], g.image_size, g.image_size))
    if A.is_cuda(sino):
        _lib.check(_lib.lib.rk_backproject(plan.handle, dt, A.ptr(sino), sino.shape[0], A.ptr(out),
                                           A.stream_of(sino)))
    else:
        _lib.check(_lib.lib.rk_backproject_host(plan.handle, dt, A.ptr(sino), sino.shape[0], A.ptr(out)))
    return out


def materialize_matrix(g: Geometry, opts: ProjectorOptions | None = None):
    """projector.hpp:34 / projector.cpp:276-294: the dense (n_angles * det_count) x s^2
    system matrix as a float64 numpy array, column c = forward of the unit image c (the
    reference refuses image_size > 64).  The columns are projected in batches through
    the host-buffer path (fp64 storage, fp32 compute like every projector call here)."""
    _check_geometry(g)
    s = int(g.image_size)
    if s > 64:
        raise ValidationError(f"materialize_matrix refuses image_size {s} (> 64); the dense matrix would be too large")
    step = float((opts or ProjectorOptions()).step)
    if not (step > 0.0):  # projector.cpp:31-33
        raise ValidationError("projector step must be positive")
    rows, cols = g.n_angles * g.det_count, s * s
    mat = np.empty((rows, cols), np.float64)
    per = max(1, min(cols, (256 << 20) // max(1, 8 * (rows + cols))))  # columns per batch, <= 256 MB
    for c0 in range(0, cols, per):
        n = min(per, cols - c0)
        units = np.zeros((n, cols), np.float64)
        units[np.arange(n), c0 + np.arange(n)] = 1.0
        mat[:, c0:c0 + n] = np.asarray(forward(g, units.reshape(n, s, s), opts)).reshape(n, rows).T
    return mat
