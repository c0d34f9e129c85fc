"""Alpha-shearlet frame — mirror of ``proj/core/include/radonkit/shearlet.hpp``
(the transform the ADMM reconstruction is built on).

A plan holds cone-adapted, real-valued alpha-shearlet windows as full-grid
Fourier multipliers, jointly normalised to a Parseval frame
(shearlet.cpp:103-198).  Coefficient k of an image x is
Re(ifft2(fft2(x) * M_k)); synthesis applies the same multipliers and sums,
the exact adjoint (shearlet.cpp:253-294).  The multipliers are built in fp64
on the host by the C library; ``forward`` / ``backward`` run on the GPU
(``csrc/shearlet.cu``: shared-memory radix-2 row FFTs with the multiply,
conjugations, normalisation and the synthesis sum fused into their loads and
stores), fp32 arithmetic for every storage dtype.

Host arrays (numpy / CPU torch) are staged through the current CUDA device
and returned on the host in their own dtype; there is no CPU transform.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _arrays as A
from . import _lib
from .errors import CudaError, ValidationError
from .linop import LinearOperator
from .npy import read_array, write_array


def _validate_config(height: int, width: int, alphas) -> None:
    """shearlet.cpp:68-80 (same messages)."""
    if height != width:
        raise ValidationError(f"shearlet plan requires a square grid, got {height}x{width}")
    if height < 2:
        raise ValidationError("shearlet plan grid must be at least 2x2")
    if len(alphas) == 0 or len(alphas) > 8:
        raise ValidationError(f"shearlet plan needs between 1 and 8 scales, got {len(alphas)}")
    for a in alphas:
        if not (0.0 <= a <= 1.0):
            raise ValidationError(f"shearlet alpha {a:f} is outside [0, 1]")


class _Handle:
    def __init__(self, h: ctypes.c_void_p):
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        lib = getattr(_lib, "lib", None) if _lib is not None else None  # None at interpreter shutdown
        if h is not None and h.value and lib is not None:
            lib.rk_shearlet_destroy(h)
            self.h = None


class ShearletPlan:
    """shearlet.hpp:16-31.  ``multipliers`` (n_coeff x h x w, fp64) is read
    from the library on first access; device copies are made per CUDA device
    on first use."""

    def __init__(self, height: int, width: int, alphas, handle: _Handle, device: int):
        self.height = int(height)
        self.width = int(width)
        self.alphas = [float(a) for a in alphas]
        self._handles = {device: handle}
        self._lock = threading.Lock()
        nc = ctypes.c_int64()
        _lib.check(_lib.lib.rk_shearlet_info(handle.h, ctypes.byref(nc), None, None))
        self.n_coeff = int(nc.value)
        self.scales = np.empty(self.n_coeff, np.float64)
        _lib.check(_lib.lib.rk_shearlet_info(handle.h, None, self.scales.ctypes.data_as(ctypes.c_void_p), None))
        self._mult = None

    @property
    def multipliers(self) -> np.ndarray:
        if self._mult is None:
            m = np.empty((self.n_coeff, self.height, self.width), np.float64)
            h = next(iter(self._handles.values()))
            _lib.check(_lib.lib.rk_shearlet_info(h.h, None, None, m.ctypes.data_as(ctypes.c_void_p)))
            self._mult = m
        return self._mult

    def _device_handle(self, device: int) -> ctypes.c_void_p:
        with self._lock:
            hd = self._handles.get(device)
            if hd is None:
                m = self.multipliers
                a = np.asarray(self.alphas, np.float64)
                h = ctypes.c_void_p()
                _lib.check(_lib.lib.rk_shearlet_create_stored(self.height, self.width,
                                                              a.ctypes.data_as(ctypes.c_void_p), len(a),
                                                              m.ctypes.data_as(ctypes.c_void_p), int(device),
                                                              ctypes.byref(h)))
                hd = self._handles[device] = _Handle(h)
            return hd.h


def _create(height: int, width: int, alphas, stored: np.ndarray | None, device: int) -> ShearletPlan:
    a = np.asarray(alphas, np.float64)
    h = ctypes.c_void_p()
    if stored is None:
        _lib.check(_lib.lib.rk_shearlet_create(int(height), int(width), a.ctypes.data_as(ctypes.c_void_p), len(a),
                                               int(device), ctypes.byref(h)))
    else:
        stored = np.ascontiguousarray(stored, np.float64)
        _lib.check(_lib.lib.rk_shearlet_create_stored(int(height), int(width), a.ctypes.data_as(ctypes.c_void_p),
                                                      len(a), stored.ctypes.data_as(ctypes.c_void_p), int(device),
                                                      ctypes.byref(h)))
    plan = ShearletPlan(height, width, alphas, _Handle(h), int(device))
    if stored is not None:
        plan._mult = stored
    return plan


def _default_device() -> int:
    """The current CUDA device, or -1 (host-only plan) when none is visible."""
    if A.torch is not None and A.torch.cuda.is_available():
        return A.torch.cuda.current_device()
    return -1


def make_plan(height: int, width: int, alphas, device: int | None = None) -> ShearletPlan:
    """shearlet.cpp:103-199; (512, 512, [0.5]*5) gives 59 coefficients."""
    alphas = [float(x) for x in alphas]
    _validate_config(int(height), int(width), alphas)
    return _create(height, width, alphas, None, _default_device() if device is None else int(device))


def _cache_name(height: int, width: int, alphas) -> str:
    """shearlet.cpp:212-219: shearlet_{h}x{w}_a{%g joined by _}_v1.npy."""
    return f"shearlet_{height}x{width}_a" + "_".join("%g" % a for a in alphas) + "_v1.npy"


def make_plan_cached(height: int, width: int, alphas, cache_dir: str = "", device: int | None = None) -> ShearletPlan:
    """shearlet.cpp:201-249: load the multipliers from ``cache_dir`` (else
    $RADONKIT_CACHE_DIR; neither set -> no caching) when a matching fp64
    n_coeff x h x w .npy exists, else build and store them.  The file format
    is the reference's, so caches are shared with it."""
    alphas = [float(x) for x in alphas]
    _validate_config(int(height), int(width), alphas)
    dev = _default_device() if device is None else int(device)
    d = cache_dir or os.environ.get("RADONKIT_CACHE_DIR", "")
    if not d:
        return make_plan(height, width, alphas, dev)
    path = os.path.join(d, _cache_name(int(height), int(width), alphas))
    k = [int(np.ceil(np.exp2(j * (1.0 - a)))) for j, a in enumerate(alphas)]
    n_coeff = 1 + sum(2 * (2 * kj + 1) for kj in k)
    if os.path.exists(path):
        try:
            stored = read_array(path)
            if stored.dtype == np.float64 and stored.shape == (n_coeff, int(height), int(width)):
                return _create(height, width, alphas, stored, dev)
        except ValidationError:
            pass  # corrupt entry: rebuild (shearlet.cpp:238-242)
    plan = make_plan(height, width, alphas, dev)
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    write_array(path, plan.multipliers)  # atomic, like the reference's cache write
    return plan


def _run(entry, plan: ShearletPlan, x, out_shape, batch: int):
    dt = A.rk_dtype(x)
    if A.is_cuda(x):
        x = x.contiguous()
        out = A.torch.empty(out_shape, dtype=x.dtype, device=x.device)
        h = plan._device_handle(x.device.index if x.device.index is not None else A.torch.cuda.current_device())
        _lib.check(entry(h, dt, A.ptr(x), batch, A.ptr(out), A.stream_of(x)))
        return out
    if A.torch is None or not A.torch.cuda.is_available():
        raise CudaError("the shearlet transform runs on the GPU and no CUDA device is visible")
    torch = A.torch
    host_np = not A.is_torch(x)
    xd = (torch.from_numpy(np.ascontiguousarray(x)) if host_np else x.contiguous()).cuda()
    out = _run(entry, plan, xd, out_shape, batch)
    out = out.cpu()
    return out.numpy() if host_np else out


def forward(plan: ShearletPlan, image):
    """shearlet.cpp:296-311: batch x H x W -> batch x n_coeff x H x W."""
    shp = tuple(int(d) for d in image.shape)
    if len(shp) != 3 or shp[1] != plan.height or shp[2] != plan.width:
        raise ValidationError(f"shearlet forward: image shape {A.shape_str(shp)} does not match plan "
                              f"{plan.height}x{plan.width}")
    return _run(_lib.lib.rk_shearlet_forward, plan, image, (shp[0], plan.n_coeff, plan.height, plan.width), shp[0])


def backward(plan: ShearletPlan, coeff):
    """shearlet.cpp:313-330: batch x n_coeff x H x W -> batch x H x W (exact adjoint)."""
    shp = tuple(int(d) for d in coeff.shape)
    if len(shp) != 4 or shp[1] != plan.n_coeff or shp[2] != plan.height or shp[3] != plan.width:
        raise ValidationError(f"shearlet backward: coefficient shape {A.shape_str(shp)} does not match plan "
                              f"({plan.n_coeff} coefficients, {plan.height}x{plan.width})")
    return _run(_lib.lib.rk_shearlet_backward, plan, coeff, (shp[0], plan.height, plan.width), shp[0])


def shearlet_operator(plan: ShearletPlan) -> LinearOperator:
    """shearlet.cpp:332-340."""
    return LinearOperator((plan.height, plan.width), (plan.n_coeff, plan.height, plan.width),
                          lambda x: forward(plan, x), lambda c: backward(plan, c))
