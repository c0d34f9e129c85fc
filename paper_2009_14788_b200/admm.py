"""l1-shearlet ADMM reconstruction — mirror of ``proj/core/include/radonkit/admm.hpp``
(paper §4.3).

``admm_reconstruct`` solves argmin_{f >= 0} ||SH(f)||_{1,w} + 0.5 ||A f - y||^2
with a shearlet split (z1, u1) and a positivity split (z2, u2); every outer
iteration warm-starts CG on (p0 A'A + (1 + p1) I) f = cg_y (admm.cpp:111-163).
For an operator made by ``projector_operator`` on CUDA data the whole loop
runs in the C library (``csrc/admm.cu``: the system term fused into the
backprojection epilogue, the shrink / dual updates fused into the shearlet
transform's last pass, no host round trip per iteration).  Any other
``LinearOperator`` runs the same recurrence composed from its apply/adjoint,
the GPU shearlet transform and ``cg``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _arrays as A
from . import _lib
from .errors import DivergenceError, ValidationError
from .linop import LinearOperator
from .projector import get_plan
from .shearlet import ShearletPlan, backward, forward


@dataclass
class AdmmParams:
    """admm.hpp:12-21."""

    p0: float = 0.02
    p1: float = 0.1
    weights: Optional[object] = None  # n_coeff values (any shape with that many), None = 3^scale / 400
    outer_iterations: int = 50
    inner_cg_iterations: int = 50


@dataclass
class AdmmState:
    """admm.hpp:23-30 (z2 >= 0 after every update)."""

    f: object = None
    z1: object = None
    u1: object = None
    z2: object = None
    u2: object = None


def default_weights(plan: ShearletPlan) -> np.ndarray:
    """admm.cpp:11-15: 3^scale / 400, shape 1 x n_coeff x 1 x 1 (fp64)."""
    return (np.power(3.0, plan.scales) / 400.0).reshape(1, plan.n_coeff, 1, 1)


def _torch():
    if A.torch is None:
        raise _lib.CudaError("torch is required for device arrays")
    return A.torch


def _on_device(x):
    """Host arrays are staged through the current CUDA device (no CPU path)."""
    torch = _torch()
    if A.is_cuda(x):
        return x, None
    if not torch.cuda.is_available():
        raise _lib.CudaError("no CUDA device is visible")
    if A.is_torch(x):
        return x.cuda(), "torch"
    return torch.from_numpy(np.ascontiguousarray(x)).cuda(), "numpy"


def _back(x, kind):
    if kind is None:
        return x
    x = x.cpu()
    return x.numpy() if kind == "numpy" else x


def _broadcast_check(ashape, bshape):
    """admm.cpp:20-37."""
    if len(ashape) != len(bshape):
        raise ValidationError(f"shrink threshold rank {len(bshape)} does not match input rank {len(ashape)}")
    for da, db in zip(ashape, bshape):
        if db != da and db != 1:
            raise ValidationError(f"shrink threshold shape {A.shape_str(bshape)} does not broadcast to "
                                  f"{A.shape_str(ashape)}")


def shrink(a, b):
    """admm.cpp:85-99: elementwise sign(a) * max(|a| - b, 0); b is a scalar or a
    tensor broadcast to a (dims of size 1 repeat), nonnegative.  fp64 storage
    computes in fp64, fp32/fp16 in fp32 (admm.cpp:67-81)."""
    torch = _torch()
    ad, kind = _on_device(a)
    if isinstance(b, (int, float)):
        if not (b >= 0.0):
            raise ValidationError(f"shrink threshold must be nonnegative, got {float(b):f}")
        bd = torch.tensor(float(b), dtype=torch.float64, device=ad.device)
        bshape = tuple(1 for _ in ad.shape)
    else:
        bd = (b if A.is_torch(b) else torch.from_numpy(np.ascontiguousarray(b))).to(ad.device).double()
        bshape = tuple(int(d) for d in bd.shape)
        _broadcast_check(tuple(int(d) for d in ad.shape), bshape)
        flat = bd.reshape(-1)
        neg = ~(flat >= 0.0)
        if bool(neg.any()):
            i = int(torch.nonzero(neg)[0])
            raise ValidationError(f"shrink threshold must be nonnegative, got {float(flat[i]):f} at index {i}")
    cdt = torch.float64 if ad.dtype == torch.float64 else torch.float32
    x = ad.to(cdt)
    t = bd.to(cdt).reshape(bshape)
    m = torch.clamp_min(x.abs() - t, 0.0)
    out = torch.where(x < 0, -m, torch.where(x > 0, m, torch.zeros_like(m)))
    return _back(out.to(ad.dtype), kind)


def _weights_vector(plan: ShearletPlan, weights) -> Optional[np.ndarray]:
    if weights is None:
        return None
    w = weights.detach().cpu().numpy() if A.is_torch(weights) else np.asarray(weights)
    w = np.ascontiguousarray(w, dtype=np.float64).reshape(-1)
    if w.size != plan.n_coeff:
        raise ValidationError(f"weights hold {w.size} values, plan has {plan.n_coeff} coefficients")
    return w


def _validate(radon_op: LinearOperator, plan: ShearletPlan, sinogram, params: AdmmParams):
    """admm.cpp:113-128 (same messages)."""
    if not (params.p0 > 0.0) or not (params.p1 > 0.0):
        raise ValidationError(f"admm penalties must be positive, got p0 = {params.p0:f}, p1 = {params.p1:f}")
    if params.outer_iterations < 0:
        raise ValidationError("admm outer_iterations must be nonnegative")
    if params.inner_cg_iterations < 1:
        raise ValidationError("admm inner_cg_iterations must be at least 1")
    if tuple(radon_op.domain_shape) != (plan.height, plan.width):
        raise ValidationError(f"operator domain {A.shape_str(radon_op.domain_shape)} does not match plan grid "
                              f"{plan.height}x{plan.width}")
    shp = tuple(int(d) for d in sinogram.shape)
    rng = tuple(radon_op.range_shape)
    if len(shp) != len(rng) + 1:
        raise ValidationError(f"sinogram shape {A.shape_str(shp)} is not batched operator range {A.shape_str(rng)}")
    if shp[1:] != rng:
        raise ValidationError(f"sinogram shape {A.shape_str(shp)} does not match operator range {A.shape_str(rng)}")


def admm_reconstruct(radon_op: LinearOperator, plan: ShearletPlan, sinogram, params: AdmmParams | None = None,
                     observer: Callable[[int, AdmmState], None] | None = None):
    """admm.cpp:111-163.  Returns f in the sinogram's storage precision;
    raises DivergenceError naming the outer iteration on a non-finite state.
    ``observer(iteration, state)`` runs after each outer iteration."""
    params = params or AdmmParams()
    _validate(radon_op, plan, sinogram, params)
    w = _weights_vector(plan, params.weights)
    y, kind = _on_device(sinogram)
    if radon_op.geometry is not None and y.dtype != _torch().float64:
        out = _admm_fused(radon_op, plan, y, params, w, observer)
    else:
        out = _admm_composed(radon_op, plan, y, params, w, observer)
    return _back(out, kind)


def _admm_fused(radon_op, plan, y, params, w, observer):
    torch = _torch()
    y = y.contiguous()
    dev = y.device.index if y.device.index is not None else torch.cuda.current_device()
    rplan = get_plan(radon_op.geometry, radon_op.options, dev)
    sh = plan._device_handle(dev)
    dt = A.rk_dtype(y)
    stream = A.stream_of(y)
    B = int(y.shape[0])
    wp = None if w is None else w.ctypes.data_as(ctypes.c_void_p)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib.rk_admm_create(rplan.handle, sh, dt, A.ptr(y), B, float(params.p0), float(params.p1), wp,
                                       int(params.inner_cg_iterations), stream, ctypes.byref(h)))
    try:
        failed = ctypes.c_int64(-1)
        if observer is None:
            st = _lib.lib.rk_admm_iterate(h, int(params.outer_iterations), ctypes.byref(failed), stream)
            _lib.check(st, failed.value)
        else:
            s, K = plan.height, plan.n_coeff
            for it in range(int(params.outer_iterations)):
                st = _lib.lib.rk_admm_iterate(h, 1, ctypes.byref(failed), stream)
                _lib.check(st, failed.value)
                shapes = [(B, s, s), (B, K, s, s), (B, K, s, s), (B, s, s), (B, s, s)]
                state = []
                cdt = torch.float32
                for which, shp in enumerate(shapes):
                    t = torch.empty(shp, dtype=cdt, device=y.device)
                    _lib.check(_lib.lib.rk_admm_read(h, which, _lib.RK_F32, A.ptr(t), stream))
                    state.append(t)
                observer(it, AdmmState(*state))
        out = torch.empty((B, plan.height, plan.width), dtype=y.dtype, device=y.device)
        _lib.check(_lib.lib.rk_admm_read(h, 0, dt, A.ptr(out), stream))
        return out
    finally:
        _lib.lib.rk_admm_destroy(h)


def _admm_composed(radon_op, plan, y, params, w, observer):
    """The same recurrence for an arbitrary LinearOperator (and fp64 storage):
    torch vector algebra on the device + the GPU shearlet transform + cg."""
    from .solvers import cg

    torch = _torch()
    store = y.dtype
    yc = y.float() if store == torch.float16 else y
    cdt = yc.dtype
    wv = torch.from_numpy(default_weights(plan).reshape(-1) if w is None else w).to(yc.device)
    thresh = (wv * (params.p0 / params.p1)).reshape(1, plan.n_coeff, 1, 1)
    if bool((~(thresh >= 0.0)).any()):
        raise ValidationError("shrink threshold must be nonnegative")
    p0, p1 = params.p0, params.p1

    def axpy(a, x, yv):  # tensor.cpp:341-347 (alpha narrowed for fp32)
        return torch.tensor(a, dtype=cdt, device=x.device) * x + yv

    def scale(x, a):
        return x * torch.tensor(a, dtype=cdt, device=x.device)

    bp = radon_op.adjoint(yc).to(cdt)
    B = bp.shape[0]
    f = torch.zeros_like(bp)
    z2 = torch.zeros_like(bp)
    u2 = torch.zeros_like(bp)
    z1 = torch.zeros((B, plan.n_coeff, plan.height, plan.width), dtype=cdt, device=bp.device)
    u1 = torch.zeros_like(z1)

    def system(x):
        return axpy(p0, radon_op.adjoint(radon_op.apply(x)), scale(x, 1.0 + p1))

    for it in range(int(params.outer_iterations)):
        cg_y = axpy(p0, bp, axpy(p1, backward(plan, z1 - u1), z2 - u2))
        f = cg(system, f, cg_y, int(params.inner_cg_iterations))
        sh_f = forward(plan, f)
        z1 = shrink(sh_f + u1, thresh.to(cdt))
        z2 = torch.clamp_min(f + u2, 0.0)
        u1 = u1 + (sh_f - z1)
        u2 = u2 + (f - z2)
        if not (bool(torch.isfinite(f).all()) and bool(torch.isfinite(u1).all()) and bool(torch.isfinite(u2).all())):
            raise DivergenceError(f"admm state became non-finite at iteration {it}", it)
        if observer is not None:
            observer(it, AdmmState(f, z1, u1, z2, u2))
    return f.to(store)


def admm_objective(radon_op: LinearOperator, plan: ShearletPlan, f, y, weights=None) -> float:
    """admm.cpp:165-184: sum |w SH(f)| + 0.5 ||A f - y||^2 accumulated in fp64."""
    torch = _torch()
    w = _weights_vector(plan, weights)
    wv = default_weights(plan).reshape(-1) if w is None else w
    fd, _ = _on_device(f)
    yd, _ = _on_device(y)
    sh = forward(plan, fd).double()
    wt = torch.from_numpy(wv).to(sh.device).reshape(1, plan.n_coeff, 1, 1)
    l1 = float((wt * sh).abs().sum())
    r = radon_op.apply(fd)
    if tuple(r.shape) != tuple(yd.shape):
        raise ValidationError(f"sinogram shape {A.shape_str(yd.shape)} does not match projected shape "
                              f"{A.shape_str(r.shape)}")
    d = r.double() - yd.double()
    return l1 + 0.5 * float((d * d).sum())
