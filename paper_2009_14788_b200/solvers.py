"""Iterative reconstruction drivers — mirror of ``proj/core/include/radonkit/solvers.hpp``
(``solvers.cpp:47-166``): power-iteration step size, Landweber, CG with
per-batch-element fp64 scalars and freeze-on-tolerance, CGNE.

For a ``projector_operator`` on CUDA tensors the whole iteration runs in the
library's fused device kernels (``rk_landweber`` / ``rk_cgne`` /
``rk_estimate_alpha``); for any other operator the same algorithm runs on
torch CUDA tensors around the operator's apply/adjoint.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _arrays as A
from . import _lib
from .errors import DivergenceError, NotPositiveDefiniteError, NumericalError, ValidationError
from .linop import LinearOperator, _np64, _work_array
from .projector import get_plan
from .rng import Rng


_FUSED = True  # fused device solvers of the C ABI (set False to run the generic torch loop)


# the fused device solvers keep whole-batch packed state in one launch (65,535 packed
# groups of four images); larger batches take the operator path, whose forward /
# backprojection calls run sub-batches (capi.cpp for_sub_batches)
_FUSED_MAX_BATCH = 65535 * 4


def _fused_ok(op: LinearOperator, batch: int = 1) -> bool:
    return (_FUSED and op.geometry is not None and A.torch is not None and A.torch.cuda.is_available()
            and batch <= _FUSED_MAX_BATCH)


def estimate_alpha(op: LinearOperator, iterations: int = 20, seed: int = 0) -> float:
    """solvers.cpp:111-128: 2 / sigma_max^2 of A'A from `iterations` power
    iterations started at Rng(seed).uniform (double), batch 1."""
    if iterations < 1:
        raise ValidationError("estimate_alpha needs at least one iteration")
    if _fused_ok(op):
        plan = get_plan(op.geometry, op.options, A.torch.cuda.current_device())
        alpha = ctypes.c_double()
        _lib.check(_lib.lib.rk_estimate_alpha(plan.handle, int(iterations), int(seed), ctypes.byref(alpha)))
        return float(alpha.value)
    x = Rng(seed).uniform_tensor((1, *op.domain_shape), np.float64)
    nx = float(np.sqrt(np.sum(x * x)))
    if nx == 0.0:
        raise NumericalError("estimate_alpha: start vector is zero")
    x = x * (1.0 / nx)
    sigma2 = 0.0
    for it in range(iterations):
        z = _np64(op.adjoint(op.apply(_work_array(x))))
        nz = float(np.sqrt(np.sum(z * z)))
        if not (nz > 0.0) or not np.isfinite(nz):
            raise NumericalError(f"estimate_alpha: power iteration collapsed at iteration {it}")
        sigma2 = nz
        x = z * (1.0 / nz)
    return 2.0 / sigma2


def _torch():
    if A.torch is None:
        raise ValidationError("solvers need torch for device vectors")
    return A.torch


def landweber(op: LinearOperator, y, guess, alpha: float, iterations: int):
    """solvers.cpp:130-145: x <- x - alpha * A'(Ax - y) in the compute precision
    (single for half/single storage), DivergenceError on a non-finite iterate."""
    if iterations < 0:
        raise ValidationError("landweber iteration count must be >= 0")
    if y.shape[0] != guess.shape[0]:
        raise ValidationError(f"landweber: y batch {y.shape[0]} does not match guess batch {guess.shape[0]}")
    if _fused_ok(op, guess.shape[0]) and A.is_cuda(y) and A.is_cuda(guess) and guess.dtype != A.torch.float64:
        return _landweber_fused(op, y, guess, alpha, iterations)
    torch = _torch()
    host = not A.is_torch(guess)
    g = torch.as_tensor(guess).cuda() if host or not guess.is_cuda else guess
    yy = torch.as_tensor(y).cuda() if not A.is_cuda(y) else y
    cdt = torch.float64 if g.dtype == torch.float64 else torch.float32
    x = g.to(cdt)
    yb = yy.to(cdt)
    a = torch.tensor(-alpha, dtype=cdt, device=x.device)
    for it in range(iterations):
        grad = op.adjoint(op.apply(x) - yb)
        x = a * grad + x
        if not bool(torch.isfinite(x).all()):
            raise DivergenceError(f"landweber produced a non-finite iterate at iteration {it}", it)
    out = x.to(g.dtype)
    return out.cpu().numpy() if host else out


def _landweber_fused(op, y, guess, alpha, iterations):
    torch = _torch()
    plan = get_plan(op.geometry, op.options, guess.device.index or 0)
    y = y.contiguous()
    guess = guess.contiguous()
    if y.dtype != guess.dtype:
        y = y.to(guess.dtype)
    out = torch.empty_like(guess)
    failed = ctypes.c_int(-1)
    st = _lib.lib.rk_landweber(plan.handle, A.rk_dtype(guess), A.ptr(y), A.ptr(guess), guess.shape[0], float(alpha),
                               int(iterations), A.ptr(out), ctypes.byref(failed), A.stream_of(guess))
    _lib.check(st, failed.value)
    return out


def cg(apply, guess, b, max_iter: int, tolerance: float = 0.0):
    """solvers.cpp:47-107,147-160: CG for an SPD apply with per-batch-element
    fp64 scalars; elements whose residual reaches tolerance * ||b|| are frozen."""
    if max_iter < 0:
        raise ValidationError("cg max_iter must be >= 0")
    if tolerance < 0.0:
        raise ValidationError("cg tolerance must be >= 0")
    if tuple(guess.shape) != tuple(b.shape):
        raise ValidationError(f"cg: guess shape {A.shape_str(guess.shape)} does not match b {A.shape_str(b.shape)}")
    torch = _torch()
    host = not A.is_torch(guess)
    g = torch.as_tensor(guess).cuda() if host or not guess.is_cuda else guess
    bb = torch.as_tensor(b).cuda() if not A.is_cuda(b) else b
    cdt = torch.float64 if g.dtype == torch.float64 else torch.float32
    x = g.to(cdt).clone()
    b0 = bb.to(cdt)
    nb = x.shape[0]
    r = b0 - apply(x)
    p = r.clone()

    def bdot(u, v):
        return (u.double() * v.double()).reshape(nb, -1).sum(1)

    rs = bdot(r, r)
    normb = torch.sqrt(bdot(b0, b0))
    done = torch.sqrt(rs) <= tolerance * normb
    for it in range(max_iter):
        if bool(done.all()):
            break
        ap = apply(p)
        pap = bdot(p, ap)
        bad = (~done) & (pap <= 0.0)
        if bool(bad.any()):
            e = int(torch.nonzero(bad)[0])
            raise NotPositiveDefiniteError(f"cg: curvature p'Ap = {float(pap[e])} is not positive for batch element "
                                           f"{e} at iteration {it}", it)
        act = (~done).view(nb, *([1] * (x.dim() - 1)))
        alpha = (rs / torch.where(done, torch.ones_like(pap), pap)).to(cdt).view_as(act.to(cdt))
        x = torch.where(act, x + alpha * p, x)
        r = torch.where(act, r - alpha * ap, r)
        rsn = bdot(r, r)
        reached = (~done) & (torch.sqrt(rsn) <= tolerance * normb)
        newly_active = (~done) & (~reached)
        beta = (rsn / rs).to(cdt).view_as(alpha)
        p = torch.where(newly_active.view_as(act), r + beta * p, p)
        rs = torch.where(done, rs, rsn)
        done = done | reached
    out = x.to(g.dtype)
    return out.cpu().numpy() if host else out


def cgne(op: LinearOperator, guess, y, max_iter: int, tolerance: float = 0.0):
    """solvers.cpp:162-166: CG on the normal equations A'A x = A'y."""
    if _fused_ok(op, guess.shape[0]) and A.is_cuda(y) and A.is_cuda(guess) and guess.dtype != A.torch.float64:
        torch = _torch()
        plan = get_plan(op.geometry, op.options, guess.device.index or 0)
        y = y.contiguous().to(guess.dtype)
        guess = guess.contiguous()
        out = torch.empty_like(guess)
        failed = ctypes.c_int(-1)
        st = _lib.lib.rk_cgne(plan.handle, A.rk_dtype(guess), A.ptr(y), A.ptr(guess), guess.shape[0], int(max_iter),
                              float(tolerance), A.ptr(out), ctypes.byref(failed), A.stream_of(guess))
        _lib.check(st, failed.value)
        return out
    b = op.adjoint(y)
    return cg(lambda x: op.adjoint(op.apply(x)), guess, b, max_iter, tolerance)
