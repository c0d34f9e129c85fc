"""The operator plug-in point of the reference (``proj/core/include/radonkit/linop.hpp``):
a batched linear map with its adjoint, plus the dot-product adjoint test and
the finite-difference gradient test (linop.cpp:33-115).

``projector_operator(g)`` returns a ``LinearOperator`` whose ``apply`` /
``adjoint`` are the B200 ``forward`` / ``backprojection``; everything the
reference builds on that struct (solvers, checks) consumes it unchanged.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _arrays as A
from .errors import ValidationError
from .geometry import Geometry
from .projector import ProjectorOptions, backprojection, forward
from .rng import Rng


@dataclass
class LinearOperator:
    """linop.hpp:14-19: shapes are per batch element (no leading batch dim)."""

    domain_shape: tuple
    range_shape: tuple
    apply: Callable
    adjoint: Callable
    geometry: Optional[Geometry] = None  # set by projector_operator (lets solvers take the fused GPU path)
    options: Optional[ProjectorOptions] = None


def projector_operator(g: Geometry, opts: ProjectorOptions | None = None) -> LinearOperator:
    """linop.cpp:33-41."""
    opts = opts or ProjectorOptions()
    s = g.image_size
    return LinearOperator((s, s), (g.n_angles, g.det_count), lambda x: forward(g, x, opts),
                          lambda y: backprojection(g, y, opts), g, opts)


def identity_operator(shape) -> LinearOperator:
    """linop.cpp:43-50."""
    shape = tuple(int(d) for d in shape)
    return LinearOperator(shape, shape, lambda x: x, lambda y: y)


def compose(a: LinearOperator, b: LinearOperator) -> LinearOperator:
    """linop.cpp:52-63: apply = a(b(x)), adjoint = b'(a'(y))."""
    if tuple(a.domain_shape) != tuple(b.range_shape):
        raise ValidationError(f"compose: inner shapes do not match, {A.shape_str(a.domain_shape)} vs "
                              f"{A.shape_str(b.range_shape)}")
    fa, fb, ga, gb = a.apply, b.apply, a.adjoint, b.adjoint
    return LinearOperator(tuple(b.domain_shape), tuple(a.range_shape), lambda x: fa(fb(x)), lambda y: gb(ga(y)))


def _work_array(host: np.ndarray):
    """Operators run on the GPU: hand them CUDA tensors when torch sees a device."""
    if A.torch is not None and A.torch.cuda.is_available():
        return A.torch.from_numpy(host).cuda()
    return host


def _np64(x) -> np.ndarray:
    if A.is_torch(x):
        return x.detach().to("cpu").double().numpy()
    return np.asarray(x, np.float64)


def dot(a, b) -> float:
    """tensor.cpp:378-384 (double accumulation)."""
    return float(np.dot(_np64(a).ravel(), _np64(b).ravel()))


def norm2(a) -> float:
    v = _np64(a).ravel()
    return float(np.sqrt(np.dot(v, v)))


def adjoint_check(op: LinearOperator, trials: int = 8, seed: int = 0) -> float:
    """linop.cpp:65-80: max over trials of |<Ax,y> - <x,A'y>| / (||Ax|| ||y|| + 1e-30),
    x, y uniform in [-1, 1) from Rng(seed), batch 1, single precision, dots in double."""
    if trials < 1:
        raise ValidationError("adjoint_check needs at least one trial")
    rng = Rng(seed)
    worst = 0.0
    for _ in range(trials):
        x = rng.uniform_pm1_tensor((1, *op.domain_shape))
        y = rng.uniform_pm1_tensor((1, *op.range_shape))
        ax = op.apply(_work_array(x))
        aty = op.adjoint(_work_array(y))
        lhs = dot(ax, y)
        rhs = dot(x, aty)
        worst = max(worst, abs(lhs - rhs) / (norm2(ax) * norm2(y) + 1e-30))
    return worst


def gradient_check(op: LinearOperator, x, step: float, n_coords: int = 32, seed: int = 0) -> float:
    """linop.cpp:82-115: central differences of L(x) = 0.5 ||Ax - y0||^2 against
    the analytic gradient A'(Ax - y0), normalised by ||grad||."""
    xs = tuple(x.shape)
    if len(xs) != len(op.domain_shape) + 1 or tuple(xs[1:]) != tuple(op.domain_shape):
        raise ValidationError(f"gradient_check point: expected batch + {A.shape_str(op.domain_shape)}, got "
                              f"{A.shape_str(xs)}")
    if not (step > 0.0):
        raise ValidationError("gradient_check step must be positive")
    if n_coords < 1:
        raise ValidationError("gradient_check needs at least one coordinate")
    rng = Rng(seed)
    xd = _np64(x)
    y0 = rng.uniform_pm1_tensor((xs[0], *op.range_shape), np.float64)
    grad = _np64(op.adjoint(_work_array(_np64(op.apply(_work_array(xd))) - y0)))
    gnorm = float(np.sqrt(np.sum(grad * grad)))
    if gnorm == 0.0:
        raise ValidationError("gradient_check: gradient vanishes at this point, the check is degenerate")

    def loss(p):
        r = _np64(op.apply(_work_array(p))) - y0
        return 0.5 * float(np.dot(r.ravel(), r.ravel()))

    n = xd.size
    samples = min(n_coords, n)
    worst = 0.0
    flat = xd.ravel()
    for k in range(samples):
        idx = k if samples == n else int(float(rng.uniform(1)[0]) * float(n))
        idx = min(idx, n - 1)
        plus = flat.copy()
        plus[idx] += step
        minus = flat.copy()
        minus[idx] -= step
        fd = (loss(plus.reshape(xd.shape)) - loss(minus.reshape(xd.shape))) / (2.0 * step)
        worst = max(worst, abs(fd - grad.ravel()[idx]))
    return worst / gnorm
