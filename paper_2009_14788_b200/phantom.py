"""Synthetic inputs: the reference's modified Shepp-Logan phantom
(``proj/core/src/phantom.cpp``) — rasterised at 400^2, bilinearly resampled
to the working size — in numpy (host-side input generation, SURVEY 8a row
a19; pinned bit-for-bit against the reference by tests/test_oracle_cpu.py).
"""
import numpy as np

from .errors import ValidationError

_SL = [(1.0, 0.69, 0.92, 0.0, 0.0, 0.0), (-0.8, 0.6624, 0.874, 0.0, -0.0184, 0.0),
       (-0.2, 0.11, 0.31, 0.22, 0.0, -18.0), (-0.2, 0.16, 0.41, -0.22, 0.0, 18.0),
       (0.1, 0.21, 0.25, 0.0, 0.35, 0.0), (0.1, 0.046, 0.046, 0.0, 0.1, 0.0), (0.1, 0.046, 0.046, 0.0, -0.1, 0.0),
       (0.1, 0.046, 0.023, -0.08, -0.605, 0.0), (0.1, 0.023, 0.023, 0.0, -0.606, 0.0),
       (0.1, 0.023, 0.046, 0.06, -0.605, 0.0)]


def shepp_logan(s, dtype=np.float32):
    """Synthetic input: modified Shepp-Logan (the reference's table, phantom.cpp:18-29)
    rasterised at 400^2 and bilinearly resampled to s^2 (phantom.cpp:61-101), numpy;
    computed in double and narrowed like Tensor::from_double_as (half via float)."""
    if int(s) < 1:  # phantom.cpp:62-63
        raise ValidationError(f"shepp_logan size must be positive, got {s}")
    base = 400
    y = (base - 1 - 2 * np.arange(base))[:, None] / base
    x = (2 * np.arange(base) + 1 - base)[None, :] / base
    img = np.zeros((base, base))
    for v, a, b, x0, y0, th in _SL:
        t = np.deg2rad(th)
        u = (x - x0) * np.cos(t) + (y - y0) * np.sin(t)
        w = -(x - x0) * np.sin(t) + (y - y0) * np.cos(t)
        img += v * ((u * u) / (a * a) + (w * w) / (b * b) <= 1.0)
    c = ((2 * np.arange(s) + 1) * base - s) / (2.0 * s)
    i0 = np.clip(np.floor(c).astype(int), 0, base - 1)
    f = np.where((c < 0) | (i0 >= base - 1), 0.0, c - np.floor(c))
    i1 = np.minimum(i0 + 1, base - 1)
    top = (1 - f)[None, :] * img[i0][:, i0] + f[None, :] * img[i0][:, i1]
    bot = (1 - f)[None, :] * img[i1][:, i0] + f[None, :] * img[i1][:, i1]
    out = np.ascontiguousarray((1 - f)[:, None] * top + f[:, None] * bot)  # row-major, like Tensor
    dtype = np.dtype(dtype)
    if dtype == np.float64:
        return out
    out = out.astype(np.float32)
    return out if dtype == np.float32 else out.astype(dtype)


