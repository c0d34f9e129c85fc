"""Array plumbing between the Python API and the C ABI.

Accepted containers: ``torch.Tensor`` on a CUDA device (device path: the
C ABI's asynchronous ``rk_*`` calls on torch's current stream), and host
``torch.Tensor`` / ``numpy.ndarray`` (the reference-shaped ``rk_*_host``
calls: synchronous, result in host memory, like the reference's
Tensor-in/Tensor-out functions).  Storage dtypes float16/float32/float64 map
onto RK_F16/RK_F32/RK_F64 (reference Precision::{Half,Single,Double}).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ValidationError

try:  # torch is plumbing (device memory + streams), not a requirement for host arrays
    import torch
except ImportError:  # pragma: no cover
    torch = None

_NP_DT = {np.dtype(np.float16): _lib.RK_F16, np.dtype(np.float32): _lib.RK_F32, np.dtype(np.float64): _lib.RK_F64}


def _torch_dt():
    return {torch.float16: _lib.RK_F16, torch.float32: _lib.RK_F32, torch.float64: _lib.RK_F64}


def is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def is_cuda(x) -> bool:
    return is_torch(x) and x.is_cuda


def rk_dtype(x) -> int:
    if is_torch(x):
        dt = _torch_dt().get(x.dtype)
    else:
        dt = _NP_DT.get(np.asarray(x).dtype)
    if dt is None:
        raise ValidationError(f"unsupported storage dtype {x.dtype} (expected float16, float32 or float64)")
    return dt


def shape_str(shape) -> str:
    return "(" + ", ".join(str(int(d)) for d in shape) + ")"


def contiguous(x):
    if is_torch(x):
        return x.contiguous()
    return np.ascontiguousarray(x)


def ptr(x) -> ctypes.c_void_p:
    if is_torch(x):
        return ctypes.c_void_p(x.data_ptr())
    return x.ctypes.data_as(ctypes.c_void_p)


def empty(like, shape):
    if is_torch(like):
        return torch.empty(tuple(int(d) for d in shape), dtype=like.dtype, device=like.device)
    return np.empty(tuple(int(d) for d in shape), dtype=np.asarray(like).dtype)


def device_index(x) -> int:
    if is_cuda(x):
        return x.device.index if x.device.index is not None else torch.cuda.current_device()
    if torch is not None and torch.cuda.is_available():
        return torch.cuda.current_device()
    return 0


def stream_of(x) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
