"""FBP sinogram filtering — mirror of ``proj/core/include/radonkit/sino_filter.hpp``.

``make_filter`` builds the band-limited Kak–Slaney ramp (spatial kernel 1/4 at
the centre tap, -1/(m pi)^2 at odd taps, laid out circularly on
P = nextpow2(2 det_count) points, doubled in the frequency domain) times one
of five windows (sino_filter.cpp:37-92).  ``filter_sinogram`` filters every
detector row in fp32 on the GPU: zero-pad, FFT, multiply, inverse FFT, crop,
scale by pi / (2 n_angles) (sino_filter.cpp:98-124).
"""
from __future__ import annotations

import ctypes
import enum
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _arrays as A
from . import _lib
from .errors import ValidationError
from .geometry import Geometry
from .projector import backprojection, get_plan


class FilterKind(enum.IntEnum):
    """sino_filter.hpp:12."""

    RamLak = 0
    SheppLogan = 1
    Cosine = 2
    Hamming = 3
    Hann = 4


def filter_kind_from_name(name: str) -> FilterKind:
    """Exact CLI spellings (sino_filter.cpp:14-22)."""
    k = ctypes.c_int()
    _lib.check(_lib.lib.rk_filter_kind_from_name(str(name).encode(), ctypes.byref(k)))
    return FilterKind(k.value)


def filter_kind_name(kind) -> str:
    return _lib.lib.rk_filter_kind_name(int(kind)).decode()


class _DeviceFilter:
    def __init__(self, kind: int, det_count: int, device: int):
        h = ctypes.c_void_p()
        _lib.check(_lib.lib.rk_filter_create(int(kind), int(det_count), int(device), ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        lib = getattr(_lib, "lib", None) if _lib is not None else None  # None at interpreter shutdown
        if h is not None and h.value and lib is not None:
            lib.rk_filter_destroy(h)
            self.handle = None


_FILTERS: dict = {}
_LOCK = threading.Lock()


def _device_filter(kind: int, det_count: int, device: int) -> _DeviceFilter:
    key = (int(kind), int(det_count), int(device))
    with _LOCK:
        f = _FILTERS.get(key)
        if f is None:
            f = _FILTERS[key] = _DeviceFilter(kind, det_count, device)
        return f


@dataclass
class FilterSpec:
    """sino_filter.hpp:18-24."""

    kind: FilterKind = FilterKind.RamLak
    det_count: int = 0
    padded_size: int = 0
    frequency_response: np.ndarray = field(default_factory=lambda: np.zeros(0))
    frequency_response_f: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))


def make_filter(kind, det_count: int, device: int | None = None) -> FilterSpec:
    """sino_filter.cpp:64-96 (kind may be a FilterKind or a name)."""
    if isinstance(kind, str):
        kind = filter_kind_from_name(kind)
    kind = FilterKind(int(kind))
    dev = A.device_index(None) if device is None else int(device)
    f = _device_filter(kind, det_count, dev)
    padded = ctypes.c_int64()
    _lib.check(_lib.lib.rk_filter_response(f.handle, ctypes.byref(padded), None, None))
    rd = np.empty(padded.value // 2 + 1, np.float64)
    rf = np.empty(padded.value // 2 + 1, np.float32)
    _lib.check(_lib.lib.rk_filter_response(f.handle, ctypes.byref(padded), rd.ctypes.data_as(ctypes.c_void_p),
                                           rf.ctypes.data_as(ctypes.c_void_p)))
    return FilterSpec(kind, int(det_count), int(padded.value), rd, rf)


def filter_sinogram(sino, filt: FilterSpec):
    """sino_filter.cpp:98-124: rows filtered in fp32, result keeps the storage precision."""
    if len(sino.shape) != 3:
        raise ValidationError(f"sinogram must be 3-dimensional (batch, angles, det), got {A.shape_str(sino.shape)}")
    if sino.shape[2] != filt.det_count:
        raise ValidationError(f"sinogram det_count {sino.shape[2]} does not match filter {filt.det_count}")
    dt = A.rk_dtype(sino)
    sino = A.contiguous(sino)
    dev = A.device_index(sino)
    f = _device_filter(filt.kind, filt.det_count, dev)
    out = A.empty(sino, sino.shape)
    B, na = int(sino.shape[0]), int(sino.shape[1])
    if A.is_cuda(sino):
        _lib.check(_lib.lib.rk_filter_sinogram(f.handle, dt, A.ptr(sino), B, na, A.ptr(out), A.stream_of(sino)))
    else:
        _lib.check(_lib.lib.rk_filter_sinogram_host(f.handle, dt, A.ptr(sino), B, na, A.ptr(out)))
    return out


def fbp(g: Geometry, sino, kind=FilterKind.RamLak):
    """sino_filter.cpp:126-136: backprojection(filter_sinogram(sino, make_filter(kind, det_count))),
    fused on the GPU (the filter writes the backprojector's packed input directly)."""
    if isinstance(kind, str):
        kind = filter_kind_from_name(kind)
    from .projector import check_sino

    check_sino(sino, g.n_angles, g.det_count)
    dt = A.rk_dtype(sino)
    sino = A.contiguous(sino)
    dev = A.device_index(sino)
    plan = get_plan(g, None, dev)
    f = _device_filter(int(kind), g.det_count, dev)
    out = A.empty(sino, (sino.shape[0], g.image_size, g.image_size))
    if A.is_cuda(sino):
        _lib.check(_lib.lib.rk_fbp(plan.handle, f.handle, dt, A.ptr(sino), sino.shape[0], A.ptr(out),
                                   A.stream_of(sino)))
    else:
        _lib.check(_lib.lib.rk_fbp_host(plan.handle, f.handle, dt, A.ptr(sino), sino.shape[0], A.ptr(out)))
    return out
