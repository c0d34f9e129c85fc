"""Acquisition geometry — mirror of ``proj/core/include/radonkit/geometry.hpp``.

Coordinate convention (geometry.hpp:10-16): the image of size s covers
[-s/2, s/2]^2; pixel (row i, col j) has centre (j - s/2 + 0.5, s/2 - i - 0.5),
so row 0 is the top; detector cell k lies at u_k = (k - det_count/2 + 0.5) *
det_spacing; angles are radians and rotate the source/detector assembly
counter-clockwise; at angle 0 parallel rays travel along +y.

Defaults and validation are applied by the C ABI (``rk_geometry_resolve``),
so Python, C++ and the CUDA plans all see one resolved geometry.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence, Union

import numpy as np

from . import _lib


@dataclass(frozen=True)
class ParallelGeometry:
    """geometry.hpp:18-23."""

    image_size: int
    angles: tuple
    det_count: int
    det_spacing: float = 1.0

    @property
    def n_angles(self) -> int:
        return len(self.angles)


@dataclass(frozen=True)
class FanbeamGeometry:
    """geometry.hpp:25-33."""

    image_size: int
    angles: tuple
    source_distance: float
    det_distance: float
    det_count: int
    det_spacing: float

    @property
    def n_angles(self) -> int:
        return len(self.angles)

    def magnification(self) -> float:
        return (self.source_distance + self.det_distance) / self.source_distance


Geometry = Union[ParallelGeometry, FanbeamGeometry]


def _to_c(kind: int, image_size: int, angles: Sequence[float], det_count=None, det_spacing=None,
          source_distance: float = 0.0, det_distance=None, step: float = 1.0):
    ang = np.ascontiguousarray(np.asarray(angles, dtype=np.float64).reshape(-1))
    g = _lib.RkGeometry()
    g.kind = kind
    g.has = ((_lib.RK_HAS_DET_COUNT if det_count is not None else 0)
             | (_lib.RK_HAS_DET_SPACING if det_spacing is not None else 0)
             | (_lib.RK_HAS_DET_DISTANCE if det_distance is not None else 0))
    g.image_size = int(image_size)
    g.n_angles = int(ang.size)
    g.angles = ang.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    g.det_count = int(det_count) if det_count is not None else 0
    g.det_spacing = float(det_spacing) if det_spacing is not None else 0.0
    g.source_distance = float(source_distance)
    g.det_distance = float(det_distance) if det_distance is not None else 0.0
    g.step = float(step)
    return g, ang


def _resolve(g_in):
    out = _lib.RkGeometry()
    _lib.check(_lib.lib.rk_geometry_resolve(ctypes.byref(g_in), ctypes.byref(out)))
    return out


def make_parallel(image_size: int, angles: Sequence[float], det_count: Optional[int] = None,
                  det_spacing: Optional[float] = None) -> ParallelGeometry:
    """geometry.cpp:22-33: det_count = image_size, det_spacing = 1.0 by default."""
    g, ang = _to_c(_lib.RK_PARALLEL, image_size, angles, det_count, det_spacing)
    r = _resolve(g)
    return ParallelGeometry(int(r.image_size), tuple(float(a) for a in ang), int(r.det_count), float(r.det_spacing))


def make_fanbeam(image_size: int, angles: Sequence[float], source_distance: float,
                 det_distance: Optional[float] = None, det_count: Optional[int] = None,
                 det_spacing: Optional[float] = None) -> FanbeamGeometry:
    """geometry.cpp:35-55: det_distance = source_distance, det_count = image_size,
    det_spacing = magnification * image_size / det_count; the source must lie
    outside the image's bounding circle."""
    g, ang = _to_c(_lib.RK_FANBEAM, image_size, angles, det_count, det_spacing, source_distance, det_distance)
    r = _resolve(g)
    return FanbeamGeometry(int(r.image_size), tuple(float(a) for a in ang), float(r.source_distance),
                           float(r.det_distance), int(r.det_count), float(r.det_spacing))


def angles_linspace(start: float, stop: float, n: int) -> list:
    """n evenly spaced angles on [start, stop), bitwise like numpy.linspace(endpoint=False)
    (geometry.cpp:67-73)."""
    out = np.empty(max(int(n), 1), np.float64)
    _lib.check(_lib.lib.rk_angles_linspace(float(start), float(stop), int(n), out.ctypes.data_as(ctypes.c_void_p)))
    return [float(v) for v in out[: int(n)]]


def geometry_image_size(g: Geometry) -> int:
    return g.image_size


def geometry_det_count(g: Geometry) -> int:
    return g.det_count


def geometry_n_angles(g: Geometry) -> int:
    return g.n_angles


def to_c_geometry(g: Geometry, step: float = 1.0):
    """Fully specified C geometry (all optional fields set) + the angle buffer to keep alive."""
    if isinstance(g, ParallelGeometry):
        return _to_c(_lib.RK_PARALLEL, g.image_size, g.angles, g.det_count, g.det_spacing, step=step)
    if isinstance(g, FanbeamGeometry):
        return _to_c(_lib.RK_FANBEAM, g.image_size, g.angles, g.det_count, g.det_spacing, g.source_distance,
                     g.det_distance, step=step)
    raise TypeError(f"not a geometry: {type(g).__name__}")
