"""ORACLE TEST INFRASTRUCTURE — not product code.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package,
and only as the checker / CPU baseline — never as the thing measured or
shipped.  The product path (``paper_2009_14788_b200``) never imports it.

Two oracles, both CPU-only:

* ``RefOracle`` — the reference itself: the UNMODIFIED radonkit sources
  under ``/root/reference/proj/core/src`` compiled in place (``oracle/Makefile``
  → ``oracle/_ref/libradonkit_ref.so``) plus an FFT shim standing in for the
  absent FFTW3 and an extern "C" face (``oracle/ref_shim``).  It is built in
  this container (where ``/root/reference`` exists) and the prebuilt ``.so``
  travels to the GPU box with the snapshot.
* ``PortOracle`` — our plain-C restatement ``oracle/radon_oracle.c``
  (→ ``oracle/_port/liboracle.so``), which follows the reference line by line
  and is pinned bit-for-bit against ``RefOracle`` and against the golden
  vectors of the reference's own tests (``tests/golden``).

Precision contract (reference ``projector.cpp:207-224``, ``tensor.cpp:111-138``):
storage dtype in == storage dtype out; projector accumulation in double;
``filter_sinogram`` arithmetic in float32.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(_HERE, "_ref", "libradonkit_ref.so")        # -march=x86-64-v3
REF_SO_V4 = os.path.join(_HERE, "_ref", "libradonkit_ref_v4.so")  # -march=x86-64-v4 (AVX-512)
_V4_FLAGS = ("avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl")


def _cpu_flags() -> set:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def cpu_model() -> str:
    """The host CPU's model name (lscpu 'Model name'), for the cpu_baseline record."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def best_ref_so() -> str:
    """The highest-ISA build of the reference this host can run (oracle/Makefile: the
    travelling stand-in for -march=native)."""
    if os.path.exists(REF_SO_V4) and all(f in _cpu_flags() for f in _V4_FLAGS):
        return REF_SO_V4
    return REF_SO
PORT_SO = os.path.join(_HERE, "_port", "liboracle.so")

FILTERS = ["ram-lak", "shepp-logan", "cosine", "hamming", "hann"]  # sino_filter.cpp:14-33
_PREC = {np.dtype(np.float16): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2}
_NO_DET = -(2**63)


@dataclass
class Geom:
    """Geometry as the reference's make_parallel / make_fanbeam receive it
    (``geometry.hpp:18-56``); ``None`` means "use the reference default"."""

    kind: str  # "parallel" | "fanbeam"
    image_size: int
    angles: np.ndarray
    det_count: Optional[int] = None
    det_spacing: Optional[float] = None
    source_distance: float = 0.0
    det_distance: Optional[float] = None
    step: float = 1.0

    @property
    def n_angles(self) -> int:
        return int(len(self.angles))

    def resolved(self) -> "Geom":
        """Apply the make_* defaults (geometry.cpp:22-55) without validation."""
        nd = self.det_count if self.det_count is not None else self.image_size
        if self.kind == "parallel":
            sp = self.det_spacing if self.det_spacing is not None else 1.0
            return Geom("parallel", self.image_size, self.angles, nd, sp, 0.0, 0.0, self.step)
        dd = self.det_distance if self.det_distance is not None else self.source_distance
        mag = (self.source_distance + dd) / self.source_distance
        sp = self.det_spacing if self.det_spacing is not None else mag * float(self.image_size) / float(nd)
        return Geom("fanbeam", self.image_size, self.angles, nd, sp, self.source_distance, dd, self.step)


class _RefGeomC(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("pad", ctypes.c_int32),
        ("image_size", ctypes.c_int64),
        ("n_angles", ctypes.c_int64),
        ("angles", ctypes.POINTER(ctypes.c_double)),
        ("det_count", ctypes.c_int64),
        ("det_spacing", ctypes.c_double),
        ("source_distance", ctypes.c_double),
        ("det_distance", ctypes.c_double),
        ("step", ctypes.c_double),
    ]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class RefOracle:
    """ctypes face of the reference compiled in place (see module doc)."""

    def __init__(self, path: str | None = None):
        path = path or best_ref_so()
        self.path = path
        self.march = "x86-64-v4" if path == REF_SO_V4 else "x86-64-v3"
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference oracle not built: {path} (run `make -C oracle ref`)")
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_adjoint_check.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]
        L.ref_estimate_alpha.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]
        L.ref_rng_uniform.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
        L.ref_landweber.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_double, ctypes.c_int, ctypes.c_void_p]
        L.ref_cgne.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
        L.ref_angles_linspace.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p]
        L.ref_float_to_half.argtypes = [ctypes.c_float]
        L.ref_float_to_half.restype = ctypes.c_uint16
        L.ref_half_to_float.argtypes = [ctypes.c_uint16]
        L.ref_half_to_float.restype = ctypes.c_float

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _geom(self, g: Geom):
        ang = np.ascontiguousarray(g.angles, dtype=np.float64)
        c = _RefGeomC()
        c.kind = 0 if g.kind == "parallel" else 1
        c.image_size = int(g.image_size)
        c.n_angles = len(ang)
        c.angles = ang.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        c.det_count = _NO_DET if g.det_count is None else int(g.det_count)
        c.det_spacing = float("nan") if g.det_spacing is None else float(g.det_spacing)
        c.source_distance = float(g.source_distance)
        c.det_distance = float("nan") if g.det_distance is None else float(g.det_distance)
        c.step = float(g.step)
        return c, ang  # keep `ang` alive while the struct is in use

    def set_num_threads(self, n: int):
        self._check(self.lib.ref_set_num_threads(int(n)))

    def num_threads(self) -> int:
        return int(self.lib.ref_num_threads())

    def resolve(self, g: Geom):
        c, keep = self._geom(g)
        nd, sp, dd = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        self._check(self.lib.ref_resolve_geometry(ctypes.byref(c), ctypes.byref(nd), ctypes.byref(sp), ctypes.byref(dd)))
        return int(nd.value), float(sp.value), float(dd.value)

    def angles_linspace(self, start, stop, n):
        out = np.empty(max(int(n), 0), np.float64)
        self._check(self.lib.ref_angles_linspace(float(start), float(stop), int(n), _ptr(out)))
        return out

    def forward(self, g: Geom, image: np.ndarray) -> np.ndarray:
        image = np.ascontiguousarray(image)
        nd = self.resolve(g)[0]
        out = np.empty((image.shape[0], g.n_angles, nd), image.dtype)
        c, keep = self._geom(g)
        self._check(self.lib.ref_forward(ctypes.byref(c), _PREC[image.dtype], ctypes.c_int64(image.shape[0]),
                                         _ptr(image), _ptr(out)))
        return out

    def backprojection(self, g: Geom, sino: np.ndarray) -> np.ndarray:
        sino = np.ascontiguousarray(sino)
        out = np.empty((sino.shape[0], g.image_size, g.image_size), sino.dtype)
        c, keep = self._geom(g)
        self._check(self.lib.ref_backprojection(ctypes.byref(c), _PREC[sino.dtype], ctypes.c_int64(sino.shape[0]),
                                                _ptr(sino), _ptr(out)))
        return out

    def make_filter(self, kind: str, det_count: int):
        k = FILTERS.index(kind)
        padded = ctypes.c_int64()
        # padded size is known only after the call: ask once for it
        p = 1
        while p < 2 * det_count:
            p <<= 1
        p = max(p, 2)
        rd = np.empty(p // 2 + 1, np.float64)
        rf = np.empty(p // 2 + 1, np.float32)
        self._check(self.lib.ref_make_filter(k, ctypes.c_int64(det_count), ctypes.byref(padded), _ptr(rd), _ptr(rf)))
        return int(padded.value), rd, rf

    def filter_sinogram(self, sino: np.ndarray, kind: str = "ram-lak") -> np.ndarray:
        sino = np.ascontiguousarray(sino)
        out = np.empty_like(sino)
        B, na, nd = sino.shape
        self._check(self.lib.ref_filter_sinogram(FILTERS.index(kind), _PREC[sino.dtype], ctypes.c_int64(B),
                                                 ctypes.c_int64(na), ctypes.c_int64(nd), _ptr(sino), _ptr(out)))
        return out

    def fbp(self, g: Geom, sino: np.ndarray, kind: str = "ram-lak") -> np.ndarray:
        sino = np.ascontiguousarray(sino)
        out = np.empty((sino.shape[0], g.image_size, g.image_size), sino.dtype)
        c, keep = self._geom(g)
        self._check(self.lib.ref_fbp(ctypes.byref(c), FILTERS.index(kind), _PREC[sino.dtype],
                                     ctypes.c_int64(sino.shape[0]), _ptr(sino), _ptr(out)))
        return out

    def shepp_logan(self, size: int, dtype=np.float32) -> np.ndarray:
        out = np.empty((1, size, size), dtype)
        self._check(self.lib.ref_shepp_logan(ctypes.c_int64(size), _PREC[np.dtype(dtype)], _ptr(out)))
        return out

    def rng_uniform(self, seed: int, n: int, pm1: bool = False) -> np.ndarray:
        out = np.empty(int(n), np.float32)
        self._check(self.lib.ref_rng_uniform(int(seed), int(n), int(bool(pm1)), _ptr(out)))
        return out

    def adjoint_check(self, g: Geom, trials: int = 8, seed: int = 0) -> float:
        c, keep = self._geom(g)
        d = ctypes.c_double()
        self._check(self.lib.ref_adjoint_check(ctypes.byref(c), int(trials), int(seed), ctypes.byref(d)))
        return float(d.value)

    def estimate_alpha(self, g: Geom, iterations: int = 20, seed: int = 0) -> float:
        c, keep = self._geom(g)
        d = ctypes.c_double()
        self._check(self.lib.ref_estimate_alpha(ctypes.byref(c), int(iterations), int(seed), ctypes.byref(d)))
        return float(d.value)

    def landweber(self, g: Geom, y: np.ndarray, guess: np.ndarray, alpha: float, iterations: int) -> np.ndarray:
        y = np.ascontiguousarray(y)
        guess = np.ascontiguousarray(guess, dtype=y.dtype)
        out = np.empty_like(guess)
        c, keep = self._geom(g)
        self._check(self.lib.ref_landweber(ctypes.byref(c), _PREC[y.dtype], y.shape[0], _ptr(y), _ptr(guess),
                                           float(alpha), int(iterations), _ptr(out)))
        return out

    def cgne(self, g: Geom, y: np.ndarray, guess: np.ndarray, max_iter: int, tolerance: float = 0.0) -> np.ndarray:
        y = np.ascontiguousarray(y)
        guess = np.ascontiguousarray(guess, dtype=y.dtype)
        out = np.empty_like(guess)
        c, keep = self._geom(g)
        self._check(self.lib.ref_cgne(ctypes.byref(c), _PREC[y.dtype], y.shape[0], _ptr(y), _ptr(guess),
                                      int(max_iter), float(tolerance), _ptr(out)))
        return out

    def float_to_half_bits(self, f: float) -> int:
        return int(self.lib.ref_float_to_half(float(f)))

    # --- shearlets (shearlet.cpp:103-330) and ADMM (admm.cpp:111-163), SURVEY 8f ranks 3-4 ---
    @staticmethod
    def _alphas(alphas):
        a = np.ascontiguousarray(alphas, dtype=np.float64)
        return a, len(a)

    def shearlet_n_coeff(self, h: int, w: int, alphas) -> int:
        a, n = self._alphas(alphas)
        nc = ctypes.c_int64()
        self._check(self.lib.ref_shearlet_plan(ctypes.c_int64(h), ctypes.c_int64(w), _ptr(a), n, ctypes.byref(nc),
                                               None, None))
        return int(nc.value)

    def shearlet_plan(self, h: int, w: int, alphas):
        """(n_coeff, scales[n_coeff], multipliers[n_coeff, h, w]) as make_plan builds them."""
        a, n = self._alphas(alphas)
        nc = ctypes.c_int64()
        self._check(self.lib.ref_shearlet_plan(ctypes.c_int64(h), ctypes.c_int64(w), _ptr(a), n, ctypes.byref(nc),
                                               None, None))
        scales = np.empty(nc.value, np.float64)
        mult = np.empty((nc.value, h, w), np.float64)
        self._check(self.lib.ref_shearlet_plan(ctypes.c_int64(h), ctypes.c_int64(w), _ptr(a), n, ctypes.byref(nc),
                                               _ptr(scales), _ptr(mult)))
        return int(nc.value), scales, mult

    def shearlet_forward(self, image: np.ndarray, alphas) -> np.ndarray:
        image = np.ascontiguousarray(image)
        B, h, w = image.shape
        nc = self.shearlet_n_coeff(h, w, alphas)
        a, n = self._alphas(alphas)
        out = np.empty((B, nc, h, w), image.dtype)
        self._check(self.lib.ref_shearlet_forward(ctypes.c_int64(h), ctypes.c_int64(w), _ptr(a), n,
                                                  _PREC[image.dtype], ctypes.c_int64(B), _ptr(image), _ptr(out)))
        return out

    def shearlet_backward(self, coeff: np.ndarray, alphas) -> np.ndarray:
        coeff = np.ascontiguousarray(coeff)
        B, nc, h, w = coeff.shape
        a, n = self._alphas(alphas)
        out = np.empty((B, h, w), coeff.dtype)
        self._check(self.lib.ref_shearlet_backward(ctypes.c_int64(h), ctypes.c_int64(w), _ptr(a), n,
                                                   _PREC[coeff.dtype], ctypes.c_int64(B), _ptr(coeff), _ptr(out)))
        return out

    def admm(self, g: Geom, sino: np.ndarray, alphas, p0: float, p1: float, outer: int, inner: int,
             weights=None) -> np.ndarray:
        sino = np.ascontiguousarray(sino)
        a, n = self._alphas(alphas)
        wts = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        out = np.empty((sino.shape[0], g.image_size, g.image_size), sino.dtype)
        c, keep = self._geom(g)
        self._check(self.lib.ref_admm(ctypes.byref(c), _ptr(a), n, _PREC[sino.dtype], ctypes.c_int64(sino.shape[0]),
                                      _ptr(sino), ctypes.c_double(p0), ctypes.c_double(p1),
                                      None if wts is None else _ptr(wts), ctypes.c_int64(outer),
                                      ctypes.c_int64(inner), _ptr(out)))
        return out


def _narrow(d: np.ndarray, dtype) -> np.ndarray:
    """Tensor::from_double_as (tensor.cpp:111-124): double -> storage, half via float."""
    dtype = np.dtype(dtype)
    if dtype == np.float64:
        return d
    if dtype == np.float32:
        return d.astype(np.float32)
    return d.astype(np.float32).astype(np.float16)


class PortOracle:
    """ctypes face of our C restatement (oracle/radon_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle port not built: {path} (run `make -C oracle port`)")
        L = self.lib = ctypes.CDLL(path)
        i64, d, vp = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        L.or_angles_linspace.argtypes = [d, d, i64, vp]
        L.or_forward_parallel.argtypes = [i64, i64, vp, i64, d, d, i64, vp, vp]
        L.or_forward_fanbeam.argtypes = [i64, i64, vp, i64, d, d, d, d, i64, vp, vp]
        L.or_backprojection_parallel.argtypes = [i64, i64, vp, i64, d, i64, vp, vp]
        L.or_backprojection_fanbeam.argtypes = [i64, i64, vp, i64, d, d, d, i64, vp, vp]
        L.or_forward_samples.argtypes = [ctypes.c_int, i64, i64, vp, i64, d, d, d, d]
        L.or_forward_samples.restype = i64
        L.or_make_filter.argtypes = [ctypes.c_int, i64, vp, vp]
        L.or_make_filter.restype = i64
        L.or_next_pow2.argtypes = [i64]
        L.or_next_pow2.restype = i64
        L.or_filter_sinogram.argtypes = [i64, i64, i64, i64, vp, vp, vp]
        L.or_shepp_logan.argtypes = [i64, vp]
        L.or_rng_uniform.argtypes = [ctypes.c_uint64, i64, ctypes.c_int, vp]
        L.or_float_to_half_array.argtypes = [i64, vp, vp]
        L.or_half_to_float_array.argtypes = [i64, vp, vp]

    def angles_linspace(self, start, stop, n):
        out = np.empty(int(n), np.float64)
        self.lib.or_angles_linspace(float(start), float(stop), int(n), _ptr(out))
        return out

    # -- projector (projector.cpp:207-274 precision dispatch around the double kernels)
    def forward(self, g: Geom, image: np.ndarray) -> np.ndarray:
        g = g.resolved()
        dt = image.dtype
        img = np.ascontiguousarray(image.astype(np.float32).astype(np.float64) if dt == np.float16
                                   else image.astype(np.float64))
        B = img.shape[0]
        out = np.empty((B, g.n_angles, g.det_count), np.float64)
        ang = np.ascontiguousarray(g.angles, np.float64)
        if g.kind == "parallel":
            self.lib.or_forward_parallel(g.image_size, g.n_angles, _ptr(ang), g.det_count, g.det_spacing, g.step, B,
                                         _ptr(img), _ptr(out))
        else:
            self.lib.or_forward_fanbeam(g.image_size, g.n_angles, _ptr(ang), g.det_count, g.det_spacing,
                                        g.source_distance, g.det_distance, g.step, B, _ptr(img), _ptr(out))
        return _narrow(out, dt)

    def backprojection(self, g: Geom, sino: np.ndarray) -> np.ndarray:
        g = g.resolved()
        dt = sino.dtype
        sg = np.ascontiguousarray(sino.astype(np.float32).astype(np.float64) if dt == np.float16
                                  else sino.astype(np.float64))
        B = sg.shape[0]
        out = np.empty((B, g.image_size, g.image_size), np.float64)
        ang = np.ascontiguousarray(g.angles, np.float64)
        if g.kind == "parallel":
            self.lib.or_backprojection_parallel(g.image_size, g.n_angles, _ptr(ang), g.det_count, g.det_spacing, B,
                                                _ptr(sg), _ptr(out))
        else:
            self.lib.or_backprojection_fanbeam(g.image_size, g.n_angles, _ptr(ang), g.det_count, g.det_spacing,
                                               g.source_distance, g.det_distance, B, _ptr(sg), _ptr(out))
        return _narrow(out, dt)

    def forward_samples(self, g: Geom) -> int:
        """Exact algorithmic forward work per image."""
        g = g.resolved()
        ang = np.ascontiguousarray(g.angles, np.float64)
        return int(self.lib.or_forward_samples(0 if g.kind == "parallel" else 1, g.image_size, g.n_angles, _ptr(ang),
                                               g.det_count, g.det_spacing, g.source_distance, g.det_distance, g.step))

    # -- filter (sino_filter.cpp:64-136)
    def make_filter(self, kind: str, det_count: int):
        p = max(int(self.lib.or_next_pow2(2 * det_count)), 2)
        rd = np.empty(p // 2 + 1, np.float64)
        rf = np.empty(p // 2 + 1, np.float32)
        padded = self.lib.or_make_filter(FILTERS.index(kind), int(det_count), _ptr(rd), _ptr(rf))
        return int(padded), rd, rf

    def filter_sinogram(self, sino: np.ndarray, kind: str = "ram-lak") -> np.ndarray:
        dt = sino.dtype
        B, na, nd = sino.shape
        padded, _, rf = self.make_filter(kind, nd)
        x = np.ascontiguousarray(sino.astype(np.float32))
        out = np.empty_like(x)
        self.lib.or_filter_sinogram(B * na, na, nd, padded, _ptr(rf), _ptr(x), _ptr(out))
        if dt == np.float64:
            return out.astype(np.float64)
        if dt == np.float16:
            return out.astype(np.float16)
        return out

    def fbp(self, g: Geom, sino: np.ndarray, kind: str = "ram-lak") -> np.ndarray:
        return self.backprojection(g, self.filter_sinogram(sino, kind))

    # -- inputs (phantom.cpp:61-101, rng.hpp:13-38)
    def shepp_logan(self, size: int, dtype=np.float32) -> np.ndarray:
        out = np.empty((1, size, size), np.float64)
        self.lib.or_shepp_logan(int(size), _ptr(out))
        return _narrow(out, dtype)

    def rng_uniform(self, seed: int, n: int, pm1: bool = False) -> np.ndarray:
        out = np.empty(int(n), np.float32)
        self.lib.or_rng_uniform(int(seed), int(n), int(bool(pm1)), _ptr(out))
        return out

    def float_to_half_bits(self, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float32)
        out = np.empty(a.shape, np.uint16)
        self.lib.or_float_to_half_array(a.size, _ptr(a), _ptr(out))
        return out

    def half_bits_to_float(self, h: np.ndarray) -> np.ndarray:
        h = np.ascontiguousarray(h, np.uint16)
        out = np.empty(h.shape, np.float32)
        self.lib.or_half_to_float_array(h.size, _ptr(h), _ptr(out))
        return out


# --------------------------------------------------------------------------
# Python restatements of the L3 drivers on top of an oracle projector, used
# for the config-5 parity tests when the reference library is unavailable.
# solvers.cpp:111-166, linop.cpp:65-80.


def rel_l2(a: np.ndarray, b: np.ndarray) -> float:
    """relative_error (tensor.cpp:406-418): ||a-b|| / ||b|| in double."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.sqrt(np.sum(b * b))
    return float(np.sqrt(np.sum((a - b) ** 2)) / den)


def mse(a: np.ndarray, b: np.ndarray) -> float:
    """mse (tensor.cpp:420-429)."""
    d = np.asarray(a, np.float64) - np.asarray(b, np.float64)
    return float(np.mean(d * d))


def batched_phantom(oracle, size: int, b: int, dtype=np.float32) -> np.ndarray:
    """test_projector.cpp:25-31: element e = phantom * (e+1) * 0.5 (set via double)."""
    base = oracle.shepp_logan(size, np.float32)[0].astype(np.float64)
    out = np.empty((b, size, size), np.float64)
    for e in range(b):
        out[e] = base * float(e + 1) * 0.5
    return _narrow(out, dtype)


def default_oracle():
    """The reference compiled in place when available, else our restatement."""
    try:
        return RefOracle()
    except (FileNotFoundError, OSError):
        return PortOracle()
