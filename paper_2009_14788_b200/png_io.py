"""png_export (png_io.hpp:12 / png_io.cpp:37-103): an H x W image (or a batch of
one) as a 16-bit grayscale PNG, window [lo, hi] mapped linearly to 0 .. 65535
(clamped, rounded half away from zero like std::lround), deflate via zlib,
written atomically (temporary file + rename).  Host-side output format beside
the .npy reader/writer; no device work."""
from __future__ import annotations

import os
import struct
import zlib

import numpy as np

from .errors import NumericalError, ValidationError


def _chunk(kind: bytes, data: bytes) -> bytes:
    return struct.pack(">I", len(data)) + kind + data + struct.pack(">I", zlib.crc32(kind + data) & 0xFFFFFFFF)


def png_export(image, path: str, lo: float, hi: float) -> None:
    """png_io.cpp:37-103 (same validation messages)."""
    if not (hi > lo):
        raise ValidationError("png_export: window_hi must exceed window_lo")
    try:  # torch tensors (any device) or numpy arrays; values as double (Tensor::at)
        import torch

        if isinstance(image, torch.Tensor):
            image = image.detach().cpu().numpy()
    except ImportError:  # pragma: no cover - torch is always present here
        pass
    x = np.asarray(image)
    if x.ndim == 2:
        h, w = x.shape
    elif x.ndim == 3 and x.shape[0] == 1:
        h, w = x.shape[1], x.shape[2]
    else:
        shape = "[" + ", ".join(str(d) for d in x.shape) + "]"
        raise ValidationError(f"png_export expects an HxW image or a batch of one, got {shape}")
    v = (x.reshape(h, w).astype(np.float64) - float(lo)) / (float(hi) - float(lo))
    v = np.clip(v, 0.0, 1.0)
    q = np.floor(v * 65535.0 + 0.5).astype(">u2")  # lround of a value in [0, 65535]
    raw = np.zeros((h, 1 + 2 * w), np.uint8)  # one filter byte (0 = none) per row
    raw[:, 1:] = q.view(np.uint8).reshape(h, 2 * w)
    try:
        comp = zlib.compress(raw.tobytes(), zlib.Z_DEFAULT_COMPRESSION)
    except zlib.error as e:  # pragma: no cover
        raise NumericalError("png_export: deflate failed") from e
    ihdr = struct.pack(">IIBBBBB", w, h, 16, 0, 0, 0, 0)
    data = b"\x89PNG\r\n\x1a\n" + _chunk(b"IHDR", ihdr) + _chunk(b"IDAT", comp) + _chunk(b"IEND", b"")
    tmp = str(path) + ".tmp"
    try:
        with open(tmp, "wb") as f:
            f.write(data)
    except OSError:
        raise ValidationError(f"{path}: cannot open for writing") from None
    try:
        os.replace(tmp, path)
    except OSError as e:
        try:
            os.remove(tmp)
        except OSError:
            pass
        raise ValidationError(f"{path}: rename failed: {e.strerror}") from None
