"""``.npy`` reader / writer with the reference's contract (``npy.hpp``,
``npy.cpp:88-199``): version-1.0 files of little-endian ``<f2``/``<f4``/``<f8``
in C order, rank >= 1 with no empty extent; anything else is a
``ValidationError`` that names the offending field or byte offset.  Writes
are byte-identical to numpy's ``np.save`` (64-byte aligned header) and atomic
(a ``.tmp`` sibling renamed into place).  Host-side file I/O only — the arrays
go to the GPU through the projector API.
"""
from __future__ import annotations

import os
import re

import numpy as np

from .errors import ValidationError

_MAGIC = b"\x93NUMPY"
_DTYPES = {"<f2": np.float16, "<f4": np.float32, "<f8": np.float64}
_DESCR = {np.dtype(np.float16): "<f2", np.dtype(np.float32): "<f4", np.dtype(np.float64): "<f8"}


def _field(header: str, key: str, path: str) -> str:
    """Value text of one key of numpy's header dict literal (npy.cpp:41-66)."""
    m = re.search(r"'" + re.escape(key) + r"':\s*", header)
    if m is None:
        raise ValidationError(f"{path}: npy header is missing the '{key}' field")
    rest = header[m.end():]
    if not rest:
        raise ValidationError(f"{path}: npy header ends inside the '{key}' field")
    if rest[0] == "'":
        end = rest.find("'", 1)
        if end < 0:
            raise ValidationError(f"{path}: unterminated string in npy header")
        return rest[1:end]
    if rest[0] == "(":
        end = rest.find(")")
        if end < 0:
            raise ValidationError(f"{path}: unterminated tuple in npy header")
        return rest[:end + 1]
    m2 = re.match(r"([^,}]*)[,}]", rest)
    if m2 is None:
        raise ValidationError(f"{path}: malformed npy header")
    return m2.group(1).rstrip()


def _shape(tup: str, path: str) -> tuple:
    dims = []
    for tok in tup[1:-1].split(","):
        tok = tok.strip()
        if not tok:
            continue
        try:
            dims.append(int(tok))
        except ValueError:
            raise ValidationError(f"{path}: bad dimension '{tok}' in npy shape") from None
    return tuple(dims)


def read_array(path: str) -> np.ndarray:
    """npy.cpp:88-158."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise ValidationError(f"{path}: cannot open file") from None
    if len(data) < 10:
        raise ValidationError(f"{path}: truncated npy preamble at byte offset 0")
    if data[:6] != _MAGIC:
        raise ValidationError(f"{path}: bad npy magic at byte offset 0")
    if data[6] != 1:
        raise ValidationError(f"{path}: unsupported npy version {data[6]} at byte offset 6")
    hlen = data[8] | (data[9] << 8)
    if len(data) < 10 + hlen:
        raise ValidationError(f"{path}: truncated npy header at byte offset 10")
    header = data[10:10 + hlen].decode("latin-1")
    descr = _field(header, "descr", path)
    order = _field(header, "fortran_order", path)
    shape = _shape(_field(header, "shape", path), path)
    if order == "True":
        raise ValidationError(f"{path}: fortran_order arrays are an unsupported layout")
    if order != "False":
        raise ValidationError(f"{path}: bad fortran_order value '{order}'")
    if descr not in _DTYPES:
        raise ValidationError(f"{path}: unsupported dtype '{descr}' (expected <f2, <f4, or <f8)")
    if not shape:
        raise ValidationError(f"{path}: 0-d arrays are not supported")
    if any(d <= 0 for d in shape):
        raise ValidationError(f"{path}: empty array (shape {shape})")
    dt = np.dtype(_DTYPES[descr])
    want = int(np.prod(shape)) * dt.itemsize
    off = 10 + hlen
    got = len(data) - off
    if got < want:
        raise ValidationError(f"{path}: truncated payload at byte offset {off + got} (expected {want} payload bytes)")
    return np.frombuffer(data, dtype=dt, count=want // dt.itemsize, offset=off).reshape(shape).copy()


def write_array(path: str, x) -> None:
    """npy.cpp:160-199: numpy-identical bytes, written to ``path + '.tmp'`` then renamed."""
    a = np.ascontiguousarray(x)
    if a.dtype not in _DESCR:
        raise ValidationError(f"write_array: unsupported dtype {a.dtype}")
    dims = ", ".join(str(d) for d in a.shape) + ("," if a.ndim == 1 else "")
    header = "{'descr': '" + _DESCR[a.dtype] + "', 'fortran_order': False, 'shape': (" + dims + "), }"
    unpadded = 10 + len(header) + 1
    header += " " * ((unpadded + 63) // 64 * 64 - unpadded) + "\n"
    hb = header.encode("latin-1")
    tmp = path + ".tmp"
    try:
        with open(tmp, "wb") as f:
            f.write(_MAGIC + bytes([1, 0, len(hb) & 0xFF, len(hb) >> 8]) + hb)
            f.write(a.tobytes())
    except OSError:
        raise ValidationError(f"{path}: cannot open for writing") from None
    try:
        os.replace(tmp, path)
    except OSError as e:
        os.remove(tmp)
        raise ValidationError(f"{path}: rename failed: {e}") from None
