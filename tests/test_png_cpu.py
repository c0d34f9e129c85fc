"""png_export restating proj/tests/test_png.cpp (CPU: the writer is host-side):
window mapping to exact 16-bit samples, shifted windows, accepted shapes, window
validation, atomic writes, half/double storage alike, and the CLI subcommand."""
import os
import struct
import subprocess
import sys
import zlib

import numpy as np
import pytest

import paper_2009_14788_b200 as rk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def decode(path):
    """Minimal decoder for the subset the writer emits (test_png.cpp:35-80)."""
    b = open(path, "rb").read()
    assert b[:8] == b"\x89PNG\r\n\x1a\n"
    pos, idat = 8, b""
    w = h = None
    saw_iend = False
    while pos + 8 <= len(b):
        n = struct.unpack(">I", b[pos:pos + 4])[0]
        kind = b[pos + 4:pos + 8]
        data = b[pos + 8:pos + 8 + n]
        assert struct.unpack(">I", b[pos + 8 + n:pos + 12 + n])[0] == zlib.crc32(kind + data) & 0xFFFFFFFF
        if kind == b"IHDR":
            w, h, depth, color, comp, filt, inter = struct.unpack(">IIBBBBB", data)
            assert (depth, color, comp, filt, inter) == (16, 0, 0, 0, 0)
        elif kind == b"IDAT":
            idat += data
        elif kind == b"IEND":
            saw_iend = True
        pos += 12 + n
    assert saw_iend and pos == len(b)
    raw = np.frombuffer(zlib.decompress(idat), np.uint8).reshape(h, 1 + 2 * w)
    assert (raw[:, 0] == 0).all()  # filter byte
    return w, h, raw[:, 1:].copy().view(">u2").astype(np.int64).reshape(-1)


def test_window_mapping_hits_exact_samples(tmp_path):
    p = str(tmp_path / "a.png")
    rk.png_export(np.array([[0.0, 1.0, 0.25], [0.5, -3.0, 7.0]], np.float32), p, 0.0, 1.0)
    w, h, s = decode(p)
    assert (w, h) == (3, 2)
    assert list(s) == [0, 65535, 16384, 32768, 0, 65535]


def test_shifted_window(tmp_path):
    p = str(tmp_path / "b.png")
    rk.png_export(np.array([[-1.0, 0.0], [1.0, 3.0]]), p, -1.0, 3.0)
    assert list(decode(p)[2]) == [0, 16384, 32768, 65535]


def test_accepts_hw_and_batch_of_one_rejects_the_rest(tmp_path):
    rk.png_export(np.zeros((4, 5), np.float32), str(tmp_path / "a.png"), 0.0, 1.0)
    rk.png_export(np.zeros((1, 4, 5), np.float32), str(tmp_path / "b.png"), 0.0, 1.0)
    assert decode(str(tmp_path / "a.png"))[:2] == (5, 4) and decode(str(tmp_path / "b.png"))[:2] == (5, 4)
    for bad in ((2, 4, 5), (5,)):
        with pytest.raises(rk.ValidationError, match="HxW image or a batch of one"):
            rk.png_export(np.zeros(bad, np.float32), str(tmp_path / "c.png"), 0.0, 1.0)


def test_window_validation(tmp_path):
    img = np.zeros((2, 2), np.float32)
    for lo, hi in ((1.0, 1.0), (2.0, -1.0)):
        with pytest.raises(rk.ValidationError, match="window_hi must exceed window_lo"):
            rk.png_export(img, str(tmp_path / "x.png"), lo, hi)


def test_atomic_write(tmp_path):
    p = tmp_path / "y.png"
    rk.png_export(np.ones((3, 3)), str(p), 0.0, 1.0)
    assert sorted(os.listdir(tmp_path)) == ["y.png"]  # no temporary left behind
    with pytest.raises(rk.ValidationError):
        rk.png_export(np.ones((3, 3)), str(tmp_path / "missing" / "y.png"), 0.0, 1.0)


def test_half_and_double_storage_alike(tmp_path):
    v = np.array([[0.0, 0.25], [0.5, 1.0]])
    rk.png_export(v.astype(np.float16), str(tmp_path / "h.png"), 0.0, 1.0)
    rk.png_export(v, str(tmp_path / "d.png"), 0.0, 1.0)
    ph, pd = decode(str(tmp_path / "h.png"))[2], decode(str(tmp_path / "d.png"))[2]
    assert list(ph) == list(pd) and pd[3] == 65535


def test_cli_png_export(tmp_path):
    src, dst = str(tmp_path / "img.npy"), str(tmp_path / "img.png")
    np.save(src, np.array([[0.0, 2.0], [4.0, 8.0]], np.float32))
    r = subprocess.run([sys.executable, "-m", "paper_2009_14788_b200", "png-export", "--in", src, "-o", dst,
                        "--lo", "0", "--hi", "8"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert list(decode(dst)[2]) == [0, 16384, 32768, 65535]
    r = subprocess.run([sys.executable, "-m", "paper_2009_14788_b200", "png-export", "--in", src, "-o", dst,
                        "--lo", "1", "--hi", "1"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 1
