"""The synthetic-input phantom (proj/tests/test_phantom.cpp:18-140): shape,
range, determinism, corners, mirror symmetry, size 1, validation and the
precision variants' exact relative errors."""
import numpy as np
import pytest

from paper_2009_14788_b200 import ValidationError
from paper_2009_14788_b200.phantom import shepp_logan


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_shape_range_determinism():
    p = shepp_logan(64)
    assert p.shape == (64, 64) and p.dtype == np.float32
    assert p.min() >= -1e-6 and p.max() == 1.0
    assert np.array_equal(p, shepp_logan(64))


@pytest.mark.parametrize("s", [32, 400, 512])
def test_corners_outside_every_ellipse(s):
    p = shepp_logan(s)
    assert p[0, 0] == p[0, s - 1] == p[s - 1, 0] == p[s - 1, s - 1] == 0.0


@pytest.mark.parametrize("s,top,bottom", [(400, 100, 50), (512, 128, 64), (64, 15, 8)])
def test_mirror_symmetry_away_from_asymmetric_ellipses(s, top, bottom):
    p = shepp_logan(s, np.float64)
    bad = (p != p[:, ::-1]).sum(1)
    assert bad[:top].sum() == 0 and bad[s - bottom:].sum() == 0
    assert bad.sum() / (s * s) < 0.10


def test_size_one_samples_the_origin():
    p = shepp_logan(1, np.float64)
    assert p.shape == (1, 1) and abs(p[0, 0] - 0.2) <= 1e-14 * 0.2


def test_validation():
    for s in (0, -8):
        with pytest.raises(ValidationError):
            shepp_logan(s)


def test_precision_variants():
    s, d, h = shepp_logan(512), shepp_logan(512, np.float64), shepp_logan(512, np.float16)
    assert (s.dtype, d.dtype, h.dtype) == (np.float32, np.float64, np.float16)
    assert _rel(s, d) < 1e-7
    assert abs(_rel(h, d) - 1.3603301311629248e-4) <= 1e-9 * 1.3603301311629248e-4
    assert abs(_rel(h, s) - 1.360358209014672e-4) <= 1e-9 * 1.360358209014672e-4
