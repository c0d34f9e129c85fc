"""Shearlet plans on the host (no GPU): the fp64 multipliers the library builds
against the reference's make_plan compiled in place (oracle/_ref), and the
plan-level cases of proj/tests/test_shearlet.cpp (structure, Parseval
partition, validation, caching)."""
import os

import numpy as np
import pytest

A5 = [0.5] * 5


def host_plan(rk, n, alphas):
    return rk.make_plan(n, n, alphas, device=-1)


def test_plan_structure_5_scales(rk):
    """test_shearlet.cpp:21-52."""
    p = host_plan(rk, 64, A5)
    assert (p.height, p.width, p.n_coeff) == (64, 64, 59)
    assert p.scales[0] == 0.0
    counts = np.bincount(p.scales.astype(int))
    assert list(counts) == [1, 6, 10, 10, 14, 18]
    assert host_plan(rk, 32, A5).n_coeff == 59
    assert host_plan(rk, 128, A5).n_coeff == 59
    assert host_plan(rk, 32, [0.5]).n_coeff == 7


@pytest.mark.parametrize("n,alphas", [(64, A5), (32, [0.5]), (64, [0.0, 1.0]), (48, [0.3, 0.7, 0.5]), (16, [1.0] * 3)])
def test_multipliers_bitwise_equal_reference(rk, ref, n, alphas):
    """make_plan (shearlet.cpp:103-198) restated in shearlet_plan.cpp: same
    fp64 operations, same results bit for bit (also for grids the device
    transform rejects)."""
    nc, scales, mult = ref.shearlet_plan(n, n, alphas)
    p = host_plan(rk, n, alphas)
    assert p.n_coeff == nc
    assert np.array_equal(p.scales, scales)
    assert np.array_equal(p.multipliers, mult)


def test_parseval_partition(rk):
    """test_shearlet.cpp:54-64: sum_k M_k^2 == 1 at every bin."""
    p = host_plan(rk, 64, A5)
    s = (p.multipliers ** 2).sum(0)
    assert np.abs(s - 1.0).max() <= 1e-12


def test_plan_validation(rk):
    """test_shearlet.cpp:141-149 (ValidationError with the reference's messages)."""
    for args in [(64, 32, A5), (1, 1, A5), (64, 64, []), (64, 64, [0.5] * 9), (64, 64, [0.5, 1.5]), (64, 64, [-0.1])]:
        with pytest.raises(rk.ValidationError):
            rk.make_plan(*args, device=-1)
    with pytest.raises(rk.ValidationError, match="square grid, got 64x32"):
        rk.make_plan(64, 32, A5, device=-1)
    host_plan(rk, 64, [0.0, 1.0])


def test_library_validation_matches_python(rk):
    """The C ABI repeats the checks (a C caller gets the same ValidationError)."""
    import ctypes

    from paper_2009_14788_b200 import _lib

    a = np.array([0.5, 1.5])
    h = ctypes.c_void_p()
    st = _lib.lib.rk_shearlet_create(64, 64, a.ctypes.data_as(ctypes.c_void_p), 2, -1, ctypes.byref(h))
    assert st == _lib.RK_ERR_VALIDATION
    assert b"outside [0, 1]" in _lib.lib.rk_last_error()


def test_plan_caching(rk, tmp_path, monkeypatch):
    """test_shearlet.cpp:159-203: stored file named like the reference's, reused,
    corrupt/stale files rebuilt, RADONKIT_CACHE_DIR honoured, no dir -> no cache."""
    d = str(tmp_path)
    fresh = host_plan(rk, 32, A5)
    stored = rk.make_plan_cached(32, 32, A5, d, device=-1)
    path = os.path.join(d, "shearlet_32x32_a0.5_0.5_0.5_0.5_0.5_v1.npy")
    assert os.path.exists(path)
    assert np.array_equal(stored.multipliers, fresh.multipliers)
    loaded = rk.make_plan_cached(32, 32, A5, d, device=-1)
    assert np.array_equal(loaded.multipliers, fresh.multipliers) and loaded.n_coeff == 59
    with open(path, "wb") as f:
        f.write(b"not an npy file")
    rebuilt = rk.make_plan_cached(32, 32, A5, d, device=-1)
    assert np.array_equal(rebuilt.multipliers, fresh.multipliers)
    np.save(path, np.zeros((3, 32, 32)))  # stale shape
    assert np.array_equal(rk.make_plan_cached(32, 32, A5, d, device=-1).multipliers, fresh.multipliers)
    assert np.load(path).shape == (59, 32, 32)
    envd = str(tmp_path / "env")
    monkeypatch.setenv("RADONKIT_CACHE_DIR", envd)
    viaenv = rk.make_plan_cached(32, 32, A5, device=-1)
    assert np.array_equal(viaenv.multipliers, fresh.multipliers)
    assert os.path.exists(os.path.join(envd, os.path.basename(path)))
    monkeypatch.delenv("RADONKIT_CACHE_DIR")
    plain = rk.make_plan_cached(32, 32, [0.5], device=-1)
    assert plain.n_coeff == 7


def test_stored_plan_uses_file_verbatim(rk, tmp_path):
    """A cache entry is used as stored (shearlet.cpp:224-237), not rebuilt."""
    d = str(tmp_path)
    p = rk.make_plan_cached(16, 16, [0.5], d, device=-1)
    path = os.path.join(d, "shearlet_16x16_a0.5_v1.npy")
    m = p.multipliers.copy()
    m[0, 0, 0] = 0.25
    np.save(path, m)
    q = rk.make_plan_cached(16, 16, [0.5], d, device=-1)
    assert q.multipliers[0, 0, 0] == 0.25


def test_reference_shearlet_matches_numpy(ref):
    """Pins the oracle: the reference's rfft2-based analysis (through the
    oracle's FFT shim) equals Re(ifft2(fft2(x) M_k)) from numpy, and
    synthesis inverts it (test_shearlet.cpp:66-97 on the oracle)."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 32, 32))
    _, _, m = ref.shearlet_plan(32, 32, A5)
    c = ref.shearlet_forward(x, A5)
    cn = np.real(np.fft.ifft2(np.fft.fft2(x)[:, None] * m[None]))
    assert np.abs(c - cn).max() <= 1e-13
    assert np.abs(ref.shearlet_backward(c, A5) - x).max() <= 1e-13
    assert abs((c * c).sum() - (x * x).sum()) <= 1e-12 * (x * x).sum()
