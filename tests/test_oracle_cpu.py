"""CPU: pin the oracles before trusting them.

* the C restatement (oracle/_port) against the golden vectors hard-coded in
  the reference's own tests (hex literals copied from proj/tests/*.cpp);
* the C restatement against fixtures produced by the reference itself
  (tests/golden/golden.npz, tests/golden/make_golden.py) — bit for bit;
* when oracle/_ref is built, the restatement against the reference live.
"""
import os

import numpy as np
import pytest

from oracle import Geom, batched_phantom, rel_l2

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")

H = float.fromhex
RAMP8 = [H(v) for v in ("0x1.9ce52a886ce40p-6 0x1.f4712465501b0p-4 0x1.00e5f4b8c5510p-2 0x1.7fb04868c92fep-2 "
                        "0x1.0p-1 0x1.4027dbcb9b681p-1 0x1.7f8d05a39d578p-1 0x1.c171db7355fcap-1 "
                        "0x1.f318d6abbc98ep-1").split()]
SHEPP8 = [H(v) for v in ("0x1.9ce52a886ce40p-6 0x1.f13b8894c0b3fp-4 0x1.f4b13cd482b44p-3 0x1.69e1bcbba26dep-2 "
                         "0x1.ccf6429be6621p-2 0x1.0f2619369764ep-1 0x1.2cc92328ac6d3p-1 0x1.40b79e0052092p-1 "
                         "0x1.3dbc2b3e3d7fap-1").split()]


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def test_filter_golden_bins(port):
    """test_sino_filter.cpp:14-31: exact double bins at det 8."""
    p, rd, rf = port.make_filter("ram-lak", 8)
    assert p == 16 and list(rd) == RAMP8
    assert np.array_equal(rf, np.asarray(RAMP8).astype(np.float32))
    _, sd, _ = port.make_filter("shepp-logan", 8)
    assert list(sd) == SHEPP8


def test_filter_windows_and_sizes(port):
    """test_sino_filter.cpp:33-75."""
    _, r, _ = port.make_filter("ram-lak", 8)
    f = np.arange(9) / 8.0
    for kind, win in (("cosine", np.cos(np.pi * f / 2)), ("hamming", 0.54 + 0.46 * np.cos(np.pi * f)),
                      ("hann", 0.5 + 0.5 * np.cos(np.pi * f))):
        _, w, _ = port.make_filter(kind, 8)
        np.testing.assert_allclose(w, r * win, rtol=1e-13, atol=0)
    assert port.make_filter("hann", 8)[1][-1] == 0.0
    for det, pad in ((2, 4), (3, 8), (8, 16), (9, 32), (725, 2048)):
        assert port.make_filter("ram-lak", det)[0] == pad
    for det in (8, 32, 725):
        assert 0.0 < port.make_filter("ram-lak", det)[1][0] < 0.05
    r, hm, hn = (port.make_filter(k, 32)[1] for k in ("ram-lak", "hamming", "hann"))
    assert np.all(hn <= hm + 1e-15) and np.all(hm <= r + 1e-15)


def test_angles_linspace_matches_numpy(port):
    """test_geometry.cpp:75-112."""
    a = port.angles_linspace(0.0, np.pi, 7)
    ref = [H(v) for v in ("0x0.0p+0 0x1.cb91f3bbba140p-2 0x1.cb91f3bbba140p-1 0x1.58ad76cccb8f0p+0 "
                          "0x1.cb91f3bbba140p+0 0x1.1f3b3855544c8p+1 0x1.58ad76cccb8f0p+1").split()]
    assert list(a) == ref
    assert list(port.angles_linspace(-50.0, 50.0, 5)) == [-50.0, -30.0, -10.0, 10.0, 30.0]
    assert list(port.angles_linspace(0.0, 100.0, 4)) == [0.0, 25.0, 50.0, 75.0]
    assert list(port.angles_linspace(0.0, np.pi, 4)) == [0.0, np.pi / 4, np.pi / 2, 3 * np.pi / 4]


def test_phantom_frozen_samples(port):
    """test_phantom.cpp:35-81."""
    p = port.shepp_logan(400, np.float64)[0]
    assert p[0, 0] == 0.0 and p[21, 176] == 1.0
    assert p[35, 165] == H("0x1.9999999999998p-3") and p[84, 187] == H("0x1.3333333333332p-2")
    assert p[147, 165] == H("0x1.9999999999996p-4") and p[175, 198] == H("0x1.9999999999998p-2")
    assert abs(p[200].sum() - H("0x1.5199999999998p+5")) <= 1e-9 * abs(H("0x1.5199999999998p+5"))
    p = port.shepp_logan(512, np.float64)[0]
    for (i, j), v in {(21, 242): "0x1.3p-2", (21, 253): "0x1.0p+0", (28, 209): "0x1.0d8p-3", (35, 319): "0x1.ab8p-3",
                      (42, 220): "0x1.cp-2", (42, 231): "0x1.9999999999998p-3", (42, 330): "0x1.68p-1",
                      (21, 232): "0x1.56p-5", (21, 279): "0x1.56p-5", (22, 226): "0x1.22p-5"}.items():
        assert p[i, j] == H(v)
    assert abs(p.sum() - H("0x1.fbdd018666665p+14")) <= 1e-9 * H("0x1.fbdd018666665p+14")
    p = port.shepp_logan(64, np.float64)[0]
    assert p[7, 22] == H("0x1.ecccccccccccdp-1") and p[21, 11] == 1.0 and p[28, 33] == H("0x1.3ffffffffffffp-2")
    # half representation error of the 512 phantom (test_phantom.cpp:130-140)
    d = port.shepp_logan(512, np.float64)
    h = port.shepp_logan(512, np.float16)
    assert abs(rel_l2(h, d) - 1.3603301311629248e-4) <= 1e-9 * 1.3603301311629248e-4


def test_half_codec_vectors(port):
    """test_tensor.cpp:11-27 (IEEE binary16 RNE)."""
    f2h = lambda v: int(port.float_to_half_bits(np.array([v], np.float32))[0])  # noqa: E731
    assert f2h(1.0) == 0x3C00 and f2h(0.3) == 0x34CD and f2h(0.1) == 0x2E66
    assert f2h(2048.0) == 0x6800 and f2h(2049.0) == 0x6800 and f2h(65504.0) == 0x7BFF
    assert f2h(65520.0) == 0x7C00  # overflow rounds to inf
    h2f = lambda b: float(port.half_bits_to_float(np.array([b], np.uint16))[0])  # noqa: E731
    assert h2f(0x34CD) == 0.300048828125 and h2f(0x2E66) == 0.0999755859375 and h2f(0x7BFF) == 65504.0
    # numpy's float16 cast is the same RNE codec (the GPU store uses __float2half_rn)
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 3000
    assert np.array_equal(port.float_to_half_bits(x), x.astype(np.float16).view(np.uint16))


def test_dense_2x2_matrix(port):
    """test_projector.cpp:57-73: one axis-aligned angle on a 2x2 image."""
    g = Geom("parallel", 2, np.array([0.0]))
    cols = []
    for c in range(4):
        e = np.zeros((1, 2, 2))
        e.flat[c] = 1.0
        cols.append(port.forward(g, e)[0, 0])
    A = np.stack(cols, axis=1)
    np.testing.assert_allclose(A, [[1, 0, 1, 0], [0, 1, 0, 1]], atol=1e-12)


def test_port_matches_reference_fixtures_bitwise(port, golden):
    """The restatement reproduces the reference's own outputs bit for bit."""
    names = sorted({k.split("/")[0] for k in golden.files if k.endswith("/meta")})
    assert names
    for name in names:
        kind, s, na, nd, sp, sd, dd, step = golden[f"{name}/meta"]
        g = Geom("parallel" if kind == 0 else "fanbeam", int(s), golden[f"{name}/angles"], int(nd),
                 None if np.isnan(sp) else float(sp), float(sd), None if np.isnan(dd) else float(dd), float(step))
        for tag in ("f32", "f64", "f16"):
            x = golden[f"{name}/{tag}/image"]
            f = port.forward(g, x)
            assert f.dtype == x.dtype
            assert np.array_equal(f.view(np.uint8), golden[f"{name}/{tag}/forward"].view(np.uint8)), (name, tag)
            b = port.backprojection(g, f)
            assert np.array_equal(b.view(np.uint8), golden[f"{name}/{tag}/backprojection"].view(np.uint8)), (name, tag)


def test_port_filter_matches_reference_fixtures(port, golden):
    for kind in ("ram-lak", "shepp-logan", "cosine", "hamming", "hann"):
        for nd in (8, 95, 725):
            _, rd, rf = port.make_filter(kind, nd)
            assert np.array_equal(rd, golden[f"make_filter/{kind}/{nd}/d"])
            assert np.array_equal(rf, golden[f"make_filter/{kind}/{nd}/f"])
    g = Geom("parallel", 64, golden["filter/angles"], 95)
    for kind in ("ram-lak", "hann"):
        for tag in ("f32", "f16"):
            x = golden[f"filter/{kind}/{tag}/in"]
            assert np.array_equal(port.filter_sinogram(x, kind).view(np.uint8),
                                  golden[f"filter/{kind}/{tag}/out"].view(np.uint8))
            assert np.array_equal(port.fbp(g, x, kind).view(np.uint8), golden[f"fbp/{kind}/{tag}/out"].view(np.uint8))


def test_rng_matches_reference_stream(port, golden):
    assert np.array_equal(port.rng_uniform(2024, 4096), golden["rng/seed2024"])
    assert np.array_equal(port.rng_uniform(0, 4096, True), golden["rng/seed0_pm1"])


def test_product_rng_matches_reference_stream(rk, golden):
    """The product's host-side Rng (adjoint_check / estimate_alpha start vectors)."""
    assert np.array_equal(rk.Rng(2024).uniform(4096), golden["rng/seed2024"])
    assert np.array_equal(rk.Rng(0).uniform_pm1(4096), golden["rng/seed0_pm1"])


def test_port_matches_reference_live(port, ref):
    """Random geometries against the reference compiled in place (skipped without oracle/_ref)."""
    rs = np.random.default_rng(5)
    for trial in range(6):
        s = int(rs.integers(4, 40))
        na = int(rs.integers(1, 30))
        nd = int(rs.integers(1, 60))
        sp = float(rs.uniform(0.3, 2.0))
        ang = rs.uniform(-4, 4, na)
        if trial % 2:
            g = Geom("fanbeam", s, ang, nd, sp, float(s) * rs.uniform(0.75, 3.0), float(rs.uniform(1, 3 * s)),
                     step=float(rs.uniform(0.3, 1.5)))
        else:
            g = Geom("parallel", s, ang, nd, sp, step=float(rs.uniform(0.3, 1.5)))
        x = rs.standard_normal((2, s, s)).astype(np.float32)
        assert np.array_equal(port.forward(g, x), ref.forward(g, x))
        y = rs.standard_normal((2, na, nd)).astype(np.float32)
        assert np.array_equal(port.backprojection(g, y), ref.backprojection(g, y))


def test_forward_sample_counts(port):
    """SURVEY 8d exact algorithmic work (the roofline unit)."""
    par = lambda s, na: Geom("parallel", s, port.angles_linspace(0.0, np.pi, na))  # noqa: E731
    assert port.forward_samples(par(256, 256)) == 15_826_600
    assert port.forward_samples(par(512, 512)) == 126_480_072
    assert port.forward_samples(par(512, 256)) == 63_237_608
    fan = Geom("fanbeam", 512, port.angles_linspace(0.0, 2 * np.pi, 512), source_distance=512.0)
    assert port.forward_samples(fan) == 130_608_848


def test_adjoint_defect_fixture(golden):
    """the reference pair's adjoint defects (linop.cpp:65-80), < 5e-3 (test_linop.cpp:24-29)."""
    assert 1e-4 < float(golden["adjoint/par64_90"]) < 5e-3
    assert 1e-4 < float(golden["adjoint/fan64_90_D128"]) < 5e-3


def test_batched_phantom_helper(port):
    b = batched_phantom(port, 16, 3)
    assert b.shape == (3, 16, 16) and np.allclose(b[2], 3 * b[0], atol=1e-6)


def test_reference_isa_builds_agree_bitwise():
    """oracle/Makefile builds the reference for x86-64-v3 and -v4 (AVX-512); RefOracle picks the
    highest the host runs.  -ffp-contract=off and no fast-math: the two must agree bit for bit."""
    import os

    import numpy as np
    import pytest

    from oracle import REF_SO, REF_SO_V4, Geom, RefOracle, _cpu_flags, _V4_FLAGS

    if not (os.path.exists(REF_SO) and os.path.exists(REF_SO_V4)):
        pytest.skip("reference oracle builds absent")
    if not all(f in _cpu_flags() for f in _V4_FLAGS):
        pytest.skip("host lacks AVX-512")
    a, b = RefOracle(REF_SO), RefOracle(REF_SO_V4)
    x = a.shepp_logan(48)
    x = np.concatenate([x, a.rng_uniform(3, 48 * 48).reshape(1, 48, 48)])
    for g in (Geom("parallel", 48, a.angles_linspace(0.0, np.pi, 37), 61),
              Geom("fanbeam", 48, a.angles_linspace(0.0, 2 * np.pi, 29), source_distance=80.0)):
        ya, yb = a.forward(g, x), b.forward(g, x)
        assert np.array_equal(ya, yb)
        assert np.array_equal(a.backprojection(g, ya), b.backprojection(g, ya))
        if g.kind == "parallel":
            assert np.array_equal(a.fbp(g, ya), b.fbp(g, ya))
