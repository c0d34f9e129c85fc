"""GPU parity of the ramp filter, FBP, the linear-operator checks and the
iterative solvers against the reference (proj/tests/test_sino_filter.cpp,
test_linop.cpp, test_solvers.cpp, acceptance.cpp criteria 1, 4, 5)."""
import os

import numpy as np
import pytest
import torch

from oracle import Geom, batched_phantom, mse, rel_l2

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


def dev(a, cuda):
    return torch.from_numpy(np.ascontiguousarray(a)).to(cuda)


def host(t):
    return t.detach().cpu().numpy()


def ogeom(g):
    if hasattr(g, "source_distance"):
        return Geom("fanbeam", g.image_size, np.asarray(g.angles), g.det_count, g.det_spacing, g.source_distance,
                    g.det_distance)
    return Geom("parallel", g.image_size, np.asarray(g.angles), g.det_count, g.det_spacing)


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def test_filter_matches_reference_fixtures(rk, cuda, golden):
    """filter_sinogram / fbp against outputs of the reference itself (tests/golden)."""
    g = rk.make_parallel(64, list(golden["filter/angles"]), 95)
    for kind in ("ram-lak", "hann"):
        for tag, tol in (("f32", 1e-5), ("f16", 1e-3)):
            x = golden[f"filter/{kind}/{tag}/in"]
            f = rk.filter_sinogram(dev(x, cuda), rk.make_filter(kind, 95))
            assert host(f).dtype == x.dtype
            assert rel_l2(host(f), golden[f"filter/{kind}/{tag}/out"]) <= tol
            r = rk.fbp(g, dev(x, cuda), kind)
            assert rel_l2(host(r), golden[f"fbp/{kind}/{tag}/out"]) <= tol


@pytest.mark.parametrize("nd,na,B", [(8, 3, 1), (64, 10, 5), (185, 30, 4), (725, 12, 3), (1024, 6, 6), (1449, 4, 2)])
def test_filter_parity(rk, oracle, cuda, nd, na, B):
    x = oracle.rng_uniform(nd * 7 + na, B * na * nd, True).reshape(B, na, nd)
    for kind in ("ram-lak", "shepp-logan", "cosine", "hamming", "hann"):
        out = host(rk.filter_sinogram(dev(x, cuda), rk.make_filter(kind, nd)))
        assert rel_l2(out, oracle.filter_sinogram(x, kind)) <= 1e-5


def test_filter_impulse_scale_zero(rk, cuda):
    """test_sino_filter.cpp:92-129."""
    f8 = rk.make_filter("ram-lak", 8)
    d = torch.zeros(1, 1, 8, device=cuda)
    d[0, 0, 4] = 1.0
    want = [0.0, -1.0 / (9.0 * np.pi), 0.0, -1.0 / np.pi, np.pi / 4.0, -1.0 / np.pi, 0.0, -1.0 / (9.0 * np.pi)]
    np.testing.assert_allclose(host(rk.filter_sinogram(d, f8))[0, 0], want, atol=1e-6)
    assert float(rk.filter_sinogram(torch.zeros(2, 10, 64, device=cuda), rk.make_filter("hann", 64)).abs().sum()) == 0
    f16 = rk.make_filter("ram-lak", 16)
    one = torch.tensor([np.sin(0.3 * k) + 1.0 for k in range(16)], dtype=torch.float32, device=cuda).view(1, 1, 16)
    two = one.repeat(1, 2, 1)
    np.testing.assert_allclose(host(rk.filter_sinogram(two, f16))[0, 0], 0.5 * host(rk.filter_sinogram(one, f16))[0, 0],
                               rtol=1e-6, atol=1e-7)
    const = host(rk.filter_sinogram(torch.ones(1, 1, 32, device=cuda), rk.make_filter("ram-lak", 32)))[0, 0]
    assert abs(const[16]) < 0.05 and np.abs(const[8:24]).max() < 0.05 and abs(const[0]) > 5 * np.abs(const[8:24]).max()
    with pytest.raises(rk.ValidationError):
        rk.filter_sinogram(torch.zeros(1, 4, 32, device=cuda), f16)


def test_fbp_equals_filter_then_backprojection(rk, oracle, cuda):
    """test_sino_filter.cpp:164-173: bitwise on the device too."""
    ph = oracle.shepp_logan(64)
    g = rk.make_parallel(64, rk.angles_linspace(0.0, np.pi, 90), 95)
    sino = rk.forward(g, dev(ph, cuda))
    for dt in (torch.float32, torch.float16):
        s = sino.to(dt)
        a = rk.fbp(g, s, rk.FilterKind.Hann)
        b = rk.backprojection(g, rk.filter_sinogram(s, rk.make_filter(rk.FilterKind.Hann, 95)))
        assert torch.equal(a, b)


def test_fbp_quality_improves_with_angles(rk, oracle, cuda):
    """test_sino_filter.cpp:151-162."""
    ph = oracle.shepp_logan(128)
    prev = 1e300
    for na in (32, 64, 128, 256):
        g = rk.make_parallel(128, rk.angles_linspace(0.0, np.pi, na), 185)
        m = mse(host(rk.fbp(g, rk.forward(g, dev(ph, cuda)))), ph)
        assert m < prev
        prev = m
    assert prev < 3e-3


def test_fan_fbp_reconstructs(rk, oracle, cuda):
    """test_sino_filter.cpp:175-180."""
    ph = oracle.shepp_logan(64)
    g = rk.make_fanbeam(64, rk.angles_linspace(0.0, 2 * np.pi, 128), 128.0)
    rec = host(rk.fbp(g, rk.forward(g, dev(ph, cuda))))
    assert mse(rec, ph) < 0.25 * mse(np.zeros_like(ph), ph)


def test_acceptance_c1_fbp_512(rk, oracle, cuda):
    """acceptance.cpp:116-127: FBP 512/512/725 ram-lak MSE in [1e-4, 5e-4], and parity with the reference."""
    ph = oracle.shepp_logan(512)
    g = rk.make_parallel(512, rk.angles_linspace(0.0, np.pi, 512), 725)
    sino = rk.forward(g, dev(ph, cuda))
    rec = host(rk.fbp(g, sino))
    m = mse(rec, ph)
    assert 1e-4 <= m <= 5e-4
    ref = oracle.fbp(ogeom(g), host(sino))
    assert rel_l2(rec, ref) <= 1e-5


def test_acceptance_c4_half_fbp(rk, oracle, cuda):
    """acceptance.cpp:224-229: FBP MSE with half storage within 1% of single."""
    ph = oracle.shepp_logan(256)
    g = rk.make_parallel(256, rk.angles_linspace(0.0, np.pi, 256), 363)
    s = rk.forward(g, dev(ph, cuda))
    ms = mse(host(rk.fbp(g, s)), ph)
    mh = mse(host(rk.fbp(g, s.half())).astype(np.float32), ph)
    assert abs(mh - ms) <= 0.01 * ms


def test_config4_fbp_parity_small_batch(rk, oracle, cuda):
    """SURVEY 8d config 4 geometry (1024^2, 720 angles, nd 1024 and 1449) on a 2-image batch."""
    ph = oracle.shepp_logan(1024)
    for nd in (1024, 1449):
        g = rk.make_parallel(1024, rk.angles_linspace(0.0, np.pi, 720), nd)
        x = np.concatenate([ph, 0.5 * ph]).astype(np.float32)
        sino = host(rk.forward(g, dev(x, cuda)))
        for dt, tol in ((np.float32, 1e-5), (np.float16, 1e-3)):
            s = sino.astype(dt)
            rec = host(rk.fbp(g, dev(s, cuda)))
            ref = oracle.fbp(ogeom(g), s)
            assert rel_l2(rec, ref) <= tol, (nd, dt)


def test_adjoint_check_matches_reference_defect(rk, oracle, cuda, golden):
    """test_linop.cpp:24-29; the GPU pair's defect equals the reference's (not 0)."""
    gp = rk.make_parallel(64, rk.angles_linspace(0.0, np.pi, 90))
    gf = rk.make_fanbeam(64, rk.angles_linspace(0.0, 2 * np.pi, 90), 128.0)
    for g, key in ((gp, "adjoint/par64_90"), (gf, "adjoint/fan64_90_D128")):
        d = rk.adjoint_check(rk.projector_operator(g), 10, 0)
        assert d < 5e-3
        assert abs(d - float(golden[key])) < 1e-6


def test_adjoint_check_flags_wrong_adjoint(rk, cuda):
    """test_linop.cpp:40-49."""
    g = rk.make_parallel(16, rk.angles_linspace(0.0, np.pi, 12))
    good = rk.projector_operator(g)
    bad = rk.LinearOperator(good.domain_shape, good.range_shape, good.apply, lambda y: 2.0 * good.adjoint(y))
    dg, db = rk.adjoint_check(good, 10, 0), rk.adjoint_check(bad, 10, 0)
    assert db > 0.05 and db > 10 * dg


def test_gradient_check(rk, oracle, cuda):
    """test_linop.cpp:52-55 (fp64 storage, fp32 arithmetic)."""
    g = rk.make_parallel(32, rk.angles_linspace(0.0, np.pi, 45))
    assert rk.gradient_check(rk.projector_operator(g), oracle.shepp_logan(32), 1e-3) < 1e-2


def test_projector_operator_matches_free_functions(rk, oracle, cuda):
    """test_linop.cpp:88-97."""
    g = rk.make_fanbeam(32, rk.angles_linspace(0.0, 2 * np.pi, 24), 64.0)
    op = rk.projector_operator(g)
    assert op.domain_shape == (32, 32) and op.range_shape == (24, 32)
    x = dev(oracle.shepp_logan(32), cuda)
    assert torch.equal(op.apply(x), rk.forward(g, x))
    y = op.apply(x)
    assert torch.equal(op.adjoint(y), rk.backprojection(g, y))


def test_solvers_match_reference_fixtures(rk, cuda, golden):
    """estimate_alpha / Landweber / CGNE against the reference's own runs (tests/golden)."""
    g = rk.make_parallel(32, list(golden["solver/angles"]))
    op = rk.projector_operator(g)
    alpha = 0.95 * rk.estimate_alpha(op, 20, 0)
    assert abs(alpha - float(golden["solver/alpha"])) <= 1e-5 * float(golden["solver/alpha"])
    y = dev(golden["solver/y"], cuda)
    x0 = torch.zeros(3, 32, 32, device=cuda)
    lw = rk.landweber(op, y, x0, float(golden["solver/alpha"]), 20)
    assert rel_l2(host(lw), golden["solver/landweber20"]) <= 1e-5
    cg = rk.cgne(op, x0, y, 10)
    assert rel_l2(host(cg), golden["solver/cgne10"]) <= 1e-3


def test_landweber_fused_equals_generic(rk, oracle, cuda):
    """The fused device Landweber (rk_landweber) equals the generic loop over apply/adjoint."""
    from paper_2009_14788_b200 import solvers

    g = rk.make_parallel(48, rk.angles_linspace(0.0, np.pi, 40))
    op = rk.projector_operator(g)
    x = dev(batched_phantom(oracle, 48, 5), cuda)
    y = rk.forward(g, x)
    a = 0.9 * rk.estimate_alpha(op)
    fused = rk.landweber(op, y, torch.zeros_like(x), a, 7)
    solvers._FUSED = False
    try:
        generic = rk.landweber(op, y, torch.zeros_like(x), a, 7)
        cg_generic = rk.cgne(op, torch.zeros_like(x), y, 6)
    finally:
        solvers._FUSED = True
    assert torch.equal(fused, generic)
    assert rel_l2(host(rk.cgne(op, torch.zeros_like(x), y, 6)), host(cg_generic)) <= 1e-5


def test_solvers_beyond_one_launch(rk, cuda):
    """262,141 images: more than the fused solvers' one-launch state (65,535 packed groups), so
    Landweber and CGNE take the operator path (sub-batched projector calls); elements on both
    sides of the launch boundary equal their single-image (fused) runs — bitwise for Landweber
    (solvers.cpp:130-145), within fp32 CG rounding for CGNE."""
    g = rk.make_parallel(4, [0.3, 1.1, 2.0], 5)
    op = rk.projector_operator(g)
    B = 65535 * 4 + 1
    x = dev(np.random.default_rng(9).uniform(0.0, 1.0, (B, 4, 4)).astype(np.float32), cuda)
    y = rk.forward(g, x)
    z = torch.zeros_like(x)
    lw = rk.landweber(op, y, z, 0.05, 3)
    ne = rk.cgne(op, z, y, 3)
    for i in (0, 65535 * 4 - 1, 65535 * 4):
        assert torch.equal(lw[i:i + 1], rk.landweber(op, y[i:i + 1], z[i:i + 1], 0.05, 3))
        assert rel_l2(host(ne[i:i + 1]), host(rk.cgne(op, z[i:i + 1], y[i:i + 1], 3))) <= 1e-5


def test_solvers_batch_invariant(rk, oracle, cuda):
    """test_solvers.cpp:267-290: batched solver runs equal single-element runs bitwise."""
    g = rk.make_parallel(32, rk.angles_linspace(0.0, np.pi, 30))
    op = rk.projector_operator(g)
    x = dev(batched_phantom(oracle, 32, 5), cuda)
    y = rk.forward(g, x)
    z = torch.zeros_like(x)
    lw = rk.landweber(op, y, z, 1e-4, 5)
    cg = rk.cgne(op, z, y, 5)
    for e in range(5):
        assert torch.equal(lw[e:e + 1], rk.landweber(op, y[e:e + 1], z[e:e + 1], 1e-4, 5))
        assert torch.equal(cg[e:e + 1], rk.cgne(op, z[e:e + 1], y[e:e + 1], 5))


def test_landweber_divergence_raises(rk, oracle, cuda):
    """solvers.cpp:140-142: a step far beyond 2/sigma^2 diverges -> DivergenceError naming the iteration."""
    g = rk.make_parallel(16, rk.angles_linspace(0.0, np.pi, 12))
    op = rk.projector_operator(g)
    x = dev(oracle.shepp_logan(16), cuda)
    y = rk.forward(g, x)
    with pytest.raises(rk.DivergenceError) as e:
        rk.landweber(op, y, torch.zeros_like(x), 1e6, 400)
    assert e.value.iteration is not None and e.value.iteration >= 0


def test_config5_landweber_parity(rk, oracle, cuda):
    """SURVEY 8d config 5 (parallel 512, 256 angles) on a small batch, few iterations: rel L2 <= 1e-5."""
    g = rk.make_parallel(512, rk.angles_linspace(0.0, np.pi, 256))
    og = ogeom(g)
    x = batched_phantom(oracle, 512, 2)
    y = oracle.forward(og, x)
    alpha = 0.95 * rk.estimate_alpha(rk.projector_operator(g), 20, 0)
    if hasattr(oracle, "estimate_alpha"):
        ref_alpha = 0.95 * oracle.estimate_alpha(og, 20, 0)
        assert abs(alpha - ref_alpha) <= 1e-5 * ref_alpha
        ref = oracle.landweber(og, y, np.zeros_like(x), ref_alpha, 3)
        out = host(rk.landweber(rk.projector_operator(g), dev(y, cuda), torch.zeros(2, 512, 512, device=cuda),
                                ref_alpha, 3))
        assert rel_l2(out, ref) <= 1e-5


@pytest.mark.parametrize("nd", [4097, 9000, 16384])
@pytest.mark.parametrize("dtype,tol", [(np.float32, 1e-5), (np.float16, 1e-3)])
def test_filter_large_detectors_cluster_kernel(rk, oracle, cuda, nd, dtype, tol):
    """det_count 4097 .. 16384 pads to 2^14 / 2^15 points: the two-CTA cluster filter kernel
    (even / odd frequency halves, combined through distributed shared memory); the reference
    filters any size (sino_filter.cpp:98-124).  Filter and FBP against the reference."""
    rs = np.random.default_rng(nd)
    scale = 0.01 if dtype == np.float16 else 1.0
    y = (rs.standard_normal((5, 3, nd)) * scale).astype(dtype)
    for kind in ("ram-lak", "shepp-logan"):
        f = host(rk.filter_sinogram(dev(y, cuda), rk.make_filter(rk.filter_kind_from_name(kind), nd)))
        assert rel_l2(f.astype(np.float64), oracle.filter_sinogram(y, kind).astype(np.float64)) <= tol, kind
    g = rk.make_parallel(48, rk.angles_linspace(0.0, np.pi, 3), nd, 0.02)
    fb = host(rk.fbp(g, dev(y, cuda)))
    assert rel_l2(fb.astype(np.float64), oracle.fbp(ogeom(g), y).astype(np.float64)) <= tol


@pytest.mark.parametrize("nd,na", [(5, 4), (185, 7), (1024, 6), (4097, 3)])
@pytest.mark.parametrize("dtype", [np.float32, np.float16])
def test_filter_and_fbp_batched_equal_per_image_bitwise(rk, cuda, nd, na, dtype):
    """The reference filters row by row (sino_filter.cpp:98-124), so a batched filter / FBP equals
    per-image calls bit for bit; here the complex sequences pair one image's rows at two angles
    (filter.cu), never two images, so the same holds — odd angle counts (a last unpaired row),
    ragged groups, the half8 path and the cluster kernel (nd 4097) included."""
    rs = np.random.default_rng(nd + na)
    scale = 0.01 if dtype == np.float16 else 1.0
    B = 11
    y = dev((rs.standard_normal((B, na, nd)) * scale).astype(dtype), cuda)
    filt = rk.make_filter("ram-lak", nd)
    g = rk.make_parallel(32, rk.angles_linspace(0.0, np.pi, na), nd, 48.0 / nd)
    fs, fb = rk.filter_sinogram(y, filt), rk.fbp(g, y)
    for i in (0, 5, 10):
        assert torch.equal(rk.filter_sinogram(y[i:i + 1], filt), fs[i:i + 1])
        assert torch.equal(rk.fbp(g, y[i:i + 1]), fb[i:i + 1])
    assert torch.equal(rk.fbp(g, y[3:9]), fb[3:9])


def test_filter_size_limit(rk):
    with pytest.raises(rk.ValidationError, match="pads to 65536 > 32768"):
        rk.make_filter(rk.FilterKind.RamLak, 16385)
