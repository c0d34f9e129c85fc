"""GPU shearlet transform (csrc/shearlet.cu) against the reference's
forward/backward compiled in place (oracle/_ref) and the transform-level
cases of proj/tests/test_shearlet.cpp: roundtrip per precision, zeros,
Parseval energy, fp32 tracking fp64, shift covariance, the operator wrapper
and shape validation."""
import numpy as np
import pytest
import torch

from oracle import rel_l2

pytestmark = pytest.mark.gpu

A5 = [0.5] * 5


def dev(a, cuda):
    return torch.from_numpy(np.ascontiguousarray(a)).to(cuda)


def host(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def plan64(rk):
    return rk.make_plan(64, 64, A5)


@pytest.mark.parametrize("n,alphas,batch", [(64, A5, 3), (32, [0.5], 5), (128, [0.0, 1.0, 0.5], 2), (16, [1.0], 1)])
def test_forward_backward_match_reference_f32(rk, ref, cuda, n, alphas, batch):
    rng = np.random.default_rng(n + batch)
    x = rng.standard_normal((batch, n, n)).astype(np.float32)
    p = rk.make_plan(n, n, alphas)
    c = host(rk.forward(p, dev(x, cuda)))
    cr = ref.shearlet_forward(x, alphas)
    assert c.shape == cr.shape
    assert rel_l2(c, cr) <= 1e-5
    for k in range(p.n_coeff):  # every coefficient plane on its own (the low-energy ones too)
        assert rel_l2(c[:, k], cr[:, k]) <= 1e-4, k
    b = host(rk.backward(p, dev(cr, cuda)))
    assert rel_l2(b, ref.shearlet_backward(cr, alphas)) <= 1e-5


def test_forward_backward_match_reference_f64(rk, ref, cuda, plan64):
    x = np.random.default_rng(7).standard_normal((2, 64, 64))
    c = host(rk.forward(plan64, dev(x, cuda)))
    cr = ref.shearlet_forward(x, A5)
    assert c.dtype == np.float64
    assert rel_l2(c, cr) <= 1e-12
    assert rel_l2(host(rk.backward(plan64, dev(cr, cuda))), ref.shearlet_backward(cr, A5)) <= 1e-12


def test_forward_matches_reference_f16(rk, ref, cuda, plan64):
    x = np.random.default_rng(8).standard_normal((2, 64, 64)).astype(np.float16)
    c = host(rk.forward(plan64, dev(x, cuda)))
    cr = ref.shearlet_forward(x, A5)
    assert c.dtype == np.float16
    assert rel_l2(c.astype(np.float64), cr.astype(np.float64)) <= 1e-3


def test_roundtrip_per_precision_and_zeros(rk, cuda, plan64):
    """test_shearlet.cpp:66-90."""
    x = np.random.default_rng(3).standard_normal((1, 64, 64))
    for dt, tol in ((np.float32, 1e-5), (np.float64, 1e-12), (np.float16, 1e-3)):
        xd = dev(x.astype(dt), cuda)
        c = rk.forward(plan64, xd)
        assert tuple(c.shape) == (1, 59, 64, 64) and c.dtype == xd.dtype
        assert rel_l2(host(rk.backward(plan64, c)).astype(np.float64), x.astype(dt).astype(np.float64)) < tol
    assert float(rk.forward(plan64, torch.zeros(1, 64, 64, device=cuda)).abs().sum()) == 0.0
    assert float(rk.backward(plan64, torch.zeros(1, 59, 64, 64, device=cuda)).abs().sum()) == 0.0


def test_parseval_energy(rk, cuda, plan64):
    """test_shearlet.cpp:92-97."""
    x = dev(np.random.default_rng(4).standard_normal((1, 64, 64)), cuda)
    c = rk.forward(plan64, x)
    assert abs(float((c * c).sum()) - float((x * x).sum())) <= 1e-12 * float((x * x).sum())


def test_single_tracks_double(rk, cuda, plan64):
    """test_shearlet.cpp:99-105."""
    x = np.random.default_rng(5).standard_normal((1, 64, 64))
    cd = host(rk.forward(plan64, dev(x, cuda)))
    cs = host(rk.forward(plan64, dev(x.astype(np.float32), cuda)))
    assert rel_l2(cs.astype(np.float64), cd) < 1e-6


def test_shift_covariance(rk, cuda, plan64):
    """test_shearlet.cpp:107-127: SH(shift(x)) == shift(SH(x)) (fp64)."""
    x = np.random.default_rng(6).standard_normal((1, 64, 64))
    c = host(rk.forward(plan64, dev(x, cuda)))
    cs = host(rk.forward(plan64, dev(np.roll(x, (5, -3), axis=(1, 2)), cuda)))
    ref_shift = np.roll(c, (5, -3), axis=(2, 3))
    assert np.sqrt(((cs - ref_shift) ** 2).sum() / (ref_shift ** 2).sum()) < 1e-10


def test_operator_wraps_transform(rk, cuda):
    """test_shearlet.cpp:130-139."""
    p = rk.make_plan(32, 32, A5)
    op = rk.shearlet_operator(p)
    assert op.domain_shape == (32, 32) and op.range_shape == (59, 32, 32)
    x = dev(np.random.default_rng(9).standard_normal((2, 32, 32)).astype(np.float32), cuda)
    assert torch.equal(op.apply(x), rk.forward(p, x))
    assert torch.equal(op.adjoint(op.apply(x)), rk.backward(p, rk.forward(p, x)))
    assert rk.adjoint_check(op, 10, 0) < 1e-5


def test_batch_invariance_bitwise(rk, cuda):
    """Each image's coefficients do not depend on the rest of the batch (the
    analysis chunks over (image, coefficient) planes)."""
    p = rk.make_plan(64, 64, [0.5] * 4)
    x = dev(np.random.default_rng(10).standard_normal((7, 64, 64)).astype(np.float32), cuda)
    c = rk.forward(p, x)
    b = rk.backward(p, c)
    for e in (0, 3, 6):
        assert torch.equal(c[e:e + 1], rk.forward(p, x[e:e + 1]))
        assert torch.equal(b[e:e + 1], rk.backward(p, c[e:e + 1]))


def test_large_batch_chunking_512(rk, ref, cuda):
    """The analysis chunk boundary falls inside an image's coefficients at 512."""
    p = rk.make_plan(512, 512, A5)
    x = np.random.default_rng(11).standard_normal((3, 512, 512)).astype(np.float32)
    c = host(rk.forward(p, dev(x, cuda)))
    cr = ref.shearlet_forward(x[:1], A5)
    assert rel_l2(c[:1], cr) <= 1e-5
    xb = host(rk.backward(p, dev(c, cuda)))
    assert rel_l2(xb, x) <= 1e-5


def test_shape_validation(rk, cuda):
    """test_shearlet.cpp:151-157."""
    p = rk.make_plan(32, 32, A5)
    for bad in ((1, 16, 16), (32, 32)):
        with pytest.raises(rk.ValidationError):
            rk.forward(p, torch.zeros(*bad, device=cuda))
    for bad in ((1, 58, 32, 32), (1, 59, 16, 16)):
        with pytest.raises(rk.ValidationError):
            rk.backward(p, torch.zeros(*bad, device=cuda))
    with pytest.raises(rk.ValidationError, match="square"):
        rk.make_plan(48, 40, [0.5])


@pytest.mark.parametrize("n,alphas,batch", [(2, [0.5], 2), (3, [0.5], 1), (10, [0.5, 0.5], 3), (24, [0.0, 1.0], 2),
                                            (48, A5[:3], 2), (100, A5, 1)])
def test_non_power_of_two_grids_match_reference(rk, ref, cuda, n, alphas, batch):
    """Any square grid >= 2, as the reference's FFTW plans (shearlet.cpp:68-80): grids that
    are not a power of two run shearlet_generic.cu's DFT-matrix transforms; fp32 and fp64
    against the reference compiled in place, and the round trip."""
    rng = np.random.default_rng(n)
    p = rk.make_plan(n, n, alphas)
    for dt, tol in ((np.float32, 1e-5), (np.float64, 1e-12)):
        x = rng.standard_normal((batch, n, n)).astype(dt)
        c = host(rk.forward(p, dev(x, cuda)))
        cr = ref.shearlet_forward(x, alphas)
        assert c.shape == cr.shape and c.dtype == dt
        assert rel_l2(c, cr) <= tol, dt
        b = host(rk.backward(p, dev(cr, cuda)))
        assert rel_l2(b, ref.shearlet_backward(cr, alphas)) <= tol, dt
        assert rel_l2(host(rk.backward(p, dev(c, cuda))), x) <= (1e-5 if dt == np.float32 else 1e-12)
    xh = rng.standard_normal((batch, n, n)).astype(np.float16)
    ch = host(rk.forward(p, dev(xh, cuda)))
    assert rel_l2(ch.astype(np.float64), ref.shearlet_forward(xh, alphas).astype(np.float64)) <= 1e-3


def test_host_arrays_round_trip_through_device(rk, ref, cuda):
    x = np.random.default_rng(12).standard_normal((1, 32, 32)).astype(np.float32)
    p = rk.make_plan(32, 32, [0.5, 0.5])
    c = rk.forward(p, x)
    assert isinstance(c, np.ndarray) and c.dtype == np.float32
    assert rel_l2(c, ref.shearlet_forward(x, [0.5, 0.5])) <= 1e-5
