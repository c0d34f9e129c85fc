"""The reference's acceptance criteria that touch the path (proj/tests/acceptance.cpp),
restated on the B200 kernels: C1 (FBP MSE band, in test_filter_solvers_gpu), C2
(solver error ordering + dense-SVD prediction), C4 (half storage), C5 (adjoint,
gradient, matrix-vector agreement), C6 (fan defaults, parallel limit), C7
(power-iteration step size vs dense SVD), C9 (batch-32 bitwise)."""
import numpy as np
import pytest
import torch

from oracle import Geom, mse, rel_l2

pytestmark = pytest.mark.gpu


def dev(a, cuda):
    return torch.from_numpy(np.ascontiguousarray(a)).to(cuda)


def host(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def dense32(port):
    """materialize_matrix of parallel 32/45 (projector.cpp:276-294) via the oracle, and its SVD."""
    ang = port.angles_linspace(0.0, np.pi, 45)
    eye = np.eye(1024).reshape(1024, 32, 32)
    cols = port.forward(Geom("parallel", 32, ang), eye)  # (1024, 45, 32) double
    A = cols.reshape(1024, -1).T
    u, s, vt = np.linalg.svd(A, full_matrices=False)
    return A, s, vt


def test_c2_solver_ordering_128(rk, cuda):
    """acceptance.cpp:128-138: cgne < landweber < fbp in MSE at 128px, 100 iterations."""
    from paper_2009_14788_b200.phantom import shepp_logan

    g = rk.make_parallel(128, rk.angles_linspace(0.0, np.pi, 128), 185)
    op = rk.projector_operator(g)
    x = shepp_logan(128)[None]
    y = rk.forward(g, dev(x, cuda))
    m_fbp = mse(host(rk.fbp(g, y)), x)
    z = torch.zeros(1, 128, 128, device=cuda)
    alpha = 0.95 * rk.estimate_alpha(op, 20, 0)
    m_lw = mse(host(rk.landweber(op, y, z, alpha, 100)), x)
    m_cg = mse(host(rk.cgne(op, z, y, 100)), x)
    assert m_cg < m_lw < m_fbp


def test_c2_dense_svd_prediction_32(rk, cuda, dense32, port):
    """acceptance.cpp:140-163: Landweber/CGNE MSE at 32px vs the dense-SVD prediction."""
    A, sig, vt = dense32
    x = port.shepp_logan(32, np.float64)[0].ravel()
    c = vt @ x
    a32 = 0.95 * 2.0 / sig[0] ** 2
    pred = float(np.sum((1.0 - a32 * sig ** 2) ** (2 * 200) * c ** 2) / 1024.0)
    g = rk.make_parallel(32, rk.angles_linspace(0.0, np.pi, 45))
    op = rk.projector_operator(g)
    xt = dev(x.reshape(1, 32, 32).astype(np.float32), cuda)
    y = rk.forward(g, xt)
    z = torch.zeros_like(xt)
    m_lw = mse(host(rk.landweber(op, y, z, a32, 200)), x.reshape(1, 32, 32))
    m_cg = mse(host(rk.cgne(op, z, y, 200)), x.reshape(1, 32, 32))
    assert m_lw <= 1.15 * pred
    assert m_cg <= pred


def test_c4_half_storage(rk, cuda):
    """acceptance.cpp:212-235 with the 725-cell detector."""
    from paper_2009_14788_b200.phantom import shepp_logan

    xd = shepp_logan(512)[None].astype(np.float64)
    xh = xd.astype(np.float32).astype(np.float16)
    g = rk.make_parallel(512, rk.angles_linspace(0.0, np.pi, 512), 725)
    yd = host(rk.forward(g, dev(xd, cuda)))
    yh = host(rk.forward(g, dev(xh, cuda)))
    assert rel_l2(yh, yd) <= 5e-4
    xs = xd.astype(np.float32)
    ys = rk.forward(g, dev(xs, cuda))
    m_s = mse(host(rk.fbp(g, ys)), xs)
    m_h = mse(host(rk.fbp(g, dev(yh, cuda))).astype(np.float32), xs)
    assert abs(m_h - m_s) / m_s <= 0.01


def test_c5_matvec_agrees_with_dense_matrix(rk, cuda, dense32, port):
    """acceptance.cpp:262-272 / test_projector.cpp:75-110: forward == A x (here within fp32 rounding:
    the reference sums in double, the device in fp32)."""
    A, _, _ = dense32
    x = port.shepp_logan(32, np.float32)[0]
    g = rk.make_parallel(32, rk.angles_linspace(0.0, np.pi, 45))
    y = host(rk.forward(g, dev(x[None], cuda)))[0].ravel()
    ax = A @ x.astype(np.float64).ravel()
    assert rel_l2(y, ax) <= 1e-6


def test_c6_fan_defaults_and_parallel_limit(rk, cuda, port):
    f = rk.make_fanbeam(512, rk.angles_linspace(0.0, 2 * np.pi, 512), 512.0)
    assert f.det_distance == 512.0 and f.det_spacing == 2.0 and f.det_count == 512
    ang = rk.angles_linspace(0.0, np.pi, 64)
    x = dev(port.shepp_logan(64, np.float64), cuda)
    rel = rel_l2(host(rk.forward(rk.make_fanbeam(64, ang, 1e6), x)), host(rk.forward(rk.make_parallel(64, ang), x)))
    assert rel <= 1e-3


def test_c7_alpha_vs_dense_svd(rk, cuda, dense32):
    _, sig, _ = dense32
    oracle_alpha = 2.0 / sig[0] ** 2
    est = rk.estimate_alpha(rk.projector_operator(rk.make_parallel(32, rk.angles_linspace(0.0, np.pi, 45))), 20, 0)
    assert abs(est - oracle_alpha) / oracle_alpha <= 0.02


def test_c9_batch32_bitwise_and_limited_angles(rk, cuda, port):
    """acceptance.cpp:340-389: a batch of 32 random images equals 32 single runs bitwise, on a
    limited-angle geometry ([-50, 50) degrees, acceptance.cpp:65-69)."""
    ang = [(i * 100.0 / 64 - 50.0) * np.pi / 180.0 for i in range(64)]
    g = rk.make_parallel(64, ang)
    x = dev(port.rng_uniform(2024, 32 * 64 * 64).reshape(32, 64, 64), cuda)
    fb = rk.forward(g, x)
    bb = rk.backprojection(g, fb)
    for e in range(32):
        assert torch.equal(fb[e:e + 1], rk.forward(g, x[e:e + 1]))
        assert torch.equal(bb[e:e + 1], rk.backprojection(g, fb[e:e + 1]))
