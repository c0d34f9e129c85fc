"""Restates proj/tests/test_solvers.cpp and the operator cases of
test_linop.cpp that the projector-parity suites do not already cover: the
generic CG's exactness and freeze rules, its errors, CGNE's identity and
quality bars, the solvers' precision rules, and the identity / compose
operators.  CG state is fp32 (fp64 for double storage) with fp64 per-element
scalars, like the reference (solvers.cpp:47-107)."""
import numpy as np
import pytest
import torch

from oracle import mse
from paper_2009_14788_b200.phantom import shepp_logan

pytestmark = pytest.mark.gpu


def _phantom(rk, s, dtype=torch.float32, cuda="cuda"):
    return torch.from_numpy(shepp_logan(s)).reshape(1, s, s).to(cuda, dtype)


# ------------------------------------------------------------------ cg (test_solvers.cpp:134-210)
def test_cg_identity_solves_in_one_iteration(rk, cuda):
    b = _phantom(rk, 8, cuda=cuda)
    x = rk.cg(lambda v: v, torch.zeros_like(b), b, 1)
    assert torch.equal(x, b)


def test_cg_2x2_spd_exact_within_two_iterations(rk, cuda):
    M = torch.tensor([[4.0, 1.0], [1.0, 3.0]], dtype=torch.float64, device=cuda)
    b = torch.tensor([[1.0, 2.0]], dtype=torch.float64, device=cuda)
    x = rk.cg(lambda v: v @ M.T, torch.zeros_like(b), b, 2)
    assert x.dtype == torch.float64
    assert abs(float(x[0, 0]) - 1.0 / 11.0) <= 1e-10 * (1.0 / 11.0)
    assert abs(float(x[0, 1]) - 7.0 / 11.0) <= 1e-10 * (7.0 / 11.0)


def test_cg_negative_curvature_raises_with_iteration(rk, cuda):
    b = torch.ones(1, 4, device=cuda)
    with pytest.raises(rk.NotPositiveDefiniteError) as ei:
        rk.cg(lambda v: -v, torch.zeros_like(b), b, 5)
    assert ei.value.iteration == 0


def test_cg_exact_termination_on_small_spd(rk, cuda):
    n = 6
    L = np.zeros((n, n))
    for i in range(n):
        for j in range(i):
            L[i, j] = 0.3 * np.sin(1.0 + i + 2 * j)
        L[i, i] = 1.5 + 0.2 * i
    M = torch.from_numpy(L @ L.T).to(cuda)
    b = torch.tensor([[1.0, -2.0, 0.5, 3.0, -1.0, 0.25]], dtype=torch.float64, device=cuda)
    x = rk.cg(lambda v: v @ M.T, torch.zeros_like(b), b, 6)
    assert float(torch.linalg.norm(x @ M.T - b) / torch.linalg.norm(b)) < 1e-8


def test_cg_tolerance_zero_and_frozen_element(rk, cuda):
    b = torch.zeros(2, 4, device=cuda)
    b[0] = torch.arange(1.0, 5.0, device=cuda)
    x = rk.cg(lambda v: v, torch.zeros_like(b), b, 3)
    single = rk.cg(lambda v: v, torch.zeros(1, 4, device=cuda), b[:1], 3)
    assert torch.equal(x[:1], single)
    assert torch.equal(x[1], torch.zeros(4, device=cuda))


def test_cg_validation(rk, cuda):
    z4, z5 = torch.zeros(1, 4, device=cuda), torch.zeros(1, 5, device=cuda)
    for args in ((z4, z5, 2), (z4, z4, -1), (z4, z4, 2, -0.5)):
        with pytest.raises(rk.ValidationError):
            rk.cg(lambda v: v, *args)


def test_cg_error_a_norm_decreases_on_regularised_normal_equations(rk, cuda):
    """test_solvers.cpp:212-235 (fp64 storage; the operator computes in fp32)."""
    g = rk.make_parallel(32, rk.angles_linspace(0.0, np.pi, 45))
    op = rk.projector_operator(g)
    p0, p1 = 0.02, 0.1

    def apply(v):
        return p0 * op.adjoint(op.apply(v)) + (1.0 + p1) * v

    ph = _phantom(rk, 32, torch.float64, cuda)
    b = apply(ph)
    guess = torch.zeros_like(ph)
    prev, resid = float("inf"), 0.0
    for k in range(1, 9):
        xk = rk.cg(apply, guess, b, k)
        e = xk - ph
        enorm = float(torch.sqrt((e * apply(e)).sum()))
        assert enorm <= prev * (1.0 + 1e-9), k
        prev = enorm
        resid = float(torch.linalg.norm(apply(xk) - b))
    assert resid < 1e-2 * float(torch.linalg.norm(b))


# ------------------------------------------------------------------ cgne (test_solvers.cpp:237-265)
def test_cgne_identity_recovers_y(rk, cuda):
    y = torch.tensor([[1.0, -2.0, 3.0, -4.0, 5.0, -6.0, 7.0, -8.0]], device=cuda)
    assert torch.equal(rk.cgne(rk.identity_operator((8,)), torch.zeros_like(y), y, 1), y)


def test_cgne_quality_improves_with_iterations_at_64(rk, cuda):
    g = rk.make_parallel(64, rk.angles_linspace(0.0, np.pi, 90))
    op = rk.projector_operator(g)
    ph = _phantom(rk, 64, torch.float64, cuda)
    y = op.apply(ph)
    guess = torch.zeros_like(ph)
    ref = ph.cpu().numpy()
    m100 = mse(rk.cgne(op, guess, y, 100).cpu().numpy(), ref)
    m200 = mse(rk.cgne(op, guess, y, 200).cpu().numpy(), ref)
    assert m100 < 2e-3 and m200 < 1.2e-3 and m200 < m100


def test_solver_precision_rules(rk, cuda):
    """test_solvers.cpp:292-301: the output keeps the storage precision."""
    g = rk.make_parallel(16, rk.angles_linspace(0.0, np.pi, 12))
    op = rk.projector_operator(g)
    y = op.apply(_phantom(rk, 16, cuda=cuda))
    x_h = rk.landweber(op, y.half(), torch.zeros(1, 16, 16, device=cuda, dtype=torch.float16), 1e-3, 3)
    assert x_h.dtype == torch.float16
    x_d = rk.cgne(op, torch.zeros(1, 16, 16, device=cuda, dtype=torch.float64), y.double(), 3)
    assert x_d.dtype == torch.float64


# ------------------------------------------------------------------ operators (test_linop.cpp)
def test_identity_operator_is_exactly_self_adjoint(rk, cuda):
    op = rk.identity_operator((16, 16))
    assert tuple(op.domain_shape) == (16, 16) and tuple(op.range_shape) == (16, 16)
    x = _phantom(rk, 16, cuda=cuda)
    assert torch.equal(op.apply(x), x) and torch.equal(op.adjoint(x), x)
    assert rk.adjoint_check(op, 10, 0) < 1e-7
    assert rk.gradient_check(op, x, 1e-3) < 1e-5


def test_adjoint_check_is_deterministic_in_the_seed(rk, cuda):
    op = rk.projector_operator(rk.make_parallel(32, rk.angles_linspace(0.0, np.pi, 20)))
    assert rk.adjoint_check(op, 5, 3) == rk.adjoint_check(op, 5, 3)
    assert rk.adjoint_check(op, 10, 0) >= rk.adjoint_check(op, 1, 0)
    with pytest.raises(rk.ValidationError):
        rk.adjoint_check(op, 0, 0)


def test_compose_with_identity(rk, cuda):
    g = rk.make_parallel(32, rk.angles_linspace(0.0, np.pi, 20))
    p = rk.projector_operator(g)
    c = rk.compose(p, rk.identity_operator((32, 32)))
    assert tuple(c.domain_shape) == (32, 32) and tuple(c.range_shape) == tuple(p.range_shape)
    x = _phantom(rk, 32, cuda=cuda)
    assert torch.equal(c.apply(x), p.apply(x))
    dc, dp = rk.adjoint_check(c, 10, 0), rk.adjoint_check(p, 10, 0)
    assert abs(dc - dp) <= 1e-12 * dp
    with pytest.raises(rk.ValidationError):
        rk.compose(p, rk.identity_operator((16, 16)))
