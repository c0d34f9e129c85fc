"""GPU l1-shearlet ADMM (csrc/admm.cu) against the reference's
admm_reconstruct compiled in place (oracle/_ref), and the cases of
proj/tests/test_admm.cpp (shrink, weights, objective, zero sinogram,
limited-angle quality + monotone objective, zero weights, divergence, zero
iterations, batch invariance, half storage, validation)."""
import math

import numpy as np
import pytest
import torch

from oracle import Geom, mse, rel_l2

pytestmark = pytest.mark.gpu


def dev(a, cuda):
    return torch.from_numpy(np.ascontiguousarray(a)).to(cuda)


def host(t):
    return t.detach().cpu().numpy()


def limited_angles(n):
    """test_admm.cpp:18-23: a 100 degree arc centred on the vertical axis."""
    return [(i * 100.0 / n - 50.0) * math.pi / 180.0 for i in range(n)]


def phantom(port, s, dtype=np.float64):
    return port.shepp_logan(s, dtype)


@pytest.mark.parametrize("s,na,alphas,outer,inner,batch", [
    (32, 32, [0.5, 0.5, 0.5], 6, 20, 1),
    (64, 48, [0.5, 0.5], 4, 15, 3),
])
def test_fused_admm_matches_reference_f32(rk, ref, port, cuda, s, na, alphas, outer, inner, batch):
    """The fused device loop against the reference's float path on the same
    sinogram.  Tolerance: the two runs differ by fp32 rounding in the projector
    sums and the FFTs (each 1e-6 relative), carried through outer x inner CG
    steps of an ill-conditioned limited-angle problem."""
    ang = limited_angles(na)
    g = rk.make_parallel(s, ang)
    x = np.concatenate([phantom(port, s) * (1.0 - 0.25 * e) for e in range(batch)]).astype(np.float32)
    y = host(rk.forward(g, dev(x, cuda)))
    p = rk.AdmmParams(outer_iterations=outer, inner_cg_iterations=inner)
    rec = host(rk.admm_reconstruct(rk.projector_operator(g), rk.make_plan(s, s, alphas), dev(y, cuda), p))
    rref = ref.admm(Geom("parallel", s, np.asarray(ang)), y, alphas, p.p0, p.p1, outer, inner)
    assert rec.dtype == np.float32
    assert rel_l2(rec, rref) <= 2e-4


def test_fused_and_composed_paths_agree(rk, port, cuda):
    """The fused C loop and the recurrence composed from apply/adjoint + cg
    (used for generic operators) compute the same thing."""
    s = 32
    g = rk.make_parallel(s, limited_angles(24))
    op = rk.projector_operator(g)
    y = rk.forward(g, dev(phantom(port, s, np.float32), cuda))
    plan = rk.make_plan(s, s, [0.5, 0.5])
    p = rk.AdmmParams(outer_iterations=3, inner_cg_iterations=10)
    fused = host(rk.admm_reconstruct(op, plan, y, p))
    generic = rk.LinearOperator(op.domain_shape, op.range_shape, op.apply, op.adjoint)
    composed = host(rk.admm_reconstruct(generic, plan, y, p))
    assert rel_l2(fused, composed) <= 1e-4


def test_shrink_hand_values(rk, cuda):
    """test_admm.cpp:27-41."""
    a = dev(np.array([3.0, 0.5, -0.5, 1.2, -4.0]), cuda)
    s = host(rk.shrink(a, 1.0))
    assert s[0] == pytest.approx(2.0, rel=1e-14) and s[1] == 0.0 and s[2] == 0.0
    assert s[3] == pytest.approx(0.2, rel=1e-12) and s[4] == pytest.approx(-3.0, rel=1e-14)
    assert torch.equal(rk.shrink(a, 0.0), a)
    with pytest.raises(rk.ValidationError):
        rk.shrink(a, -0.1)


def test_shrink_broadcast(rk, cuda):
    """test_admm.cpp:43-77."""
    rng = np.random.default_rng(0)
    a = rng.standard_normal((2, 3, 4, 5))
    b = np.abs(rng.standard_normal((1, 3, 1, 1)))
    s = host(rk.shrink(dev(a, cuda), dev(b, cuda)))
    want = np.sign(a) * np.maximum(np.abs(a) - b, 0.0)
    assert np.allclose(s, want, rtol=1e-14, atol=0)
    assert torch.equal(rk.shrink(dev(a, cuda), dev(np.zeros((1, 3, 1, 1)), cuda)), dev(a, cuda))
    for bad in (np.ones((1, 2, 1, 1)), np.ones((3, 1, 1))):
        with pytest.raises(rk.ValidationError):
            rk.shrink(dev(a, cuda), dev(bad, cuda))
    with pytest.raises(rk.ValidationError):
        rk.shrink(dev(a, cuda), dev(-np.ones((1, 3, 1, 1)), cuda))


def test_default_weights(rk):
    """test_admm.cpp:79-87."""
    plan = rk.make_plan(32, 32, [0.5] * 3, device=-1)
    w = rk.default_weights(plan)
    assert w.dtype == np.float64 and w.shape == (1, plan.n_coeff, 1, 1)
    for k in range(plan.n_coeff):
        assert w.reshape(-1)[k] == 3.0 ** plan.scales[k] / 400.0
    assert w.reshape(-1)[0] == 0.0025


def test_objective_definition(rk, port, cuda):
    """test_admm.cpp:89-127."""
    s = 32
    g = rk.make_parallel(s, limited_angles(32))
    op = rk.projector_operator(g)
    plan = rk.make_plan(s, s, [0.5] * 3)
    f0 = torch.zeros(1, s, s, dtype=torch.float64, device=cuda)
    y0 = rk.forward(g, f0)
    assert rk.admm_objective(op, plan, f0, y0) == 0.0
    f = dev(phantom(port, s), cuda)
    y = rk.forward(g, f) * 0.9
    w0 = np.zeros((1, plan.n_coeff, 1, 1))
    r = host(rk.forward(g, f)) - host(y)
    assert rk.admm_objective(op, plan, f, y, w0) == pytest.approx(0.5 * (r * r).sum(), rel=1e-12)
    sh = host(rk.forward(plan, f))
    want = float(np.abs(rk.default_weights(plan) * sh).sum()) + 0.5 * (r * r).sum()
    assert rk.admm_objective(op, plan, f, y) == pytest.approx(want, rel=1e-12)
    with pytest.raises(rk.ValidationError):
        rk.admm_objective(op, plan, f, y[:, :5])


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_zero_sinogram_exact_zeros(rk, cuda, dtype):
    """test_admm.cpp:129-139."""
    s = 16
    g = rk.make_parallel(s, limited_angles(16))
    rec = rk.admm_reconstruct(rk.projector_operator(g), rk.make_plan(s, s, [0.5, 0.5]),
                              torch.zeros(1, 16, s, dtype=dtype, device=cuda), rk.AdmmParams(outer_iterations=6))
    assert rec.dtype == dtype and torch.equal(rec, torch.zeros(1, s, s, dtype=dtype, device=cuda))


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_limited_angle_beats_fbp_monotone_objective(rk, port, cuda, dtype):
    """test_admm.cpp:141-180 (reference measured 1.19e-2 vs fbp 2.24e-2)."""
    s = 32
    g = rk.make_parallel(s, limited_angles(32))
    op = rk.projector_operator(g)
    plan = rk.make_plan(s, s, [0.5] * 3)
    x = dev(phantom(port, s), cuda).to(dtype)
    y = rk.forward(g, x)
    fbp_mse = mse(host(rk.fbp(g, y)), host(x))
    objs, its, min_z2 = [], [], [0.0]

    def obs(it, st):
        its.append(it)
        objs.append(rk.admm_objective(op, plan, st.f, y))
        min_z2[0] = min(min_z2[0], float(st.z2.min()))
        assert tuple(st.f.shape) == (1, s, s) and tuple(st.z1.shape) == (1, plan.n_coeff, s, s)

    rec = rk.admm_reconstruct(op, plan, y, rk.AdmmParams(outer_iterations=20), obs)
    admm_mse = mse(host(rec), host(x))
    assert admm_mse < 1.5e-2 and admm_mse < fbp_mse
    assert its == list(range(20))
    assert min_z2[0] == 0.0
    for i in range(1, len(objs)):
        assert objs[i] <= objs[i - 1] * 1.01
    assert objs[-1] < objs[0]


def test_zero_weights_fit_tighter(rk, port, cuda):
    """test_admm.cpp:182-202."""
    s = 32
    g = rk.make_parallel(s, limited_angles(32))
    op = rk.projector_operator(g)
    plan = rk.make_plan(s, s, [0.5] * 3)
    y = rk.forward(g, dev(phantom(port, s, np.float32), cuda))
    rec_def = rk.admm_reconstruct(op, plan, y, rk.AdmmParams(outer_iterations=20))
    w0 = np.zeros((1, plan.n_coeff, 1, 1))
    rec0 = rk.admm_reconstruct(op, plan, y, rk.AdmmParams(outer_iterations=20, weights=w0))
    assert rk.admm_objective(op, plan, rec0, y, w0) < rk.admm_objective(op, plan, rec_def, y, w0)


def test_runaway_penalty_diverges_at_iteration_0(rk, port, cuda):
    """test_admm.cpp:204-219."""
    s = 32
    g = rk.make_parallel(s, limited_angles(16))
    y = rk.forward(g, dev(phantom(port, s, np.float32), cuda))
    with pytest.raises(rk.DivergenceError) as e:
        rk.admm_reconstruct(rk.projector_operator(g), rk.make_plan(s, s, [0.5, 0.5]), y,
                            rk.AdmmParams(outer_iterations=5, p0=1e30))
    assert e.value.iteration == 0


def test_zero_outer_iterations(rk, port, cuda):
    """test_admm.cpp:221-234."""
    s = 16
    g = rk.make_parallel(s, limited_angles(12))
    y = rk.forward(g, dev(phantom(port, s, np.float32), cuda))
    calls = []
    rec = rk.admm_reconstruct(rk.projector_operator(g), rk.make_plan(s, s, [0.5]), y,
                              rk.AdmmParams(outer_iterations=0), lambda it, st: calls.append(it))
    assert torch.equal(rec, torch.zeros_like(rec)) and calls == []


def test_batched_bitwise_equals_single_runs(rk, port, cuda):
    """test_admm.cpp:236-258 (the fused path: per-element CG scalars, fixed reductions)."""
    s = 16
    g = rk.make_parallel(s, limited_angles(16))
    op = rk.projector_operator(g)
    plan = rk.make_plan(s, s, [0.5, 0.5])
    x = dev(phantom(port, s, np.float32), cuda)
    ys = [rk.forward(g, x * c) for c in (1.0, 0.5, 0.25, 0.8, 1.3)]
    p = rk.AdmmParams(outer_iterations=4)
    rb = rk.admm_reconstruct(op, plan, torch.cat(ys), p)
    for e, y in enumerate(ys):
        assert torch.equal(rb[e:e + 1], rk.admm_reconstruct(op, plan, y, p))


def test_half_sinogram(rk, port, cuda):
    """test_admm.cpp:260-271."""
    s = 16
    g = rk.make_parallel(s, limited_angles(12))
    y = rk.forward(g, dev(phantom(port, s, np.float32), cuda)).half()
    rec = rk.admm_reconstruct(rk.projector_operator(g), rk.make_plan(s, s, [0.5]), y,
                              rk.AdmmParams(outer_iterations=2))
    assert rec.dtype == torch.float16 and tuple(rec.shape) == (1, s, s)
    r32 = rk.admm_reconstruct(rk.projector_operator(g), rk.make_plan(s, s, [0.5]), y.float(),
                              rk.AdmmParams(outer_iterations=2))
    assert torch.equal(rec, r32.half())


def test_parameter_validation(rk, cuda):
    """test_admm.cpp:273-314."""
    s = 16
    g = rk.make_parallel(s, limited_angles(12))
    op = rk.projector_operator(g)
    plan = rk.make_plan(s, s, [0.5])
    y = torch.zeros(1, 12, s, device=cuda)
    for kw in ({"p0": 0.0}, {"p1": -1.0}, {"outer_iterations": -1}, {"inner_cg_iterations": 0},
               {"weights": np.ones(plan.n_coeff + 1)}):
        with pytest.raises(rk.ValidationError):
            rk.admm_reconstruct(op, plan, y, rk.AdmmParams(**kw))
    with pytest.raises(rk.ValidationError):
        rk.admm_reconstruct(op, plan, torch.zeros(1, 11, s, device=cuda))
    with pytest.raises(rk.ValidationError, match="does not match plan grid"):
        rk.admm_reconstruct(op, rk.make_plan(8, 8, [0.5]), y)


def test_graph_replay_equals_direct_launches(rk, port, cuda, monkeypatch):
    """admm.cu replays one captured outer iteration as a CUDA graph (RK_ADMM_GRAPH, default on):
    the same kernels with the same arguments, so the result is bit-identical to direct launches —
    for a one-shot run, for an observer stepping one iteration per call (capture after the first,
    replays after), and when a divergence must still name its outer iteration."""
    s = 32
    g = rk.make_parallel(s, limited_angles(24))
    op = rk.projector_operator(g)
    y = rk.forward(g, dev(phantom(port, s, np.float32), cuda))
    plan = rk.make_plan(s, s, [0.5, 0.5])
    p = rk.AdmmParams(outer_iterations=6, inner_cg_iterations=12)
    seen = {}
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("RK_ADMM_GRAPH", mode)
        out[mode] = host(rk.admm_reconstruct(op, plan, y, p))
        its = []
        seen[mode] = host(rk.admm_reconstruct(op, plan, y, p, lambda it, st: its.append(it)))
        assert its == list(range(6))
    assert np.array_equal(out["1"], out["0"])
    assert np.array_equal(seen["1"], seen["0"]) and np.array_equal(seen["1"], out["0"])
    monkeypatch.setenv("RK_ADMM_GRAPH", "1")
    with pytest.raises(rk.DivergenceError) as e:
        rk.admm_reconstruct(op, plan, y, rk.AdmmParams(outer_iterations=5, p0=1e30))
    assert e.value.iteration == 0


def test_repeated_calls_reuse_state_bitwise(rk, port, cuda):
    """A finished ADMM's buffers and captured graph are kept for the next compatible call
    (capi.cpp admm_take_idle): repeated calls, interleaved with an incompatible one (other
    penalties) and a different batch, return bit-identical results; a shearlet plan freed
    while a state built on it is idle does not leave a dangling state behind."""
    import gc

    s, na = 32, 24
    g = rk.make_parallel(s, limited_angles(na))
    op = rk.projector_operator(g)
    y = rk.forward(g, dev(np.concatenate([phantom(port, s, np.float32)] * 3), cuda))
    plan = rk.make_plan(s, s, [0.5, 0.5])
    prm = rk.AdmmParams(p0=0.5, p1=0.1, outer_iterations=4, inner_cg_iterations=5)
    first = rk.admm_reconstruct(op, plan, y, prm)
    other = rk.admm_reconstruct(op, plan, y, rk.AdmmParams(p0=0.7, p1=0.1, outer_iterations=4, inner_cg_iterations=5))
    single = rk.admm_reconstruct(op, plan, y[:1], prm)
    again = rk.admm_reconstruct(op, plan, y, prm)
    assert torch.equal(first, again)
    assert torch.equal(single[0], first[0])
    assert not torch.equal(other, first)
    del plan
    gc.collect()
    plan2 = rk.make_plan(s, s, [0.5, 0.5])
    assert torch.equal(rk.admm_reconstruct(op, plan2, y, prm), first)
