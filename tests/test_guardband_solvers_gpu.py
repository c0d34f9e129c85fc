"""Guard-band out-of-bounds checks (see tests/test_guardband_gpu.py) for the
remaining device entry points: the fused Landweber and CGNE solvers
(solvers.cpp:130-166), the shearlet analysis / synthesis (shearlet.cpp:296-330,
radix-2 and DFT-matrix grids) and the fused ADMM (admm.cpp:111-163).  Each is
called through the C ABI on inputs and outputs embedded in sentinel-filled
buffers; the output guard must stay untouched and two sentinel pairs must give
results bitwise equal to the plain call.
"""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

PAD = 4096
SENT = {torch.float32: ((1.0e6, -3.0e5), (-2.0e5, 7.0e5)), torch.float16: ((6.0e4, -5.0e4), (-4.0e4, 3.0e4))}


def _guarded(call, inputs, out_shape, want):
    dt, dev = inputs[0].dtype, inputs[0].device
    n_out = int(np.prod(out_shape))
    for fill_in, fill_out in SENT[dt]:
        views = []
        for x in inputs:
            buf = torch.full((x.numel() + 2 * PAD,), fill_in, dtype=dt, device=dev)
            v = buf[PAD:PAD + x.numel()].view(x.shape)
            v.copy_(x)
            views.append(v)
        obuf = torch.full((n_out + 2 * PAD,), fill_out, dtype=dt, device=dev)
        ov = obuf[PAD:PAD + n_out].view(out_shape)
        call(*views, ov)
        torch.cuda.synchronize()
        assert bool((obuf[:PAD] == fill_out).all()) and bool((obuf[PAD + n_out:] == fill_out).all()), \
            "write outside the output region"
        assert torch.equal(ov, want), "result depends on memory outside the input regions (or cells left unwritten)"


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16], ids=["fp32", "fp16"])
@pytest.mark.parametrize("s,na", [(33, 40), (64, 64)])
def test_solvers_stay_in_bounds(rk, cuda, s, na, dtype):
    from paper_2009_14788_b200 import _lib
    from paper_2009_14788_b200._arrays import ptr, rk_dtype, stream_of
    from paper_2009_14788_b200.projector import get_plan

    g = rk.make_parallel(s, rk.angles_linspace(0.0, np.pi, na))
    op = rk.projector_operator(g)
    plan = get_plan(g, None, cuda.index or 0)
    B = 3
    gen = torch.Generator(device="cpu").manual_seed(s + na)
    x_true = torch.rand((B, s, s), generator=gen).to(cuda)
    y = rk.forward(g, x_true).to(dtype)
    guess = torch.zeros((B, s, s), dtype=dtype, device=cuda)
    alpha = 1.0 / (s * na)

    def lw(yv, gv, ov):
        failed = ctypes.c_int(-1)
        _lib.check(_lib.lib.rk_landweber(plan.handle, rk_dtype(gv), ptr(yv), ptr(gv), B, alpha, 4, ptr(ov),
                                         ctypes.byref(failed), stream_of(gv)), failed.value)

    _guarded(lw, [y, guess], (B, s, s), rk.landweber(op, y, guess, alpha, 4))

    def cg(yv, gv, ov):
        failed = ctypes.c_int(-1)
        _lib.check(_lib.lib.rk_cgne(plan.handle, rk_dtype(gv), ptr(yv), ptr(gv), B, 5, 0.0, ptr(ov),
                                    ctypes.byref(failed), stream_of(gv)), failed.value)

    _guarded(cg, [y, guess], (B, s, s), rk.cgne(op, guess, y, 5, 0.0))


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16], ids=["fp32", "fp16"])
@pytest.mark.parametrize("n,alphas", [(64, [0.5, 0.5, 1.0]), (48, [0.5, 1.0])])
def test_shearlets_stay_in_bounds(rk, cuda, n, alphas, dtype):
    from paper_2009_14788_b200 import _lib
    from paper_2009_14788_b200._arrays import ptr, rk_dtype, stream_of

    p = rk.make_plan(n, n, alphas)
    h = p._device_handle(cuda.index or 0)
    B = 3
    gen = torch.Generator(device="cpu").manual_seed(n)
    x = torch.randn((B, n, n), generator=gen).to(dtype).to(cuda)

    def fwd(xv, ov):
        _lib.check(_lib.lib.rk_shearlet_forward(h, rk_dtype(xv), ptr(xv), B, ptr(ov), stream_of(xv)))

    c = rk.forward(p, x)
    _guarded(fwd, [x], (B, p.n_coeff, n, n), c)

    def bwd(cv, ov):
        _lib.check(_lib.lib.rk_shearlet_backward(h, rk_dtype(cv), ptr(cv), B, ptr(ov), stream_of(cv)))

    _guarded(bwd, [c], (B, n, n), rk.backward(p, c))


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16], ids=["fp32", "fp16"])
def test_admm_stays_in_bounds(rk, cuda, dtype):
    from paper_2009_14788_b200 import _lib
    from paper_2009_14788_b200._arrays import ptr, rk_dtype, stream_of
    from paper_2009_14788_b200.projector import get_plan

    s, na, B = 32, 48, 2
    g = rk.make_parallel(s, rk.angles_linspace(0.0, np.pi, na))
    op = rk.projector_operator(g)
    plan = get_plan(g, None, cuda.index or 0)
    sp = rk.make_plan(s, s, [0.5, 0.5])
    sh = sp._device_handle(cuda.index or 0)
    gen = torch.Generator(device="cpu").manual_seed(7)
    y = rk.forward(g, torch.rand((B, s, s), generator=gen).to(cuda)).to(dtype)
    prm = rk.AdmmParams(outer_iterations=3, inner_cg_iterations=4)
    want = rk.admm_reconstruct(op, sp, y, prm)

    def admm(yv, ov):
        failed = ctypes.c_int64(-1)
        _lib.check(_lib.lib.rk_admm(plan.handle, sh, rk_dtype(yv), ptr(yv), B, prm.p0, prm.p1, None, 3, 4, ptr(ov),
                                    ctypes.byref(failed), stream_of(yv)), failed.value)

    _guarded(admm, [y], (B, s, s), want)
