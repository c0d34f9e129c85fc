"""Out-of-bounds checks without compute-sanitizer (which this GPU pool no
longer runs): every device entry point is called through the C ABI on input
and output regions that sit inside larger allocations whose guard bands are
filled with a sentinel.

* a write outside the output region changes the output guard band;
* a read outside the input region that reaches the result changes the result
  when the input guard band changes (two different sentinels, both compared
  bitwise with the plain call on a standalone tensor).

Covers the forward / backprojection kernels of both beam types (single-lane
batch 1, partial lane groups, the group-major launch order beyond 8 groups, the 512 tiers of configs 2 and 3), fp32 and fp16
storage, the ramp filter and the fused FBP.  Reference contract: outputs are
exactly (B, n_angles, det_count) / (B, s, s) (projector.cpp:228-274,
sino_filter.cpp:98-136).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

PAD = 4096  # elements of guard band on each side (keeps every region 16 B aligned)


def _geom(rk, kind, s, na, **kw):
    if kind == "par":
        return rk.make_parallel(s, rk.angles_linspace(0.0, np.pi, na), kw.get("det"))
    return rk.make_fanbeam(s, rk.angles_linspace(0.0, 2 * np.pi, na), kw["src"], det_count=kw.get("det"))


CASES = [
    ("par-37-29-det41", "par", 37, 29, {"det": 41}),
    ("par-64-90", "par", 64, 90, {}),
    ("fan-45-33-D80-det51", "fan", 45, 33, {"src": 80.0, "det": 51}),
    ("par-512-512", "par", 512, 512, {}),
    ("fan-512-512-D512", "fan", 512, 512, {"src": 512.0}),
]
SENT = {torch.float32: (1.0e6, -3.0e5), torch.float16: (6.0e4, -5.0e4)}


def _embedded(src, fill):
    """src copied into the middle of a flat buffer whose guard bands hold `fill`."""
    n = src.numel()
    buf = torch.full((n + 2 * PAD,), fill, dtype=src.dtype, device=src.device)
    view = buf[PAD:PAD + n].view(src.shape)
    view.copy_(src)
    return buf, view


def _out_region(shape, dtype, device, fill):
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * PAD,), fill, dtype=dtype, device=device)
    return buf, buf[PAD:PAD + n].view(shape)


def _call_guarded(call, x, out_shape):
    """Run call(x_view, out_view) for both sentinel pairs; return the outputs, checking the guard bands."""
    outs = []
    for fill_in, fill_out in (SENT[x.dtype], SENT[x.dtype][::-1]):
        _, xv = _embedded(x, fill_in)
        obuf, ov = _out_region(out_shape, x.dtype, x.device, fill_out)
        call(xv, ov)
        torch.cuda.synchronize()
        guard = torch.cat([obuf[:PAD], obuf[PAD + ov.numel():]])
        assert bool((guard == fill_out).all()), "write outside the output region"
        outs.append(ov.clone())
    return outs


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16], ids=["fp32", "fp16"])
@pytest.mark.parametrize("kind,s,na,kw", [c[1:] for c in CASES], ids=[c[0] for c in CASES])
def test_projectors_stay_in_bounds(rk, cuda, kind, s, na, kw, dtype):
    from paper_2009_14788_b200 import _lib
    from paper_2009_14788_b200._arrays import ptr, rk_dtype, stream_of
    from paper_2009_14788_b200.projector import get_plan

    g = _geom(rk, kind, s, na, **kw)
    plan = get_plan(g, None, cuda.index or 0)
    batches = (1, 3, 9) if s >= 512 else (1, 3, 8, 37)  # single-lane, partial group, > 8 packed groups
    gen = torch.Generator(device="cpu").manual_seed(s * 1000 + na)
    for B in batches:
        img = torch.rand((B, s, s), generator=gen).to(dtype).to(cuda)
        sino_shape = (B, g.n_angles, g.det_count)

        def fwd(xv, ov):
            _lib.check(_lib.lib.rk_forward(plan.handle, rk_dtype(xv), ptr(xv), B, ptr(ov), stream_of(xv)))

        want = rk.forward(g, img)
        for got in _call_guarded(fwd, img, sino_shape):
            assert torch.equal(got, want), f"forward B={B}: result depends on memory outside the image"

        sino = (want.float() / max(s, 1)).to(dtype)

        def bp(xv, ov):
            _lib.check(_lib.lib.rk_backproject(plan.handle, rk_dtype(xv), ptr(xv), B, ptr(ov), stream_of(xv)))

        want_bp = rk.backprojection(g, sino)
        for got in _call_guarded(bp, sino, (B, s, s)):
            assert torch.equal(got, want_bp), f"backprojection B={B}: result depends on memory outside the sinogram"


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16], ids=["fp32", "fp16"])
@pytest.mark.parametrize("s,na,det", [(40, 30, 57), (128, 96, 181), (512, 256, 1024)])
def test_filter_and_fbp_stay_in_bounds(rk, cuda, s, na, det, dtype):
    from paper_2009_14788_b200 import _lib
    from paper_2009_14788_b200._arrays import ptr, rk_dtype, stream_of
    from paper_2009_14788_b200.projector import get_plan
    from paper_2009_14788_b200.sino_filter import FilterKind, _device_filter, make_filter

    g = rk.make_parallel(s, rk.angles_linspace(0.0, np.pi, na), det)
    dev = cuda.index or 0
    plan = get_plan(g, None, dev)
    spec = make_filter(FilterKind.RamLak, det, dev)
    f = _device_filter(int(spec.kind), det, dev)
    gen = torch.Generator(device="cpu").manual_seed(det)
    for B in (1, 3):
        sino = torch.rand((B, na, det), generator=gen).to(dtype).to(cuda)

        def filt(xv, ov):
            _lib.check(_lib.lib.rk_filter_sinogram(f.handle, rk_dtype(xv), ptr(xv), B, na, ptr(ov), stream_of(xv)))

        want = rk.filter_sinogram(sino, spec)
        for got in _call_guarded(filt, sino, (B, na, det)):
            assert torch.equal(got, want), f"filter B={B}: result depends on memory outside the sinogram"

        def fbp(xv, ov):
            _lib.check(_lib.lib.rk_fbp(plan.handle, f.handle, rk_dtype(xv), ptr(xv), B, ptr(ov), stream_of(xv)))

        want_fbp = rk.fbp(g, sino)
        for got in _call_guarded(fbp, sino, (B, s, s)):
            assert torch.equal(got, want_fbp), f"fbp B={B}: result depends on memory outside the sinogram"
