"""GPU parity of forward / backprojection against the reference oracle.

Restates the projector assertions of proj/tests/test_projector.cpp and
acceptance.cpp (criteria 4, 9) on the B200 kernels, plus oracle parity at
rel-L2 <= 1e-5 (fp32) / 1e-3 (fp16) as the north star requires.
"""
import numpy as np
import pytest
import torch

from oracle import Geom, batched_phantom, rel_l2

pytestmark = pytest.mark.gpu

TOL32 = 1e-5  # north star: fp32 storage vs the CPU reference
TOL16 = 1e-3  # north star: fp16 storage


def par(rk, s, na, det=None, spacing=None):
    return rk.make_parallel(s, rk.angles_linspace(0.0, np.pi, na), det, spacing)


def fan(rk, s, na, src, **kw):
    return rk.make_fanbeam(s, rk.angles_linspace(0.0, 2 * np.pi, na), src, **kw)


def ogeom(g, step=1.0):
    if hasattr(g, "source_distance"):
        return Geom("fanbeam", g.image_size, np.asarray(g.angles), g.det_count, g.det_spacing, g.source_distance,
                    g.det_distance, step)
    return Geom("parallel", g.image_size, np.asarray(g.angles), g.det_count, g.det_spacing, step=step)


def dev(a, cuda):
    return torch.from_numpy(np.ascontiguousarray(a)).to(cuda)


def host(t):
    return t.detach().cpu().numpy()


CASES = [
    ("par-32-45", lambda rk: par(rk, 32, 45)),
    ("par-64-90-det96", lambda rk: par(rk, 64, 90, 96)),
    ("par-100-33-det77-sp1.3", lambda rk: par(rk, 100, 33, 77, 1.3)),
    ("fan-32-24-D64", lambda rk: fan(rk, 32, 24, 64.0)),
    ("fan-64-90-D128", lambda rk: fan(rk, 64, 90, 128.0)),
    ("fan-80-40-D60-dd150-det101", lambda rk: fan(rk, 80, 40, 60.0, det_distance=150.0, det_count=101)),
]


@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
def test_parity_fp32(rk, oracle, cuda, name, mk):
    g = mk(rk)
    B = 5
    img = batched_phantom(oracle, g.image_size, B)
    img[2] = oracle.rng_uniform(2024, g.image_size ** 2).reshape(g.image_size, g.image_size)
    sino = rk.forward(g, dev(img, cuda))
    ref_sino = oracle.forward(ogeom(g), img)
    assert sino.dtype == torch.float32 and tuple(sino.shape) == ref_sino.shape
    assert rel_l2(host(sino), ref_sino) <= TOL32
    bp = rk.backprojection(g, dev(ref_sino, cuda))
    ref_bp = oracle.backprojection(ogeom(g), ref_sino)
    assert rel_l2(host(bp), ref_bp) <= TOL32


@pytest.mark.parametrize("name,mk", CASES[:4], ids=[c[0] for c in CASES[:4]])
def test_parity_fp16_and_fp64_storage(rk, oracle, cuda, name, mk):
    g = mk(rk)
    img = batched_phantom(oracle, g.image_size, 3)
    for dt, tol in ((np.float16, TOL16), (np.float64, TOL32)):
        x = img.astype(dt)
        sino = rk.forward(g, dev(x, cuda))
        assert host(sino).dtype == dt  # output keeps the input precision (test_projector.cpp:206-214)
        ref_sino = oracle.forward(ogeom(g), x)
        assert rel_l2(host(sino), ref_sino) <= tol
        bp = rk.backprojection(g, dev(ref_sino, cuda))
        assert rel_l2(host(bp), oracle.backprojection(ogeom(g), ref_sino)) <= tol


def test_config1_parity(rk, oracle, cuda):
    """parallel 256/256/256, batch 8, fp32; phantom batch and Rng(2024) uniform."""
    g = par(rk, 256, 256)
    for img in (batched_phantom(oracle, 256, 8),
                oracle.rng_uniform(2024, 8 * 256 * 256).reshape(8, 256, 256)):
        sino = rk.forward(g, dev(img, cuda))
        ref_sino = oracle.forward(ogeom(g), img)
        assert rel_l2(host(sino), ref_sino) <= TOL32
        bp = rk.backprojection(g, sino)
        ref_bp = oracle.backprojection(ogeom(g), ref_sino)
        assert rel_l2(host(bp), ref_bp) <= TOL32


def test_zero_maps_to_zero(rk, cuda):
    """test_projector.cpp:44-55."""
    for s in (8, 32):
        for g in (par(rk, s, 10), fan(rk, s, 10, 2.0 * s)):
            zi = torch.zeros(1, s, s, device=cuda)
            zs = torch.zeros(1, 10, s, device=cuda)
            assert float(rk.forward(g, zi).abs().sum()) == 0.0
            assert float(rk.backprojection(g, zs).abs().sum()) == 0.0


def test_axis_aligned_closed_forms(rk, oracle, cuda):
    """test_projector.cpp:135-164."""
    s = 16
    img = oracle.shepp_logan(s, np.float64)
    g = rk.make_parallel(s, [0.0])
    f = host(rk.forward(g, dev(img, cuda)))[0, 0]
    np.testing.assert_allclose(f, img[0].sum(axis=0), rtol=1e-6, atol=1e-6)
    delta = np.zeros((1, 1, s))
    delta[0, 0, 5] = 1.0
    bp = host(rk.backprojection(g, dev(delta, cuda)))[0]
    assert np.all(bp[:, 5] == 1.0) and np.all(np.delete(bp, 5, axis=1) == 0.0)
    gw = par(rk, 32, 90, 48)
    bp = host(rk.backprojection(gw, torch.ones(1, 90, 48, device=cuda)))
    np.testing.assert_allclose(bp, 90.0, rtol=1e-6)


def test_opposite_angles_reverse_detector(rk, oracle, cuda):
    """test_projector.cpp:166-181."""
    s, na, det = 64, 12, 80
    both = rk.angles_linspace(0.0, np.pi, na)
    both = both + [a + np.pi for a in both]
    g = rk.make_parallel(s, both, det)
    f = host(rk.forward(g, dev(oracle.shepp_logan(s), cuda)))[0]
    assert rel_l2(f[na:, ::-1], f[:na]) < 1e-5


def test_linearity(rk, oracle, cuda):
    """test_projector.cpp:183-194 at fp32 roundoff."""
    g = par(rk, 32, 20)
    a = oracle.rng_uniform(3, 32 * 32, True).reshape(1, 32, 32).astype(np.float64)
    b = oracle.rng_uniform(4, 32 * 32, True).reshape(1, 32, 32).astype(np.float64)
    lhs = host(rk.forward(g, dev(2.0 * a - 0.5 * b, cuda)))
    rhs = 2.0 * host(rk.forward(g, dev(a, cuda))) - 0.5 * host(rk.forward(g, dev(b, cuda)))
    assert rel_l2(lhs, rhs) < 1e-5


def test_fan_far_source_approaches_parallel(rk, oracle, cuda):
    """test_projector.cpp:196-204."""
    img = dev(oracle.shepp_logan(64), cuda)
    ang = rk.angles_linspace(0.0, np.pi, 48)
    fp = host(rk.forward(rk.make_parallel(64, ang), img))
    ff = host(rk.forward(rk.make_fanbeam(64, ang, 1e6), img))
    assert rel_l2(ff, fp) < 1e-3


def test_batched_equals_per_element_bitwise(rk, oracle, cuda):
    """test_projector.cpp:234-250 / acceptance.cpp:340-389 (C9)."""
    s, B = 32, 7
    imgs = dev(batched_phantom(oracle, s, B), cuda)
    for g in (par(rk, s, 24), fan(rk, s, 24, 64.0)):
        fb = rk.forward(g, imgs)
        bb = rk.backprojection(g, fb)
        for e in range(B):
            fe = rk.forward(g, imgs[e:e + 1])
            assert torch.equal(fb[e:e + 1], fe)
            assert torch.equal(bb[e:e + 1], rk.backprojection(g, fe))


@pytest.mark.parametrize("name,mk", [
    ("par-160-120", lambda rk: par(rk, 160, 120)),
    ("par-96-70-det131-sp0.8", lambda rk: par(rk, 96, 70, 131, 0.8)),
    ("fan-128-100-D200", lambda rk: fan(rk, 128, 100, 200.0)),
    ("fan-96-64-D70-fp64map", lambda rk: fan(rk, 96, 64, 70.0, det_distance=300.0)),
])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float16])
def test_single_lane_equals_packed_bitwise(rk, oracle, cuda, name, mk, dtype):
    """Batch 1 runs the single-lane kernels (kernels.cu, LANE); they must equal
    the packed kernels' lane results bit for bit (acceptance.cpp:340-389, C9)."""
    g = mk(rk)
    B = 6
    imgs = batched_phantom(oracle, g.image_size, B)
    imgs[3] = oracle.rng_uniform(7, g.image_size ** 2).reshape(g.image_size, g.image_size)
    x = dev(imgs, cuda).to(dtype)
    fb = rk.forward(g, x)
    bb = rk.backprojection(g, fb)
    for e in (0, 3, 5):
        fe = rk.forward(g, x[e:e + 1])
        assert torch.equal(fb[e:e + 1], fe)
        assert torch.equal(bb[e:e + 1], rk.backprojection(g, fe))


def test_quadrature_step(rk, oracle, cuda):
    """test_projector.cpp:268-279 + oracle parity at step 0.5."""
    img = oracle.shepp_logan(32, np.float64)
    g = par(rk, 32, 16)
    f1 = host(rk.forward(g, dev(img, cuda)))
    fh = host(rk.forward(g, dev(img, cuda), rk.ProjectorOptions(0.5)))
    rel = rel_l2(fh, f1)
    assert 0.0 < rel < 0.05
    assert rel_l2(fh, oracle.forward(ogeom(g, 0.5), img)) <= TOL32
    with pytest.raises(rk.ValidationError):
        rk.forward(g, dev(img, cuda), rk.ProjectorOptions(0.0))
    with pytest.raises(rk.ValidationError):
        rk.forward(g, dev(img, cuda), rk.ProjectorOptions(-1.0))


def test_shape_validation(rk, cuda):
    """test_projector.cpp:281-288."""
    g = par(rk, 32, 10)
    for bad in ((1, 16, 16), (32, 32)):
        with pytest.raises(rk.ValidationError):
            rk.forward(g, torch.zeros(*bad, device=cuda))
    for bad in ((1, 10, 16), (1, 5, 32), (10, 32)):
        with pytest.raises(rk.ValidationError):
            rk.backprojection(g, torch.zeros(*bad, device=cuda))


def test_host_path_matches_device_path(rk, oracle, cuda):
    """*_host entry points (reference-shaped host buffers, pipelined copies) == device entry points."""
    g = par(rk, 64, 40)
    img = batched_phantom(oracle, 64, 13)
    sd = host(rk.forward(g, dev(img, cuda)))
    sh = rk.forward(g, img)  # numpy in -> numpy out through rk_forward_host
    assert isinstance(sh, np.ndarray) and np.array_equal(sd, sh)
    pinned = torch.from_numpy(sh).pin_memory()
    bh = rk.backprojection(g, pinned)
    assert torch.equal(bh, rk.backprojection(g, dev(sh, cuda)).cpu())


@pytest.mark.parametrize("dtype", [np.float16, np.float64])
def test_host_path_matches_device_path_other_storage(rk, oracle, cuda, dtype):
    """fp16 (half8 texels, chunked host pipeline with partial groups) and fp64
    storage: host-buffer entry points == device entry points, bit for bit."""
    for g in (par(rk, 48, 36), fan(rk, 48, 30, 96.0)):
        img = batched_phantom(oracle, 48, 37).astype(dtype)
        sd = host(rk.forward(g, dev(img, cuda)))
        sh = rk.forward(g, img)
        assert sh.dtype == dtype and np.array_equal(sd, sh)
        assert np.array_equal(host(rk.backprojection(g, dev(sh, cuda))), rk.backprojection(g, sh))
        assert np.array_equal(host(rk.fbp(g, dev(sh, cuda))), rk.fbp(g, sh))


def test_half_accuracy_vs_single(rk, oracle, cuda):
    """acceptance.cpp:212-235 (C4) / test_projector.cpp:226-231: fp16 storage within 5e-4 of fp32."""
    g = par(rk, 256, 256)
    p = oracle.shepp_logan(256)
    fs = host(rk.forward(g, dev(p, cuda)))
    fh = host(rk.forward(g, dev(p.astype(np.float16), cuda)))
    assert rel_l2(fh, fs) <= 5e-4
    bs = host(rk.backprojection(g, dev(fs, cuda)))
    bh = host(rk.backprojection(g, dev(fs.astype(np.float16), cuda)))
    assert rel_l2(bh, bs) < 1e-3


def _random_geometry(rk, rs, fan):
    s = int(rs.choice([1, 2, 3, 5, 17, 40, 64, 97, 131, 160]))
    na = int(rs.integers(1, 40))
    nd = int(rs.integers(1, 3 * s + 8))
    sp = float(rs.uniform(0.3, 2.5))
    ang = list(rs.uniform(-7.0, 7.0, na))  # arbitrary, unsorted, beyond 2 pi (geometry.cpp:12-18)
    if not fan:
        return rk.make_parallel(s, ang, nd, sp)
    src = float(s) * float(rs.uniform(0.75, 4.0))
    return rk.make_fanbeam(s, ang, src, float(rs.uniform(0.5, 3.0)) * s, nd, sp)


@pytest.mark.parametrize("seed", range(24))
def test_random_geometry_parity(rk, oracle, cuda, seed):
    """Arbitrary angle lists, tiny and odd sizes, any detector count/spacing, fan distances, steps."""
    rs = np.random.default_rng(100 + seed)
    g = _random_geometry(rk, rs, fan=seed % 2 == 1)
    step = float(rs.choice([1.0, 0.5, 1.7]))
    B = int(rs.integers(1, 7))
    x = rs.standard_normal((B, g.image_size, g.image_size)).astype(np.float32)
    f = host(rk.forward(g, dev(x, cuda), rk.ProjectorOptions(step)))
    rf = oracle.forward(ogeom(g, step), x)
    if np.abs(rf).max() > 0:
        assert rel_l2(f, rf) <= TOL32, (g, step)
    else:
        assert np.abs(f).max() == 0
    y = rs.standard_normal((B, g.n_angles, g.det_count)).astype(np.float32)
    b = host(rk.backprojection(g, dev(y, cuda)))
    rb = oracle.backprojection(ogeom(g), y)
    if np.abs(rb).max() > 0:
        assert rel_l2(b, rb) <= TOL32, g
    else:
        assert np.abs(b).max() == 0


def test_half_overflow_is_unchecked_inf(rk, oracle, cuda):
    """Tensor::from_double_as narrows to half unchecked (tensor.cpp:121-122): overflow -> inf, like the reference."""
    g = par(rk, 64, 512)
    y = np.full((1, 512, 64), 200.0, np.float16)
    b = host(rk.backprojection(g, dev(y, cuda)))
    rb = oracle.backprojection(ogeom(g), y)
    assert np.array_equal(np.isinf(b), np.isinf(rb)) and np.isinf(b).any()
    fin = np.isfinite(rb)
    assert rel_l2(b[fin], rb[fin]) <= TOL16


def test_large_batch_shards_equal(rk, oracle, cuda):
    """Config-2 geometry: results are independent of how the batch is split (GPU-count invariance)."""
    g = par(rk, 512, 512)
    x = dev(batched_phantom(oracle, 512, 10), cuda)
    full = rk.forward(g, x)
    parts = torch.cat([rk.forward(g, x[:3]), rk.forward(g, x[3:8]), rk.forward(g, x[8:])])
    assert torch.equal(full, parts)
    bf = rk.backprojection(g, full)
    bp = torch.cat([rk.backprojection(g, full[:6]), rk.backprojection(g, full[6:])])
    assert torch.equal(bf, bp)


@pytest.mark.parametrize("name,mk", [("par", lambda rk: par(rk, 100, 37, 77, 1.3)),
                                     ("fan", lambda rk: fan(rk, 96, 40, 150.0)),
                                     ("fan-close", lambda rk: fan(rk, 64, 48, 50.0, det_distance=200.0))])
def test_small_batch_wide_backprojection_equals_batched_bitwise(rk, oracle, cuda, name, mk):
    """Batches of one packed group run the 512-thread backprojector (kernels.cu WIDE); per
    pixel it is the 256-thread kernel's arithmetic, so a 4-image call equals the first four
    images of a 12-image call bit for bit (and matches the oracle)."""
    g = mk(rk)
    rs = np.random.default_rng(11)
    y = rs.standard_normal((12, g.n_angles, g.det_count)).astype(np.float32)
    full = rk.backprojection(g, dev(y, cuda))
    small = rk.backprojection(g, dev(y[:4], cuda))
    assert torch.equal(small, full[:4])
    assert rel_l2(host(small), oracle.backprojection(ogeom(g), y[:4])) <= TOL32


def test_host_only_plan_teardown_leaves_no_cuda_error(rk, oracle, cuda):
    """A host-only plan / filter (device -1) destroyed in a process that then launches kernels:
    teardown must neither fail nor leave a sticky CUDA error for the next launch."""
    import gc

    import ctypes

    from paper_2009_14788_b200 import _lib
    from paper_2009_14788_b200.projector import Plan

    g = par(rk, 32, 20)
    hp = Plan(g, 1.0, -1)
    assert hp.info()["device"] == -1
    del hp
    gc.collect()
    fh = ctypes.c_void_p()
    _lib.check(_lib.lib.rk_filter_create(0, 32, -1, ctypes.byref(fh)))
    _lib.check(_lib.lib.rk_filter_destroy(fh))
    x = dev(batched_phantom(oracle, 32, 2), cuda)
    before = torch.cuda.current_device()
    sino = rk.forward(g, x)
    torch.cuda.synchronize()
    assert torch.cuda.current_device() == before
    assert rel_l2(host(sino), oracle.forward(ogeom(g), host(x))) <= TOL32


@pytest.mark.parametrize("kind", ["parallel", "fanbeam"])
def test_device_plan_from_cache_projects_bitwise_equal(rk, oracle, cuda, tmp_path, monkeypatch, kind):
    """A device plan whose forward schedule comes from the on-disk plan cache (plan_cache.cpp)
    launches exactly what a freshly planned one does: same digest, bit-identical sinograms."""
    from paper_2009_14788_b200.projector import Plan

    s = 96
    if kind == "parallel":
        g = rk.make_parallel(s, rk.angles_linspace(0.0, np.pi, 70))
    else:
        g = rk.make_fanbeam(s, rk.angles_linspace(0.0, 2 * np.pi, 70), 1.4 * s)
    x = dev(batched_phantom(oracle, s, 6), cuda)
    monkeypatch.setenv("RK_PLAN_CACHE", "off")
    fresh = Plan(g, 1.0, cuda.index or 0)
    h_fresh = fresh.prepare()
    monkeypatch.setenv("RK_PLAN_CACHE", str(tmp_path))
    Plan(g, 1.0, cuda.index or 0).prepare()  # plans and stores
    cached = Plan(g, 1.0, cuda.index or 0)
    assert cached.prepare() == h_fresh and cached.info()["schedule_from_cache"]
    import ctypes

    from paper_2009_14788_b200 import _lib

    outs = []
    for p in (fresh, cached):
        y = torch.empty(6, 70, g.det_count, device=cuda)
        _lib.check(_lib.lib.rk_forward(p.handle, _lib.RK_F32, ctypes.c_void_p(x.data_ptr()), 6,
                                       ctypes.c_void_p(y.data_ptr()), None))
        outs.append(y)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


_SHAPE_SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, {root!r})
import paper_2009_14788_b200 as rk
y = np.load({src!r})
out = {{}}
for name, g in [("par", rk.make_parallel(100, rk.angles_linspace(0.0, np.pi, 37), 77, 1.3)),
                ("par512", rk.make_parallel(64, rk.angles_linspace(0.0, np.pi, 64))),
                ("fan", rk.make_fanbeam(96, rk.angles_linspace(0.0, 2 * np.pi, 40), 150.0))]:
    yy = np.ascontiguousarray(y[:, :g.n_angles, :g.det_count])
    out[name] = rk.backprojection(g, torch.from_numpy(yy).cuda()).cpu().numpy()
np.savez({dst!r}, **out)
"""


def test_backprojector_thread_shapes_equal_bitwise(rk, oracle, cuda, tmp_path):
    """The 128-thread x 8-pixel backprojector (r2 default, kernels.cu NARROW) and the r1
    256 x 4 shape (RK_BP_NARROW=0) run the same per-pixel arithmetic: a 12-image batch
    (three packed groups) gives identical bits for parallel beam and the fan fp32 map."""
    import os
    import subprocess
    import sys

    rs = np.random.default_rng(5)
    y = rs.standard_normal((12, 64, 100)).astype(np.float32)
    src, res = str(tmp_path / "y.npy"), {}
    np.save(src, y)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for flag in ("1", "0"):
        dst = str(tmp_path / f"bp{flag}.npz")
        env = dict(os.environ, RK_BP_NARROW=flag)
        r = subprocess.run([sys.executable, "-c", _SHAPE_SCRIPT.format(root=root, src=src, dst=dst)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[flag] = np.load(dst)
    for name in ("par", "par512", "fan"):
        assert np.array_equal(res["1"][name], res["0"][name]), name
        assert np.isfinite(res["1"][name]).all()


_ORDER_SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, {root!r})
import paper_2009_14788_b200 as rk
x = np.load({src!r})
out = {{}}
for name, g in [("par", rk.make_parallel(96, rk.angles_linspace(0.0, np.pi, 70), 131, 0.8)),
                ("fan", rk.make_fanbeam(96, rk.angles_linspace(0.0, 2 * np.pi, 40), 150.0)),
                ("coarse", rk.make_fanbeam(128, rk.angles_linspace(0.0, 2 * np.pi, 40), 128.0, det_count=16))]:
    for dt in ("float32", "float16"):
        xx = torch.from_numpy(np.ascontiguousarray(x[:, :g.image_size, :g.image_size]).astype(dt)).cuda()
        out[name + dt] = rk.forward(g, xx).cpu().numpy()
np.savez({dst!r}, **out)
"""


def test_forward_launch_orders_equal_bitwise(rk, oracle, cuda, tmp_path):
    """The forward's CTA-major grid for few packed groups (kernels.cu launch_forward, CM) and
    the group-major grid (RK_FWD_CTA_MAJOR_GROUPS=0) run the same CTAs: 13 images (four
    float4 groups, two half8 groups), parallel / fan / narrow-warp schedules, identical bits."""
    import os
    import subprocess
    import sys

    src = str(tmp_path / "x.npy")
    np.save(src, np.random.default_rng(31).uniform(0.0, 1.0, (13, 128, 128)).astype(np.float32))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("8", "0"):
        dst = str(tmp_path / f"f{flag}.npz")
        env = dict(os.environ, RK_FWD_CTA_MAJOR_GROUPS=flag)
        script = _ORDER_SCRIPT.format(root=root, src=src, dst=dst)
        r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[flag] = np.load(dst)
    for k in res["8"].files:
        assert np.array_equal(res["8"][k], res["0"][k]), k


@pytest.mark.parametrize("name,mk", [
    ("fan-128-det16", lambda rk: fan(rk, 128, 40, 128.0, det_count=16)),      # spacing 16: narrow-warp tiers
    ("fan-96-det12", lambda rk: fan(rk, 96, 24, 96.0, det_count=12)),
    ("par-128-det10-sp14", lambda rk: par(rk, 128, 33, 10, 14.0)),
    ("par-160-det20-sp8", lambda rk: par(rk, 160, 50, 20, 8.0)),
    ("par-100-det35-one-angle", lambda rk: rk.make_parallel(100, [-2.8931329237874532], 35, 1.0)),
    # fine detectors: backprojection windows of hundreds of cells (kBpParHP, fp64 fan map)
    ("par-128-det1800-sp0.1", lambda rk: par(rk, 128, 30, 1800, 0.1)),
    ("par-96-det4096-sp0.03", lambda rk: par(rk, 96, 12, 4096, 0.03)),
    ("fan-128-det1200-sp0.25", lambda rk: fan(rk, 128, 24, 256.0, det_count=1200, det_spacing=0.25)),
])
@pytest.mark.parametrize("B", [1, 5])
def test_coarse_detector_and_narrow_detector_parity(rk, oracle, cuda, name, mk, B):
    """Detectors much coarser than the pixels (rays several pixels apart: the forward planner's
    narrow-warp tiers), detectors narrower than the image (the backprojection window must
    cover every tile row, plan.cpp) and much finer ones (kf spans hundreds of cells: the
    two-part parallel kernel, the fp64 fan map) — found by tools/stress_parity.py and
    tools/stress_extreme.py in r2."""
    g = mk(rk)
    rs = np.random.default_rng(17)
    x = rs.uniform(0.0, 1.0, (B, g.image_size, g.image_size)).astype(np.float32)
    f = host(rk.forward(g, dev(x, cuda)))
    assert rel_l2(f, oracle.forward(ogeom(g), x)) <= TOL32
    y = rs.standard_normal((B, g.n_angles, g.det_count)).astype(np.float32)
    b = host(rk.backprojection(g, dev(y, cuda)))
    assert rel_l2(b, oracle.backprojection(ogeom(g), y)) <= TOL32


@pytest.mark.parametrize("name,mk", [
    ("fan-128-det16", lambda rk: fan(rk, 128, 40, 128.0, det_count=16)),
    ("par-160-det20-sp8", lambda rk: par(rk, 160, 50, 20, 8.0)),
])
def test_coarse_detector_fp16_storage(rk, oracle, cuda, name, mk):
    """fp16 storage on narrow-warp schedules: batch 9 runs the half8 forward with the
    narrow-lane check compiled in (ForwardSchedule::any_narrow), batch 1 the single-lane
    kernel; both within the fp16 tolerance of the reference and each batched image
    bitwise equal to its single-image call (acceptance.cpp:340-389)."""
    g = mk(rk)
    rs = np.random.default_rng(23)
    x = rs.uniform(0.0, 1.0, (9, g.image_size, g.image_size)).astype(np.float16)
    f = host(rk.forward(g, dev(x, cuda)))
    assert f.dtype == np.float16
    assert rel_l2(f, oracle.forward(ogeom(g), x)) <= TOL16
    for i in (0, 4, 8):
        assert np.array_equal(host(rk.forward(g, dev(x[i:i + 1], cuda))), f[i:i + 1])
    y = rs.standard_normal((9, g.n_angles, g.det_count)).astype(np.float16)
    b = host(rk.backprojection(g, dev(y, cuda)))
    assert rel_l2(b, oracle.backprojection(ogeom(g), y)) <= TOL16
    assert np.array_equal(host(rk.backprojection(g, dev(y[3:4], cuda))), b[3:4])


def test_materialize_matrix(rk, oracle, cuda):
    """projector.cpp:276-294 / test_projector.cpp:57-110: the 2x2 single-angle matrix exactly,
    the dense matrix against the reference's forward columns and A x against forward(x), and
    the > 64 refusal."""
    A = rk.materialize_matrix(rk.make_parallel(2, [0.0]))
    assert A.shape == (2, 4) and A.dtype == np.float64
    assert np.array_equal(A, np.array([[1.0, 0.0, 1.0, 0.0], [0.0, 1.0, 0.0, 1.0]]))
    for g in (par(rk, 32, 45), fan(rk, 16, 24, 32.0)):
        M = rk.materialize_matrix(g)
        s = g.image_size
        units = np.eye(s * s).reshape(s * s, s, s)
        ref = oracle.forward(ogeom(g), units).reshape(s * s, -1).T
        assert rel_l2(M, ref) <= TOL32
        x = np.random.default_rng(7).uniform(-1.0, 1.0, (1, s, s))
        fx = np.asarray(rk.forward(g, x)).reshape(-1)
        assert rel_l2(M @ x.reshape(-1), fx) <= TOL32
    with pytest.raises(rk.ValidationError, match="refuses image_size 65"):
        rk.materialize_matrix(rk.make_parallel(65, [0.0]))


def test_very_large_batch(rk, oracle, cuda):
    """2,049 images of 512^2 (2 GB in, 64-bit indexing, 513 packed groups): the first and last
    elements match the reference and equal their single-image results bit for bit."""
    import subprocess
    import sys

    root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
    r = subprocess.run([sys.executable, __import__("os").path.join(root, "tools", "big_batch_probe.py"), "2049"],
                       capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_batch_beyond_one_launch(rk, oracle, cuda):
    """262,145 tiny images: more packed groups than one launch's grid.y / grid.z holds (65,535),
    so the device calls run consecutive sub-batches (capi.cpp for_sub_batches). Elements on both
    sides of the launch boundary equal their single-image results bit for bit and the reference;
    fp16 (half8 groups) too."""
    g = rk.make_parallel(4, [0.3, 1.1, 2.0], 5)
    B = 65535 * 4 + 5
    rs = np.random.default_rng(3)
    x = rs.uniform(0.0, 1.0, (B, 4, 4)).astype(np.float32)
    xd = dev(x, cuda)
    f = rk.forward(g, xd)
    b = rk.backprojection(g, f)
    fb = rk.fbp(g, f)
    fs = rk.filter_sinogram(f, rk.make_filter("ram-lak", g.det_count))
    torch.cuda.synchronize()
    idx = [0, 65535 * 4 - 1, 65535 * 4, B - 1]
    fh = host(f)
    assert rel_l2(fh[idx], oracle.forward(ogeom(g), x[idx])) <= TOL32
    for i in idx:
        f1 = rk.forward(g, xd[i:i + 1])
        assert torch.equal(f1, f[i:i + 1])
        assert torch.equal(rk.backprojection(g, f1), b[i:i + 1])
        assert torch.equal(rk.fbp(g, f1), fb[i:i + 1])
    xh = x.astype(np.float16)
    fh16 = rk.forward(g, dev(xh, cuda))
    for i in idx:
        assert torch.equal(rk.forward(g, dev(xh[i:i + 1], cuda)), fh16[i:i + 1])
    assert np.isfinite(host(fs)).all()
