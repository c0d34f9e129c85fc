"""CPU: the C-ABI library loads, exports every symbol include/*.h declares,
and the host-side logic (geometry defaults/validation, ray-table work counts,
the filter response) matches the reference without touching a GPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import Geom

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "radon_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(rk_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_abi():
    fns = declared_functions()
    for must in ("rk_plan_create", "rk_forward", "rk_backproject", "rk_filter_sinogram", "rk_fbp", "rk_forward_host",
                 "rk_landweber", "rk_cgne", "rk_estimate_alpha", "rk_last_error"):
        assert must in fns


def test_library_exports_every_declared_symbol(rk):
    from paper_2009_14788_b200 import _lib

    fns = declared_functions()
    for name in fns:
        assert hasattr(_lib.lib, name), name
    assert set(_lib.SIGNATURES) == set(fns)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(rk_\w+)\b", out))
    assert set(fns) <= exported


def test_library_is_sm100a(rk):
    from paper_2009_14788_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_geometry_defaults(rk):
    """test_geometry.cpp:10-59."""
    g = rk.make_parallel(512, rk.angles_linspace(0.0, np.pi, 512))
    assert (g.image_size, g.det_count, g.det_spacing, g.n_angles) == (512, 512, 1.0, 512)
    assert rk.make_parallel(512, [0.0], 725).det_count == 725
    assert rk.make_parallel(1, [0.0]).det_count == 1
    f = rk.make_fanbeam(512, rk.angles_linspace(0.0, 2 * np.pi, 512), 512.0)
    assert (f.det_distance, f.det_count, f.magnification(), f.det_spacing) == (512.0, 512, 2.0, 2.0)
    far = rk.make_fanbeam(512, [0.0], 10000.0)
    assert far.det_distance == 10000.0 and far.det_spacing == 2.0
    asym = rk.make_fanbeam(512, [0.0], 512.0, 1024.0)
    assert asym.magnification() == 3.0 and asym.det_spacing == 3.0
    assert rk.make_fanbeam(512, [0.0], 512.0, det_count=1024).det_spacing == 1.0
    assert rk.make_fanbeam(512, [0.0], 512.0, det_spacing=1.5).det_spacing == 1.5


@pytest.mark.parametrize("call", [
    lambda rk: rk.make_parallel(0, [0.0]), lambda rk: rk.make_parallel(-4, [0.0]), lambda rk: rk.make_parallel(8, []),
    lambda rk: rk.make_parallel(8, [0.0], 0), lambda rk: rk.make_parallel(8, [0.0], 8, 0.0),
    lambda rk: rk.make_parallel(8, [0.0], 8, -1.0), lambda rk: rk.make_parallel(8, [float("nan")]),
    lambda rk: rk.make_fanbeam(512, [0.0], 300.0), lambda rk: rk.make_fanbeam(512, [0.0], 0.0),
    lambda rk: rk.make_fanbeam(512, [0.0], -512.0), lambda rk: rk.make_fanbeam(0, [0.0], 512.0),
    lambda rk: rk.make_fanbeam(512, [], 512.0), lambda rk: rk.make_fanbeam(512, [0.0], 512.0, 0.0),
    lambda rk: rk.make_fanbeam(512, [0.0], 512.0, -1.0), lambda rk: rk.make_fanbeam(512, [0.0], 512.0, det_count=-3),
    lambda rk: rk.make_fanbeam(512, [0.0], 512.0, det_spacing=0.0), lambda rk: rk.angles_linspace(0.0, 1.0, 0),
    lambda rk: rk.filter_kind_from_name("butterworth"),
])
def test_validation_errors(rk, call):
    """test_geometry.cpp:26-33,61-73; test_sino_filter.cpp:77-90."""
    with pytest.raises(rk.ValidationError):
        call(rk)


def test_fan_source_boundary_accepted(rk):
    rk.make_fanbeam(512, [0.0], 400.0)


def test_angles_linspace_bitwise(rk):
    for (a, b, n) in ((0.0, np.pi, 7), (0.0, np.pi, 512), (-50.0, 50.0, 5), (0.0, 2 * np.pi, 1), (0.0, 100.0, 4)):
        assert rk.angles_linspace(a, b, n) == list(np.linspace(a, b, n, endpoint=False))


def test_filter_names(rk):
    for n in ("ram-lak", "shepp-logan", "cosine", "hamming", "hann"):
        assert rk.filter_kind_name(rk.filter_kind_from_name(n)) == n
    with pytest.raises(rk.ValidationError) as e:
        rk.filter_kind_from_name("butterworth")
    assert "ram-lak" in str(e.value)


def _host_plan(rk, g, step=1.0):
    from paper_2009_14788_b200 import _lib
    from paper_2009_14788_b200.geometry import to_c_geometry

    cg, keep = to_c_geometry(g, step)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib.rk_plan_create(ctypes.byref(cg), -1, ctypes.byref(h)))
    info = _lib.RkPlanInfo()
    _lib.check(_lib.lib.rk_plan_info_get(h, ctypes.byref(info)))
    _lib.check(_lib.lib.rk_plan_destroy(h))
    return info


def test_host_plan_work_counts_match_reference(rk, port):
    """The product's fp64 ray setup reproduces the reference's per-ray sample
    counts exactly (n = max(1, ceil(len/step)))."""
    cases = [rk.make_parallel(512, rk.angles_linspace(0.0, np.pi, 512)),
             rk.make_parallel(256, rk.angles_linspace(0.0, np.pi, 256)),
             rk.make_fanbeam(512, rk.angles_linspace(0.0, 2 * np.pi, 512), 512.0),
             rk.make_parallel(100, list(np.random.default_rng(1).uniform(-3, 3, 77)), 131, 0.83),
             rk.make_fanbeam(64, rk.angles_linspace(0.0, 2 * np.pi, 90), 50.0, 170.0, 97)]
    for g in cases:
        for step in (1.0, 0.37):
            info = _host_plan(rk, g, step)
            if hasattr(g, "source_distance"):
                og = Geom("fanbeam", g.image_size, np.asarray(g.angles), g.det_count, g.det_spacing,
                          g.source_distance, g.det_distance, step)
            else:
                og = Geom("parallel", g.image_size, np.asarray(g.angles), g.det_count, g.det_spacing, step=step)
            assert info.forward_samples == port.forward_samples(og)
            assert info.backproject_samples == g.image_size ** 2 * g.n_angles


def test_host_plan_rejects_bad_step(rk):
    with pytest.raises(rk.ValidationError):
        _host_plan(rk, rk.make_parallel(8, [0.0]), 0.0)


def test_filter_response_matches_reference(rk, port):
    """make_filter (sino_filter.cpp:64-92) of the product, built host-only: golden
    det-8 bins exactly, other sizes bit-equal to the restated reference."""
    from paper_2009_14788_b200 import _lib

    for kind in range(5):
        for nd in (2, 8, 95, 725, 1024, 1449):
            h = ctypes.c_void_p()
            _lib.check(_lib.lib.rk_filter_create(kind, nd, -1, ctypes.byref(h)))
            p = ctypes.c_int64()
            _lib.check(_lib.lib.rk_filter_response(h, ctypes.byref(p), None, None))
            rd = np.empty(p.value // 2 + 1)
            rf = np.empty(p.value // 2 + 1, np.float32)
            _lib.check(_lib.lib.rk_filter_response(h, ctypes.byref(p), rd.ctypes.data_as(ctypes.c_void_p),
                                                   rf.ctypes.data_as(ctypes.c_void_p)))
            _lib.check(_lib.lib.rk_filter_destroy(h))
            pp, od, of = port.make_filter(["ram-lak", "shepp-logan", "cosine", "hamming", "hann"][kind], nd)
            assert p.value == pp and np.array_equal(rd, od) and np.array_equal(rf, of)
    with pytest.raises(rk.ValidationError):
        h = ctypes.c_void_p()
        _lib.check(_lib.lib.rk_filter_create(0, 1, -1, ctypes.byref(h)))


def test_host_only_plan_refuses_kernels(rk):
    from paper_2009_14788_b200 import _lib
    from paper_2009_14788_b200.geometry import to_c_geometry

    cg, keep = to_c_geometry(rk.make_parallel(8, [0.0]))
    h = ctypes.c_void_p()
    _lib.check(_lib.lib.rk_plan_create(ctypes.byref(cg), -1, ctypes.byref(h)))
    buf = np.zeros(64, np.float32)
    p = buf.ctypes.data_as(ctypes.c_void_p)
    st = _lib.lib.rk_forward(h, _lib.RK_F32, p, 1, p, None)
    assert st == _lib.RK_ERR_VALIDATION and b"host-only" in _lib.lib.rk_last_error()
    _lib.check(_lib.lib.rk_plan_destroy(h))


def test_plan_cache_is_lru(rk):
    """get_plan keeps the most recently used plans (host-only plans here) and evicts the oldest."""
    import math

    from paper_2009_14788_b200 import projector as P

    old = P._MAX_PLANS
    try:
        P._MAX_PLANS = 3
        P._PLANS.clear()
        gs = [rk.make_parallel(16 + i, rk.angles_linspace(0.0, math.pi, 8)) for i in range(4)]
        a = rk.get_plan(gs[0], None, -1)
        rk.get_plan(gs[1], None, -1)
        assert rk.get_plan(gs[0], None, -1) is a  # hit refreshes gs[0]
        rk.get_plan(gs[2], None, -1)
        rk.get_plan(gs[3], None, -1)  # evicts gs[1], the least recently used
        assert [k[0].image_size for k in P._PLANS] == [16, 18, 19]
        assert rk.get_plan(gs[0], None, -1) is a
    finally:
        P._MAX_PLANS = old
        P._PLANS.clear()


def test_set_num_threads_contract():
    """threading.cpp:24-32: n >= 1 is kept, n < 1 is a ValidationError, the default is the
    hardware count (here: the forward planner's host threads)."""
    import os

    import paper_2009_14788_b200 as rk

    saved = os.environ.pop("RK_PLAN_THREADS", None)
    try:
        assert rk.num_threads() == (os.cpu_count() or 1)
        rk.set_num_threads(3)
        assert rk.num_threads() == 3
        with pytest.raises(rk.ValidationError, match="thread count must be >= 1, got 0"):
            rk.set_num_threads(0)
    finally:
        os.environ.pop("RK_PLAN_THREADS", None)
        if saved is not None:
            os.environ["RK_PLAN_THREADS"] = saved
