"""Concurrent callers (threading row): the reference's projector
functions are pure and safe to call from many threads (threading.hpp:12-15);
here several host threads share plans and issue calls on their own CUDA
streams, or through the synchronous host-buffer entry points, and every
result must equal the serial result bit for bit."""
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _geoms(rk):
    # plans of different sizes need different dynamic shared memory for the same
    # kernels: the per-function cap must never be lowered under another thread
    return [rk.make_parallel(96, rk.angles_linspace(0.0, np.pi, 72)),
            rk.make_fanbeam(96, rk.angles_linspace(0.0, 2 * np.pi, 64), 150.0),
            rk.make_parallel(256, rk.angles_linspace(0.0, np.pi, 48)),
            rk.make_fanbeam(200, rk.angles_linspace(0.0, 2 * np.pi, 40), 300.0)]


def _run_threads(fn, n):
    errs = []

    def wrap(i):
        try:
            fn(i)
        except BaseException as e:  # noqa: BLE001 (re-raised below)
            errs.append(e)

    ts = [threading.Thread(target=wrap, args=(i,)) for i in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


def test_threads_on_own_streams_match_serial(rk, cuda):
    gs = _geoms(rk)
    rs = np.random.default_rng(5)
    xs = [torch.from_numpy(rs.standard_normal((6, g.image_size, g.image_size)).astype(np.float32)).to(cuda)
          for g in gs for _ in range(3)]
    ref = []
    for i, x in enumerate(xs):
        g = gs[i // 3]
        s = rk.forward(g, x)
        ref.append((s, rk.backprojection(g, s), rk.fbp(g, s)))
    torch.cuda.synchronize()
    got = [None] * len(xs)

    def work(i):
        st = torch.cuda.Stream(device=cuda)
        with torch.cuda.stream(st):
            for _ in range(4):
                g = gs[i // 3]
                s = rk.forward(g, xs[i])
                got[i] = (s, rk.backprojection(g, s), rk.fbp(g, s))
        st.synchronize()

    _run_threads(work, len(xs))
    for a, b in zip(ref, got):
        for u, v in zip(a, b):
            assert torch.equal(u, v)


def test_threads_on_host_buffers_match_serial(rk, cuda):
    gs = _geoms(rk)
    rs = np.random.default_rng(6)
    xs = [rs.standard_normal((5, 96, 96)).astype(np.float32) for _ in range(6)]
    ref = []
    for i, x in enumerate(xs):
        s = rk.forward(gs[i % 2], x)
        ref.append((s, rk.backprojection(gs[i % 2], s)))
    got = [None] * len(xs)

    def work(i):
        for _ in range(2):
            s = rk.forward(gs[i % 2], xs[i])
            got[i] = (s, rk.backprojection(gs[i % 2], s))

    _run_threads(work, len(xs))
    for a, b in zip(ref, got):
        for u, v in zip(a, b):
            assert np.array_equal(np.asarray(u), np.asarray(v))


@pytest.mark.parametrize("n", [128, 96])  # radix-2 passes / DFT-matrix passes (any other grid)
def test_shearlet_plan_shared_across_streams(rk, cuda, n):
    """One shearlet plan, several threads on their own streams: the plan's spectra scratch
    is ordered across streams by its event (capi.cpp ShearletLease), so concurrent analysis /
    synthesis calls of different batch sizes equal the serial results bit for bit."""
    p = rk.make_plan(n, n, [0.5, 0.5, 0.5])
    rs = np.random.default_rng(n)
    xs = [torch.from_numpy(rs.standard_normal((b, n, n)).astype(np.float32)).to(cuda) for b in (1, 3, 2, 4, 1, 2)]
    ref = []
    for x in xs:
        c = rk.forward(p, x)
        ref.append((c, rk.backward(p, c)))
    torch.cuda.synchronize()
    got = [None] * len(xs)

    def work(i):
        st = torch.cuda.Stream(device=cuda)
        with torch.cuda.stream(st):
            for _ in range(3):
                c = rk.forward(p, xs[i])
                got[i] = (c, rk.backward(p, c))
        st.synchronize()

    _run_threads(work, len(xs))
    torch.cuda.synchronize()
    for (c, b), (rc, rb) in zip(got, ref):
        assert torch.equal(c, rc) and torch.equal(b, rb)
