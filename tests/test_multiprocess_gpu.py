"""Two processes, one B200: the sharded path end to end on real kernels.

Each rank projects only its contiguous shard of the batch through the C ABI
(forward + backprojection, no data-path collective), then `gather_batch`
reassembles the batch on rank 0; the result must equal the single-process run
bit for bit (batched == per-element, acceptance.cpp:340-389), and match the
reference.  Both ranks share cuda:0 (gpurun gives one GPU); NCCL refuses two
ranks on one device, so the gather runs over gloo through host memory — the
code path a multi-GPU box takes with NCCL differs only in the backend call.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, kind, B, out_path):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import paper_2009_14788_b200 as rk
    from paper_2009_14788_b200.phantom import shepp_logan
    from paper_2009_14788_b200.sharding import gather_batch, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = 96
    if kind == "parallel":
        g = rk.make_parallel(s, rk.angles_linspace(0.0, np.pi, 80))
    else:
        g = rk.make_fanbeam(s, rk.angles_linspace(0.0, 2 * np.pi, 80), 1.5 * s)
    lo, hi = shard_range(B, world, rank)
    ph = shepp_logan(s)
    x = torch.from_numpy(np.stack([ph * np.float32((e + 1) / B) for e in range(lo, hi)])).cuda()
    sino = rk.forward(g, x)
    bp = rk.backprojection(g, sino)
    torch.cuda.synchronize()
    full_sino = gather_batch(sino, B)
    full_bp = gather_batch(bp, B)
    if rank == 0:
        np.savez(out_path, sino=full_sino.cpu().numpy(), bp=full_bp.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["parallel", "fanbeam"])
def test_two_rank_shards_equal_single_process(rk, oracle, cuda, tmp_path, kind):
    import torch
    import torch.multiprocessing as mp

    from oracle import Geom, rel_l2
    from paper_2009_14788_b200.phantom import shepp_logan

    B = 11  # ragged: shards of 6 and 5 images (a partial packed group on each rank)
    out = str(tmp_path / "gathered.npz")
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, kind, B, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    got = np.load(out)

    s = 96
    if kind == "parallel":
        g = rk.make_parallel(s, rk.angles_linspace(0.0, np.pi, 80))
        og = Geom("parallel", s, np.asarray(g.angles))
    else:
        g = rk.make_fanbeam(s, rk.angles_linspace(0.0, 2 * np.pi, 80), 1.5 * s)
        og = Geom("fanbeam", s, np.asarray(g.angles), source_distance=1.5 * s)
    ph = shepp_logan(s)
    xs = np.stack([ph * np.float32((e + 1) / B) for e in range(B)])
    x = torch.from_numpy(xs).to(cuda)
    sino = rk.forward(g, x)
    bp = rk.backprojection(g, sino)
    assert np.array_equal(got["sino"], sino.cpu().numpy())
    assert np.array_equal(got["bp"], bp.cpu().numpy())
    ref = oracle.forward(og, xs)
    assert rel_l2(got["sino"], ref) <= 1e-5
