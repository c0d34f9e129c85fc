"""CPU (gloo, world_size 2): the batch-shard plumbing of the multi-GPU path —
contiguous ceil(B/world) shards, no data-path collective, and the optional
final gather reassembles the batch in order."""
import os
import socket

import numpy as np
import pytest

from paper_2009_14788_b200.sharding import gather_batch, shard_range


def test_shard_ranges_cover_batch():
    for B in (1, 7, 8, 128, 129, 256):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(B, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a0 <= a1
            assert max(h - l for l, h in spans) == -(-B // world)
    assert shard_range(128, 8, 3) == (48, 64)
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _projector_worker(rank, world, port, B, q):
    """Each rank runs the reference projector (the CPU oracle, the checker) on its shard only;
    the gathered result must equal the single-process batch bit for bit (acceptance.cpp:340-389)."""
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import Geom, PortOracle, batched_phantom

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = PortOracle()
    g = Geom("parallel", 24, orc.angles_linspace(0.0, np.pi, 18))
    full = batched_phantom(orc, 24, B)
    lo, hi = shard_range(B, world, rank)
    local = torch.from_numpy(orc.forward(g, full[lo:hi]))
    out = gather_batch(local, B)
    if rank == 0:
        q.put(bool(np.array_equal(out.numpy(), orc.forward(g, full))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [5, 8])
def test_gloo_world2_sharded_projector(B):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_projector_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


def _worker(rank, world, port, B, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = torch.arange(B * 6, dtype=torch.float32).view(B, 2, 3)
    lo, hi = shard_range(B, world, rank)
    local = 2.0 * full[lo:hi]  # stand-in for the per-shard projector work (independent per element)
    out = gather_batch(local, B)
    if rank == 0:
        q.put(bool(torch.equal(out, 2.0 * full)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [7, 8])
def test_gloo_world2_gather(B):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
