"""Batch sharding across GPUs (one process per GPU) — SURVEY 8e.

Every batch element is independent in the reference (no cross-element term in
forward / backprojection / filter, per-element solver scalars,
solvers.cpp:56-104), so the batch is split into contiguous shards of
ceil(B / world) elements with NO collective on the data path.  The only
communication is the optional final gather of results to one rank
(``gather_batch``), outside any timed region.
"""
from __future__ import annotations

import numpy as np


def shard_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of rank `rank` (may be empty for trailing ranks)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    per = -(-int(batch) // int(world))
    lo = min(int(batch), rank * per)
    return lo, min(int(batch), lo + per)


def gather_batch(local, global_batch: int, dst: int = 0, group=None):
    """Concatenate every rank's shard on rank `dst` (torch.distributed: NCCL
    all-gather for CUDA tensors; gloo gathers through host memory, so CUDA
    shards under gloo — e.g. several ranks sharing one GPU, which NCCL
    rejects — are staged on the CPU).  Returns the full batch on `dst`, on the
    shard's device, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = -(-int(global_batch) // world)
    shape = tuple(local.shape[1:])
    nccl = dist.get_backend(group) == "nccl"
    home = local.device
    work = home if nccl else torch.device("cpu")
    padded = torch.zeros((per, *shape), dtype=local.dtype, device=work)
    padded[: local.shape[0]] = local.to(work)
    if nccl:
        parts = [torch.empty_like(padded) for _ in range(world)]
        dist.all_gather(parts, padded, group=group)
    else:
        parts = [torch.empty_like(padded) for _ in range(world)] if rank == dst else None
        dist.gather(padded, parts, dst=dst, group=group)
    if rank != dst:
        return None
    out = []
    for r in range(world):
        lo, hi = shard_range(global_batch, world, r)
        out.append(parts[r][: hi - lo])
    return torch.cat(out, 0).to(home)


def shard_numpy(x: np.ndarray, world: int, rank: int) -> np.ndarray:
    lo, hi = shard_range(x.shape[0], world, rank)
    return x[lo:hi]
