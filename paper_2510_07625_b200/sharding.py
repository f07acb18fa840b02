"""Multi-GPU data parallelism over independent solves.

One process per GPU (torch.distributed).  Solves are independent, so the batch is split into
contiguous index ranges [g*M/G, (g+1)*M/G), each rank solves its range with its own engine
and there is NO collective on the solve path; the only communication is the final gather of
X, U, trace and status words to rank 0 (NCCL over NVLink on GPUs; gloo in the CPU tests).
Results are bitwise independent of the number of shards and of a solve's position in its
shard: every reduction inside a solve is a fixed tree that never mixes solves.
"""

from __future__ import annotations

import numpy as np

from .batch import shard_bounds
from .engine import PackedBatch, PackedResult


def local_shard(batch: PackedBatch, rank: int, world: int) -> tuple[PackedBatch, tuple[int, int]]:
    lo, hi = shard_bounds(batch.size, world)[rank]
    return batch.slice(lo, hi), (lo, hi)


def gather_results(local: PackedResult, sizes: list[int], rank: int, world: int, device=None,
                   group=None) -> PackedResult | None:
    """Gather per-shard results to rank 0 in batch order.  ``sizes[g]`` = solves of shard g.
    Tensors travel on ``device`` (cuda for NCCL, cpu for gloo)."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    out = {}
    mmax = max(sizes)
    for name in ("X", "U", "trace", "info"):
        arr = getattr(local, name)
        pad = np.zeros((mmax,) + arr.shape[1:], dtype=arr.dtype)
        pad[:arr.shape[0]] = arr
        t = torch.from_numpy(pad)
        if device is not None:
            t = t.to(device)
        bucket = [torch.empty_like(t) for _ in range(world)] if rank == 0 else None
        dist.gather(t, bucket, dst=0, group=group)
        if rank == 0:
            out[name] = np.concatenate([bucket[g][:sizes[g]].cpu().numpy() for g in range(world)], axis=0)
    ms = torch.tensor([local.device_ms], dtype=torch.float64)
    if device is not None:
        ms = ms.to(device)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=group)
    if rank != 0:
        return None
    return PackedResult(out["X"], out["U"], out["trace"], out["info"], float(ms.item()))


def solve_sharded(batch: PackedBatch, solve_fn, rank: int, world: int, device=None, group=None):
    """Rank-local solve of this rank's contiguous shard + final gather to rank 0.

    ``solve_fn(PackedBatch) -> PackedResult`` is the rank's engine (BatchEngine.solve on a GPU)."""
    if batch.size < world:
        raise ValueError("sharded solve needs at least one solve per rank")
    shard, _ = local_shard(batch, rank, world)
    sizes = [hi - lo for lo, hi in shard_bounds(batch.size, world)]
    return gather_results(solve_fn(shard), sizes, rank, world, device=device, group=group)
