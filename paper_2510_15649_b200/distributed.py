"""Sharding of independent LAD-LASSO problems across GPUs (one process per GPU).

The reference's only concurrency is a ProcessPoolExecutor over independent
problems (cli.py:191-193); solvers are pure per problem (README.md:133-135).
On B200 the same holds across GPUs: problems are split by global index into
contiguous shards with no exchange step on the solve path.
The only collectives are bookkeeping: a barrier + max-reduce of the timing,
and an optional final gather of the per-problem results.
"""

from __future__ import annotations

import numpy as np


def shard_range(B: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, end) of problems owned by `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    base, extra = divmod(B, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def block_for_step(step: int, world: int, rank: int, nblocks: int) -> int:
    """Weak-scaling schedule: at step s rank r solves block (s * world + r) mod nblocks."""
    return (step * world + rank) % nblocks


def solve_sharded(X, y, lam, solve, group=None, gather: bool = True):
    """Solve the rank's shard of (X, y, lam) with `solve` and optionally all-gather the results.

    `solve(X_shard, y_shard, lam_shard)` returns a dict of per-problem arrays
    (numpy or torch).  Works with any torch.distributed backend (NCCL across
    GPUs; gloo in the CPU tests).  Returns (start, end, local_result,
    gathered_or_None).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B = X.shape[0]
    s, e = shard_range(B, world, rank)
    local = solve(X[s:e], y[s:e], lam[s:e])
    if not gather or world == 1:
        return s, e, local, (local if world == 1 else None)
    return s, e, local, gather_results(local, B, group)


def gather_results(local: dict, B: int, group=None) -> dict:
    """All-gather per-problem result arrays (numpy or torch, first axis = the rank's contiguous
    shard of B problems) into global index order on every rank, as numpy arrays.  With NCCL the
    buffers go through the current CUDA device; with gloo they stay on the host."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return {k: np.asarray(v.cpu() if torch.is_tensor(v) else v) for k, v in local.items()}
    counts = [shard_range(B, world, r)[1] - shard_range(B, world, r)[0] for r in range(world)]
    cap = max(counts)
    gathered = {}
    for key, val in local.items():
        t = torch.as_tensor(np.asarray(val.cpu() if torch.is_tensor(val) else val))
        if t.dtype == torch.bool:
            t = t.to(torch.uint8)
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else t.device
        pad = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype)
        pad[: t.shape[0]] = t
        pad = pad.to(dev)
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad, group=group)
        gathered[key] = torch.cat([b[:c].cpu() for b, c in zip(bufs, counts)]).numpy()
    return gathered
