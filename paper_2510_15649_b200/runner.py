"""Chunked, sharded solve of a whole BASELINE config (config 4: all 2^26 problems).

The reference's only concurrency is a process pool over independent problems
(cli.py:191-193; solvers are pure per problem, README.md:133-135).  Here each
rank (one process per GPU, torch.distributed with any backend) takes the
contiguous shard ``shard_range(total, world, rank)`` of the problem index
space and walks it in chunks: generate the chunk on the device
(lad_generate_f64, keyed by (seed, global index), so no input crosses the
host or the network), solve it, copy the results to the host.  Device memory
is bounded by one chunk; the host keeps only per-chunk statistics unless
``out_dir`` asks for per-chunk result files.  The only collectives are the
final max-reduce of the time and the sum of the statistics (plus an optional
gather of the per-problem results, for tests and small totals).

    python -m paper_2510_15649_b200.runner --config 4 --total 67108864 --chunk 1048576 [--dtype f32]
    torchrun --nproc-per-node 8 -m paper_2510_15649_b200.runner --config 4 ...
"""

from __future__ import annotations

import argparse
import json
import os
import time

import numpy as np

from .distributed import shard_range

SEEDS = {c: 15649 + c for c in range(5)}
FIELDS = ("beta", "objective", "iterations", "objective_evals", "converged", "status", "descents", "steps")


def run_sharded(config: int = 4, total: int = 1 << 26, chunk: int = 1 << 20, dtype: str = "f64",
                variant: str = "ternary", seed: int | None = None, out_dir: str | None = None,
                gather: bool = False, group=None):
    """Solve problems [0, total) of `config` across the ranks of `group`; returns a dict with the
    aggregate statistics (identical on every rank) and, with gather=True, the per-problem
    results in global index order (rank 0 only)."""
    import torch
    import torch.distributed as dist

    import paper_2510_15649_b200 as lad
    from . import configgen as G

    if config not in (0, 1, 2, 4):
        raise ValueError("run_sharded generates configs 0, 1, 2 and 4 (config 3 is one dataset's subsets)")
    seed = SEEDS[config] if seed is None else seed
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    dev = torch.device("cuda", torch.cuda.current_device())
    s0, e0 = shard_range(total, world, rank)
    cfg = lad.LocusConfig(outer_search=variant)
    stats = np.zeros(6)  # solves, status!=0, converged, coordinate steps, descents, sum of objectives
    local = {k: [] for k in FIELDS} if gather else None
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(group)
    ev0.record()
    for first in range(s0, e0, chunk):
        B = min(chunk, e0 - first)
        X, Y, L = G.generate(config, B, seed=seed, first=first, device=dev)
        if dtype == "f32":
            X, Y, L = X.float(), Y.float(), L.float()
        r = lad.solve_locus_batched(X, Y, L, cfg)
        res = {k: getattr(r, k) for k in FIELDS}
        stats += np.array([B, float((r.status != 0).sum()), float(r.converged.sum()), float(r.steps.sum()),
                           float(r.descents.sum()), float(r.objective.double().sum())])
        if out_dir or gather:
            host = {k: v.cpu().numpy() for k, v in res.items()}
            if out_dir:
                np.savez(os.path.join(out_dir, f"config{config}_{dtype}_{first:012d}.npz"), first=first, **host)
            if gather:
                for k in FIELDS:
                    local[k].append(host[k])
    ev1.record()
    torch.cuda.synchronize()
    elapsed = ev0.elapsed_time(ev1) / 1e3
    on_gpu = dist.is_initialized() and dist.get_backend(group) == "nccl"
    t = torch.tensor([elapsed], dtype=torch.float64, device=dev if on_gpu else "cpu")
    st = torch.tensor(stats, dtype=torch.float64, device=dev if on_gpu else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(st, op=dist.ReduceOp.SUM, group=group)
    st = st.cpu().numpy()
    out = {"config": config, "dtype": dtype, "variant": variant, "total": total, "chunk": chunk, "world": world,
           "seconds_max_over_ranks": float(t.item()), "solves_per_s": total / float(t.item()),
           "solves": int(st[0]), "status_nonzero": int(st[1]), "converged": int(st[2]),
           "coord_steps": int(st[3]), "descents": int(st[4]), "objective_sum": float(st[5])}
    if gather:
        from .distributed import gather_results

        mine = {k: (np.concatenate(v) if v else np.zeros((0,) + ((cfg_p(config),) if k == "beta" else ())))
                for k, v in local.items()}
        out["results"] = gather_results(mine, total, group)
    return out


def cfg_p(config: int) -> int:
    return {0: 5, 1: 2, 2: 5, 4: 8}[config]


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--total", type=int, default=1 << 26)
    ap.add_argument("--chunk", type=int, default=1 << 20)
    ap.add_argument("--dtype", choices=["f64", "f32"], default="f64")
    ap.add_argument("--variant", choices=["ternary", "quadrature"], default="ternary")
    ap.add_argument("--out-dir", default=None, help="write one result file per chunk")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group(a.dist_backend, **({"device_id": dev} if a.dist_backend == "nccl" else {}))
    res = run_sharded(a.config, a.total, a.chunk, a.dtype, a.variant, out_dir=a.out_dir)
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
