"""Multi-process sharding on CPU (gloo, world_size 2): shards are disjoint and complete,
and gathered per-problem results equal the single-process solve.  The solve
callback here is the CPU oracle (test infrastructure); on GPUs bench.py uses
the same shard logic with the CUDA solver and NCCL."""

import os
import socket

import numpy as np
import pytest

from paper_2510_15649_b200.distributed import block_for_step, shard_range


def test_shard_range_partitions():
    for B in (0, 1, 7, 256, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_range(B, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == B
            for (s0, e0), (s1, e1) in zip(ranges, ranges[1:]):
                assert e0 == s1
            sizes = [e - s for s, e in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_weak_scaling_schedule_is_disjoint_per_step():
    for world in (1, 2, 4, 8):
        for step in range(5):
            blocks = [block_for_step(step, world, r, 64) for r in range(world)]
            assert len(set(blocks)) == world


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, X, Y, L, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2510_15649_b200.distributed import solve_sharded

    def solve(x, y, lam):
        r = O.solve_locus_batch(x, y, lam, nthreads=1)
        return {"beta": r["beta"], "objective": r["objective"], "steps": r["steps"]}

    s, e, local, gathered = solve_sharded(X, Y, L, solve)
    if rank == 0:
        np.savez(out, **gathered)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather_equals_serial(tmp_path, oracle):
    import torch.multiprocessing as mp

    rng = np.random.default_rng(3)
    X = rng.standard_normal((9, 8, 2))
    Y = rng.standard_normal((9, 8))
    L = rng.uniform(0.05, 1.0, 9)
    out = str(tmp_path / "g.npz")
    mp.start_processes(_worker, args=(2, _free_port(), X, Y, L, out), nprocs=2, join=True, start_method="spawn")
    g = np.load(out)
    ref = oracle.solve_locus_batch(X, Y, L, nthreads=1)
    assert np.array_equal(g["objective"], ref["objective"])
    assert np.array_equal(g["beta"], ref["beta"])
    assert np.array_equal(g["steps"], ref["steps"])
