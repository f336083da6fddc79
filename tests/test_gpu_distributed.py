"""The sharded CUDA path with more than one rank (two processes on the single B200, gloo).

Problems are independent (cli.py:191-193, README.md:133-135), so the ranks' kernels
never wait on one another; gloo carries only the host-side barrier, the timing
max-reduce and the result gather.  Checked: solve_sharded with the CUDA solver,
the chunked config runner (runner.run_sharded) and bench.py's rank logic under
torchrun all reproduce the single-process results bit for bit.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = ("beta", "objective", "steps", "descents", "iterations", "objective_evals", "converged", "status")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, out):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2510_15649_b200 as lad
    from paper_2510_15649_b200 import configgen as G
    from paper_2510_15649_b200.distributed import solve_sharded
    from paper_2510_15649_b200.runner import run_sharded

    if kind == "sharded":
        X, Y, L = G.generate(0, 333, seed=15649)

        def solve(x, y, lam):
            r = lad.solve_locus_batched(x, y, lam, lad.LocusConfig(outer_search="quadrature"))
            return {k: getattr(r, k) for k in FIELDS}

        s, e, local, gathered = solve_sharded(X, Y, L, solve)
        assert local["objective"].shape[0] == e - s
    else:
        res = run_sharded(config=4, total=2500, chunk=700, dtype=kind, gather=True)
        gathered = res.pop("results")
        gathered["stats"] = np.array(json.dumps(res))
    if rank == 0:
        np.savez(out, **gathered)
    dist.barrier()
    dist.destroy_process_group()


def _spawn(kind, tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / f"{kind}.npz")
    mp.start_processes(_worker, args=(2, _free_port(), kind, out), nprocs=2, join=True, start_method="spawn")
    return dict(np.load(out))


def _assert_equal(gathered, r):
    for k in FIELDS:
        mine = getattr(r, k).cpu().numpy()
        got = gathered[k]
        assert np.array_equal(got.astype(mine.dtype), mine), k


def test_solve_sharded_cuda_world2_equals_single_process(tmp_path):
    import paper_2510_15649_b200 as lad
    from paper_2510_15649_b200 import configgen as G

    g = _spawn("sharded", tmp_path)
    X, Y, L = G.generate(0, 333, seed=15649)
    _assert_equal(g, lad.solve_locus_batched(X, Y, L, lad.LocusConfig(outer_search="quadrature")))


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_chunked_runner_world2_equals_single_launch(tmp_path, dtype):
    """Config 4 at reduced size: 2 ranks x 700-problem chunks == one launch over all 2,500."""
    import paper_2510_15649_b200 as lad
    from paper_2510_15649_b200 import configgen as G

    g = _spawn(dtype, tmp_path)
    stats = json.loads(str(g.pop("stats")))
    X, Y, L = G.generate(4, 2500, seed=15653)
    if dtype == "f32":
        X, Y, L = X.float(), Y.float(), L.float()
    r = lad.solve_locus_batched(X, Y, L)
    _assert_equal(g, r)
    assert stats["solves"] == 2500 and stats["world"] == 2
    assert stats["coord_steps"] == int(r.steps.sum()) and stats["status_nonzero"] == 0


def test_runner_single_rank_writes_chunk_files(tmp_path):
    import paper_2510_15649_b200 as lad
    from paper_2510_15649_b200 import configgen as G
    from paper_2510_15649_b200.runner import run_sharded

    res = run_sharded(config=1, total=5000, chunk=2048, out_dir=str(tmp_path))
    files = sorted(os.listdir(tmp_path))
    assert len(files) == 3 and res["solves"] == 5000
    X, Y, L = G.generate(1, 5000, seed=15650)
    r = lad.solve_locus_batched(X, Y, L)
    obj = np.concatenate([np.load(os.path.join(tmp_path, f))["objective"] for f in files])
    assert np.array_equal(obj, r.objective.cpu().numpy())


def test_bench_torchrun_world2_gloo():
    """bench.py's rank > 0 path and max-over-ranks reduce, two ranks on the one GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--block", "512", "--no-cpu", "--dist-backend", "gloo"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, p.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["status_ok"] and line["config"]["solves_per_step_per_gpu"] == 512 * 16 * 2
    assert line["value"] > 0 and line["e2e"]["value"] > 0
