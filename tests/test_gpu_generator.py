"""The device config generator (lad_generate_f64 / lad_subsets_f64) against its host
restatement (oracle/gen_host.c): byte-identical problems.

This equality is what lets the CPU reference arm (bench.py --impl reference), the
cpu_baseline leg and the reference-held goldens (tests/golden/bench_cfg*.npz) use
exactly the problems the GPU solves without loading the product library.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2510_15649_b200 import configgen as G  # noqa: E402


@pytest.mark.parametrize("config", [0, 1, 2, 4])
@pytest.mark.parametrize("first", [0, 1 << 20, (1 << 26) - 4096, (1 << 40) + 12345])
def test_generate_bytes_equal_host_port(oracle, config, first):
    seed = 15649 + config
    B = 4096
    X, Y, L, bt = G.generate(config, B, seed=seed, first=first, with_beta=True)
    hX, hY, hL, hbt = oracle.generate(config, B, seed, first, with_beta=True)
    assert np.array_equal(X.cpu().numpy().view(np.uint64), hX.view(np.uint64))
    assert np.array_equal(Y.cpu().numpy().view(np.uint64), hY.view(np.uint64))
    assert np.array_equal(L.cpu().numpy().view(np.uint64), hL.view(np.uint64))
    assert np.array_equal(bt.cpu().numpy().view(np.uint64), hbt.view(np.uint64))


def test_generate_bench_steps_equal_host_port(oracle):
    """The config-2 bench blocks (seed 15651, 16384 datasets per block) at two block offsets."""
    for first in (0, 63 * 16384):
        X, Y, _ = G.generate(2, 16384, seed=15651, first=first)
        hX, hY, _ = oracle.generate(2, 16384, 15651, first)
        assert np.array_equal(X.cpu().numpy(), hX) and np.array_equal(Y.cpu().numpy(), hY)


def test_subsets_all_config3_equal_host_port(oracle):
    X0, Y0 = G.config3_dataset()
    hX0, hY0 = oracle.config3_dataset()
    assert np.array_equal(X0.cpu().numpy(), hX0) and np.array_equal(Y0.cpu().numpy(), hY0)
    total = G.CONFIG_BATCH[3]
    Xs, Ys = G.subsets(X0, Y0, 25, 0, total)
    hXs, hYs = oracle.subsets(hX0, hY0, 25, 0, total)
    assert np.array_equal(Xs.cpu().numpy(), hXs) and np.array_equal(Ys.cpu().numpy(), hYs)
