"""Device-side generation of the BASELINE.json config problems (csrc/lad_gen.cuh).

Config shapes (BASELINE.json ``configs``):
  0  B=256,   n=30, p=5, lambda=1                   ternary
  1  B=2^20,  n=10, p=2, lambda~U(0.1,2)            both variants + brute check
  2  B=2^20,  n=30, p=5, 16-point lambda grid 1e-2..1e1 (16.8M solves), both variants
  3  C(30,25)=142,506 subsets of one n=30 dataset, lambda=0.5, quadrature
  4  B=64M (2^26), n=31, p=8, heavy tails, lambda=1 ternary
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .solver import _check

CONFIG_SHAPES = {0: (30, 5), 1: (10, 2), 2: (30, 5), 3: (25, 5), 4: (31, 8)}
CONFIG_BATCH = {0: 256, 1: 1 << 20, 2: 1 << 20, 3: math.comb(30, 25), 4: 1 << 26}
LAMBDA_GRID = 10.0 ** np.linspace(-2.0, 1.0, 16)
DEFAULT_SEED = 15649


def generate(config: int, B: int, seed: int = DEFAULT_SEED, first: int = 0, device="cuda", with_beta=False):
    """Problems [first, first + B) of a config as CUDA tensors (X, y, lam[, beta_true])."""
    import torch

    if config == 3:
        raise ValueError("config 3 problems are subsets: use subsets()")
    n, p = CONFIG_SHAPES[config]
    dev = torch.device(device)
    X = torch.empty((B, n, p), dtype=torch.float64, device=dev)
    y = torch.empty((B, n), dtype=torch.float64, device=dev)
    lam = torch.empty(B, dtype=torch.float64, device=dev)
    bt = torch.empty((B, p), dtype=torch.float64, device=dev) if with_beta else None
    L = _lib.load()
    _check(L.lad_generate_f64(config, seed, first, B, n, p, X.data_ptr(), y.data_ptr(), lam.data_ptr(),
                              bt.data_ptr() if bt is not None else None, torch.cuda.current_stream(dev).cuda_stream))
    return (X, y, lam, bt) if with_beta else (X, y, lam)


def subsets(X0, y0, keep: int, first: int, B: int):
    """Config 3: the k-th ``keep``-row subsets (lexicographic) of one dataset, k in [first, first+B)."""
    import torch

    X0 = X0.contiguous()
    y0 = y0.contiguous()
    n0, p = X0.shape
    X = torch.empty((B, keep, p), dtype=torch.float64, device=X0.device)
    y = torch.empty((B, keep), dtype=torch.float64, device=X0.device)
    L = _lib.load()
    _check(L.lad_subsets_f64(X0.data_ptr(), y0.data_ptr(), n0, p, keep, first, B, X.data_ptr(), y.data_ptr(),
                             torch.cuda.current_stream(X0.device).cuda_stream))
    return X, y


def config3_dataset(seed: int = DEFAULT_SEED + 3, device="cuda"):
    """The one n=30, p=5 dataset config 3 subsets (generated as config 0, problem 0)."""
    X, y, _ = generate(0, 1, seed=seed, device=device)
    return X[0], y[0]
