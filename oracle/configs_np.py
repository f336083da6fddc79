"""Host-side (numpy) generators for BASELINE.json-shaped problems.

TEST INFRASTRUCTURE ONLY: these build the *inputs* of the golden fixtures in
tests/golden (oracle/gen_golden.py) and of CPU-only tests.  The product
generates its benchmark problems on the device (csrc/ladlasso_gen.cuh); parity
at full size copies those exact device bytes back to the host for the oracle.

Distributions follow BASELINE.json ``configs`` (no dataset is involved; the
reference's own datagen.py cannot produce them):
  cfg0/2  X ~ N(0,1); beta_true: 2 nonzeros +-U[1,3] at random positions;
          y = X beta + Laplace(0, 0.5); 10% of rows get y += +-10.
  cfg1    X ~ U(-1,1); beta_true ~ N(0,1); Laplace(0, 0.3); lambda ~ U(0.1, 2).
  cfg3    one cfg0 dataset; problem k = k-th 25-of-30 row subset (lexicographic).
  cfg4    X ~ Student-t(3); 3 nonzeros +-U[1,3]; noise Cauchy(0, 0.2); lambda = 1.
"""

from __future__ import annotations

import itertools

import numpy as np

LAMBDA_GRID = 10.0 ** np.linspace(-2.0, 1.0, 16)


def cfg0(rng, B, n=30, p=5, k_true=2, laplace=0.5, outlier_frac=0.1, outlier=10.0):
    X = rng.standard_normal((B, n, p))
    beta = np.zeros((B, p))
    for b in range(B):
        pos = rng.choice(p, k_true, replace=False)
        beta[b, pos] = rng.choice([-1.0, 1.0], k_true) * rng.uniform(1.0, 3.0, k_true)
    y = np.einsum("bij,bj->bi", X, beta) + rng.laplace(0.0, laplace, (B, n))
    n_out = int(round(outlier_frac * n))
    for b in range(B):
        rows = rng.choice(n, n_out, replace=False)
        y[b, rows] += rng.choice([-outlier, outlier], n_out)
    return X, y, beta


def cfg1(rng, B, n=10, p=2):
    X = rng.uniform(-1.0, 1.0, (B, n, p))
    beta = rng.standard_normal((B, p))
    y = np.einsum("bij,bj->bi", X, beta) + rng.laplace(0.0, 0.3, (B, n))
    lam = rng.uniform(0.1, 2.0, B)
    return X, y, lam


def cfg3_subsets(X0, y0, ks, keep=25):
    n = X0.shape[0]
    combos = list(itertools.combinations(range(n), keep))
    Xs = np.stack([X0[list(combos[k])] for k in ks])
    ys = np.stack([y0[list(combos[k])] for k in ks])
    return Xs, ys


def cfg4(rng, B, n=31, p=8, k_true=3):
    X = rng.standard_t(3.0, (B, n, p))
    beta = np.zeros((B, p))
    for b in range(B):
        pos = rng.choice(p, k_true, replace=False)
        beta[b, pos] = rng.choice([-1.0, 1.0], k_true) * rng.uniform(1.0, 3.0, k_true)
    y = np.einsum("bij,bj->bi", X, beta) + 0.2 * rng.standard_cauchy((B, n))
    return X, y, beta
