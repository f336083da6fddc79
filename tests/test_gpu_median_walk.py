"""The weighted median's order-neighbour walk on tie-heavy inputs, against the oracle bit for bit.

The walk (lad_locus_warp.cuh, lad_locus_block.cuh) steps from an axis' previous median to
the new one through neighbours in the stable (location, index) order, which on equal
locations is decided by the index alone, and folds -0.0 onto +0.0 in its order key.
Integer-valued data with small-integer columns make many breakpoints r_i / x_ij + b_j
coincide exactly (and zero residuals give signed zeros), so these cases pin the tie rules
of ccd.py:83-88 (stable argsort, first index with cum >= total / 2) through every path:
the warp kernel (n <= 31), its fp32 mode, and the block kernel (n >= 32).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_15649_b200 as lad  # noqa: E402


def _tie_heavy(n, p, B, seed, zero_rows=0):
    rng = np.random.default_rng(seed)
    X = rng.choice([-2.0, -1.0, 1.0, 2.0], size=(B, n, p))
    beta = rng.integers(-2, 3, size=(B, p)).astype(np.float64)
    Y = np.einsum("bij,bj->bi", X, beta) + rng.integers(-3, 4, size=(B, n))
    if zero_rows:
        Y[:, :zero_rows] = 0.0  # with beta = 0 starts: zero residuals, signed-zero breakpoints
    L = rng.choice([0.25, 0.5, 1.0, 2.0, 4.0], B)
    return X, Y, L


def _assert_exact(r, o, what):
    assert np.array_equal(r.status, o["status"]), what
    ok = np.asarray(o["status"]) == 0
    assert np.array_equal(r.beta[ok], o["beta"][ok]), what
    assert np.array_equal(r.objective[ok], o["objective"][ok]), what
    assert np.array_equal(r.steps, o["steps"]) and np.array_equal(r.descents, o["descents"]), what
    assert np.array_equal(r.iterations[ok], o["iterations"][ok]), what


@pytest.mark.parametrize("n,p", [(30, 5), (25, 5), (31, 8), (12, 3), (31, 2)])
@pytest.mark.parametrize("variant", ["ternary", "quadrature"])
def test_warp_walk_ties_bit_exact(oracle, n, p, variant):
    X, Y, L = _tie_heavy(n, p, 48, 100 * n + p, zero_rows=3)
    r = lad.solve_locus_batched(X, Y, L, lad.LocusConfig(outer_search=variant))
    o = oracle.solve_locus_batch(X, Y, L, outer_search=variant)
    _assert_exact(r, o, (n, p, variant))


@pytest.mark.parametrize("n,p", [(30, 5), (31, 8)])
def test_warp_walk_ties_fp32_bit_exact(oracle, n, p):
    X, Y, L = (a.astype(np.float32) for a in _tie_heavy(n, p, 32, 7 * n + p, zero_rows=2))
    r = lad.solve_locus_batched(X, Y, L)
    o = oracle.solve_locus_batch(X, Y, L)
    _assert_exact(r, o, (n, p, "fp32"))


@pytest.mark.parametrize("n,p", [(40, 5), (64, 3), (100, 4), (200, 2)])
def test_block_walk_ties_bit_exact(oracle, n, p):
    X, Y, L = _tie_heavy(n, p, 6, 31 * n + p, zero_rows=4)
    r = lad.solve_locus_batched(X, Y, L)
    o = oracle.solve_locus_batch(X, Y, L)
    _assert_exact(r, o, (n, p, "block"))


def test_ccd_descend_from_tied_starts(oracle):
    """Plain descents from integer starts: every first step's median sits on a tie."""
    X, Y, L = _tie_heavy(30, 5, 64, 5, zero_rows=4)
    rng = np.random.default_rng(9)
    start = rng.integers(-2, 3, size=(64, 5)).astype(np.float64)
    r = lad.ccd_descend_batched(X, Y, L, start, lad.CcdConfig())
    for b in range(64):
        d = oracle.ccd_descend(X[b], Y[b], float(L[b]), start[b])
        assert np.array_equal(r.beta[b], d.beta) and r.objective[b] == d.objective, b
        assert (r.iterations[b], r.objective_evals[b]) == (d.iterations, d.objective_evals), b
