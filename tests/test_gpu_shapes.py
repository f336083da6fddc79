"""GPU shape sweep: every kernel variant against the oracle, bit for bit.

Rows n = 1..46 and variables p = 1..8 reach every instantiation: the warp kernel's
compile-time shapes and its runtime <3|5|8, 0> variants (n <= 31), the thread kernel's
(10,2) config-1 variant and its runtime (16,4), (32,8), (48,4), (48,8) variants
(n <= 46: the modelled OpenBLAS ddot range), the simplex (m <= 46), the certificate and
brute force.  n = 47 is rejected (LAD_E_UNSUPPORTED -> InvalidInputError).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_15649_b200 as lad  # noqa: E402

SHAPES = [(1, 1), (2, 1), (5, 2), (9, 3), (10, 2), (16, 4), (17, 5), (24, 6), (25, 5), (30, 5), (31, 8), (32, 3),
          (33, 2), (38, 4), (40, 6), (46, 8)]


def _problems(n, p, B, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((B, n, p))
    if n > 3:
        X[::4, rng.integers(0, n), rng.integers(0, p)] = 0.0  # a zero entry: the sparse path
    beta = np.where(rng.random(p) < 0.5, rng.uniform(1, 3, p), 0.0)
    Y = X @ beta + rng.laplace(0, 0.5, (B, n))
    L = rng.choice([0.01, 0.3, 1.5], B)
    return X, Y, L


@pytest.mark.parametrize("n,p", SHAPES)
def test_locus_all_shapes_bit_exact(oracle, n, p):
    X, Y, L = _problems(n, p, 8, 1000 * n + p)
    for variant in ("ternary", "quadrature"):
        r = lad.solve_locus_batched(X, Y, L, lad.LocusConfig(outer_search=variant))
        o = oracle.solve_locus_batch(X, Y, L, outer_search=variant)
        assert np.array_equal(r.status, o["status"]), (n, p, variant)
        ok = np.asarray(o["status"]) == 0
        assert np.array_equal(r.beta[ok], o["beta"][ok]) and np.array_equal(r.objective[ok], o["objective"][ok])
        assert np.array_equal(r.steps, o["steps"]) and np.array_equal(r.descents, o["descents"]), (n, p, variant)
        assert np.array_equal(r.iterations[ok], o["iterations"][ok])


@pytest.mark.parametrize("n,p", [s for s in SHAPES if s[0] >= 2])
def test_lp_and_certificate_all_shapes(oracle, n, p):
    X, Y, L = _problems(n, p, 6, 2000 * n + p)
    lp = lad.solve_lp_batched(X, Y, L, full=True)
    cert = lad.axiswise_minimum_batched(X, Y, L, lp.beta)
    for i in range(len(L)):
        o = oracle.lp_solve(X[i], Y[i], max(float(L[i]), 1e-9))
        assert np.array_equal(lp.x[i], o.x) and int(lp.pivots[i]) == o.pivots, (n, p, i)
        assert np.array_equal(lp.beta[i], o.beta) and lp.objective[i] == o.objective
        assert bool(cert[i]) == oracle.is_axiswise_minimum(X[i], Y[i], max(float(L[i]), 1e-9), lp.beta[i])


@pytest.mark.parametrize("n,p", [(12, 2), (40, 2), (46, 3)])
def test_brute_beyond_32_rows(oracle, n, p):
    X, Y, L = _problems(n, p, 4, 3000 * n + p)
    beta, obj, nv = lad.solve_brute_batched(X, Y, L)
    for i in range(len(L)):
        ob, oo, ov = oracle.solve_brute(X[i], Y[i], max(float(L[i]), 1e-9))
        assert np.array_equal(beta[i], ob) and obj[i] == oo and nv[i] == ov


def test_shape_limits_are_reported():
    X, Y, L = _problems(1024, 2, 2, 5)
    with pytest.raises(lad.InvalidInputError):
        lad.solve_locus_batched(X, Y, L)
    X, Y, L = _problems(47, 2, 2, 5)
    with pytest.raises(lad.InvalidInputError):
        lad.solve_lp_batched(X, Y, L)
    X32 = X[:, :32].astype(np.float32)
    with pytest.raises(lad.InvalidInputError):  # fp32 mode: warp kernel only (n <= 31)
        lad.solve_locus_batched(X32, Y[:, :32].astype(np.float32), L.astype(np.float32))


def test_block_kernel_large_goldens():
    """47 <= n <= 1023 (block per problem) against the reference: ccd_descend up to 1000 rows,
    solve_locus (both variants, work counters) up to 256 rows (tests/golden/large.npz)."""
    from conftest import load_golden

    g = load_golden("large")
    for i in range(len(g["ccd_lam"])):
        m, d = int(g["ccd_m"][i]), int(g["ccd_d"][i])
        if m <= 46:
            continue
        fr = int(g["ccd_frozen"][i])
        r = lad.ccd_descend_batched(g["ccd_x"][i, :m, :d][None], g["ccd_y"][i, :m][None], g["ccd_lam"][i:i + 1],
                                    g["ccd_start"][i, :d][None], lad.CcdConfig(), frozen=None if fr < 0 else fr)
        assert np.array_equal(r.beta[0], g["ccd_beta"][i, :d]) and r.objective[0] == g["ccd_objective"][i], (i, m, d)
        assert (r.iterations[0], r.objective_evals[0]) == (g["ccd_iterations"][i], g["ccd_objective_evals"][i])
    for i in range(len(g["locus_lam"])):
        m, d = int(g["locus_m"][i]), int(g["locus_d"][i])
        v = "quadrature" if g["locus_variant"][i] else "ternary"
        r = lad.solve_locus_batched(g["locus_x"][i, :m, :d][None], g["locus_y"][i, :m][None], g["locus_lam"][i:i + 1],
                                    lad.LocusConfig(outer_search=v))
        assert r.status[0] == 0
        assert np.array_equal(r.beta[0], g["locus_beta"][i, :d]) and r.objective[0] == g["locus_objective"][i], (i, m)
        assert (r.descents[0], r.steps[0]) == (g["locus_D"][i], g["locus_S"][i]), (i, m)
        assert (r.iterations[0], r.objective_evals[0]) == (g["locus_iterations"][i], g["locus_objective_evals"][i])


@pytest.mark.parametrize("n,p", [(47, 2), (64, 5), (100, 3), (129, 8), (200, 4), (333, 1), (1023, 2)])
def test_block_kernel_against_oracle(oracle, n, p):
    X, Y, L = _problems(n, p, 3, 4000 + n * p)
    r = lad.solve_locus_batched(X, Y, L)
    o = oracle.solve_locus_batch(X, Y, L)
    assert np.array_equal(r.status, o["status"])
    assert np.array_equal(r.beta, o["beta"]) and np.array_equal(r.objective, o["objective"]), (n, p)
    assert np.array_equal(r.steps, o["steps"]) and np.array_equal(r.descents, o["descents"]), (n, p)
