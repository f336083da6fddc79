"""fp32 mode (BASELINE config 4 "fp64 and fp32"): GPU against the binary32 oracle.

The reference has no binary32 path (model.py:33 casts inputs to float64), so the
fp32 mode is this library's definition (include/ladlasso_b200.h): binary32 data
and coordinate descents, binary64 outer search.  The oracle restates exactly
that (oracle/orc_descent.inc compiled with REAL=float), so the bar here is
again bit-exact: beta, objective, counters.  Distance to the fp64 reference is
measured and bounded loosely (it is a statistic of the heuristic, not a
contract): |f32 objective - f64 objective| / f64 objective <= 1e-2 per problem.
"""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_15649_b200 as lad  # noqa: E402
from paper_2510_15649_b200 import _lib  # noqa: E402
from paper_2510_15649_b200 import configgen as G  # noqa: E402


def _np(a):
    return a.cpu().numpy() if torch.is_tensor(a) else np.asarray(a)


def _exact(oracle, X, Y, L, r, variant="ternary", idx=None):
    X, Y, L = (np.asarray(_np(a), dtype=np.float32) for a in (X, Y, L))
    idx = np.arange(len(L)) if idx is None else idx
    ref = oracle.solve_locus_batch(X[idx], Y[idx], L[idx], outer_search=variant)
    got = {k: _np(getattr(r, k))[idx] for k in ("beta", "objective", "iterations", "objective_evals", "converged",
                                                  "descents", "steps")}
    assert np.array_equal(got["beta"], ref["beta"])
    assert np.array_equal(got["objective"], ref["objective"])
    for k in ("iterations", "objective_evals", "converged", "descents", "steps"):
        assert np.array_equal(got[k].astype(np.int64), np.asarray(ref[k]).astype(np.int64)), k
    return ref


@pytest.mark.parametrize("axis_parallel", [False, True])
def test_cfg4_golden_inputs_fp32_bit_exact(oracle, axis_parallel):
    g = load_golden("cfg4")
    X, Y, L = (g["x"].astype(np.float32), g["y"].astype(np.float32), g["lam"].astype(np.float32))
    _lib.set_axis_parallel(axis_parallel)
    try:
        r = lad.solve_locus_batched(X, Y, L)
    finally:
        _lib.set_axis_parallel(True)
    assert (r.status == 0).all()
    _exact(oracle, X, Y, L, r)
    # distance to the fp64 reference on the same (binary32-representable) data
    r64 = lad.solve_locus_batched(X.astype(np.float64), Y.astype(np.float64), L.astype(np.float64))
    gap = np.abs(r.objective - r64.objective) / np.abs(r64.objective)
    assert gap.max() <= 1e-2, gap.max()


def test_cfg4_device_shard_fp32_against_oracle(oracle):
    """Device-generated config 4 shard cast to binary32 on the device; oracle on a sample."""
    X, Y, L = G.generate(4, 2048, seed=404, first=99)
    Xf, Yf, Lf = X.float(), Y.float(), L.float()
    r = lad.solve_locus_batched(Xf, Yf, Lf)
    torch.cuda.synchronize()
    assert bool((r.status == 0).all())
    _exact(oracle, Xf, Yf, Lf, r, idx=np.arange(0, 2048, 64))


@pytest.mark.parametrize("variant", ["ternary", "quadrature"])
def test_fp32_generic_shapes_and_sparse_columns(oracle, variant):
    """Runtime-shape fp32 kernels (<3,0>, <5,0>, <8,0>, <5,30>), zero columns (sparse path), per-problem lambdas."""
    rng = np.random.default_rng(7)
    for (n, p) in ((12, 2), (9, 3), (17, 4), (30, 5), (23, 7), (31, 8)):
        B = 24
        X = rng.standard_normal((B, n, p)).astype(np.float32)
        X[::3, rng.integers(0, n, 3), rng.integers(0, p)] = 0.0
        X[1::5, :, 0] = 0.0  # a whole zero column
        Y = (X[:, :, 0] * 2 - X[:, :, -1] + rng.laplace(0, 0.5, (B, n))).astype(np.float32)
        L = rng.uniform(0.05, 2.0, B).astype(np.float32)
        r = lad.solve_locus_batched(X, Y, L, lad.LocusConfig(outer_search=variant))
        assert (r.status == 0).all(), (n, p)
        _exact(oracle, X, Y, L, r, variant)


def test_fp32_ccd_descend_bit_exact(oracle):
    rng = np.random.default_rng(11)
    n, p, B = 25, 5, 16
    X = rng.standard_normal((B, n, p)).astype(np.float32)
    Y = rng.standard_normal((B, n)).astype(np.float32)
    L = np.full(B, 0.3, np.float32)
    start = rng.standard_normal((B, p))
    for frozen in (None, 2):
        r = lad.ccd_descend_batched(X, Y, L, start, lad.CcdConfig(), frozen=frozen)
        for b in range(B):
            d = oracle.ccd_descend(X[b], Y[b], float(L[b]), start[b], frozen_axis=frozen)
            assert np.array_equal(r.beta[b], d.beta) and r.objective[b] == d.objective
            assert (r.iterations[b], r.objective_evals[b], bool(r.converged[b])) == \
                (d.iterations, d.objective_evals, d.converged)


def test_fp32_invalid_inputs_flagged():
    X = np.ones((3, 6, 2), np.float32)
    X[1, 2, 1] = np.nan
    Y = np.arange(18, dtype=np.float32).reshape(3, 6)
    L = np.array([0.1, 0.1, -1.0], np.float32)
    r = lad.solve_locus_batched(X, Y, L)
    assert list(r.status) == [0, 2, 2]


def test_fp32_peak_probe():
    assert lad.solver.fp32_peak_tflops() > lad.solver.fp64_peak_tflops() > 1.0
