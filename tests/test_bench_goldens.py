"""The bench's ACTUAL inputs against the unmodified reference (CPU side).

tests/golden/bench_cfg*.npz hold problems produced by the host restatement of
the device generator (oracle/gen_host.c, byte-identical to lad_generate_f64 --
tests/test_gpu_generator.py) at bench.py's seeds and block offsets, and the
outputs of the reference's own solve_locus / solve_brute on them
(oracle/gen_golden.py gen_bench).  Here: the host generator still reproduces
those inputs, and the oracle reproduces the reference bit for bit on them.
objective.npz pins model.evaluate_objective (model.py:151-154) for every
p <= 8 and row counts up to 1023 (numpy's pairwise recursion above 128 terms).
"""

import numpy as np
import pytest

from conftest import load_golden
from parity import locus_report

BENCH = [("bench_cfg0", 0, ("ternary", "quadrature")), ("bench_cfg1", 1, ("ternary", "quadrature")),
         ("bench_cfg2", 2, ("ternary", "quadrature")), ("bench_cfg3", 3, ("quadrature",)),
         ("bench_cfg4", 4, ("ternary",))]


def _inputs(oracle, g, config):
    """Regenerate the fixture's inputs with the host generator (the bench's recipe)."""
    seed = int(g["seed"])
    if config in (0, 4):
        return oracle.generate(config, len(g["lam"]), seed, int(g["first"]))
    if config == 1:
        parts = [oracle.generate(1, 1, seed, int(i)) for i in g["problem_index"]]
        return tuple(np.concatenate([p[k] for p in parts]) for k in range(3))
    if config == 2:
        X = np.concatenate([oracle.generate(2, 1, seed, int(f))[0] for f in g["dataset_index"]])
        Y = np.concatenate([oracle.generate(2, 1, seed, int(f))[1] for f in g["dataset_index"]])
        return np.repeat(X, 16, axis=0), np.repeat(Y, 16, axis=0), g["lam"]
    X0, Y0 = oracle.config3_dataset(seed)
    assert np.array_equal(X0, g["dataset_x"]) and np.array_equal(Y0, g["dataset_y"])
    Xs = np.concatenate([oracle.subsets(X0, Y0, 25, int(k), 1)[0] for k in g["subset_index"]])
    Ys = np.concatenate([oracle.subsets(X0, Y0, 25, int(k), 1)[1] for k in g["subset_index"]])
    return Xs, Ys, g["lam"]


@pytest.mark.parametrize("name,config,variants", BENCH)
def test_host_generator_reproduces_fixture_inputs(oracle, name, config, variants):
    g = load_golden(name)
    X, Y, L = _inputs(oracle, g, config)
    assert np.array_equal(X.view(np.uint64), g["x"].view(np.uint64))
    assert np.array_equal(Y.view(np.uint64), g["y"].view(np.uint64))
    assert np.array_equal(np.asarray(L, float), g["lam"])


@pytest.mark.parametrize("name,config,variants", BENCH)
def test_oracle_matches_reference_on_bench_inputs(oracle, name, config, variants):
    g = load_golden(name)
    B = len(g["lam"])
    for v in variants:
        r = oracle.solve_locus_batch(g["x"], g["y"], g["lam"], outer_search=v)
        rep = locus_report(r["beta"], r["objective"], g[f"{v}_beta"], g[f"{v}_objective"],
                           {"iterations": r["iterations"], "objective_evals": r["objective_evals"],
                            "D": r["descents"], "S": r["steps"]},
                           {k: g[f"{v}_{k}"] for k in ("iterations", "objective_evals", "D", "S")})
        assert rep["exact"] == B and rep["S_equal"] == B and rep["D_equal"] == B, (name, v, rep)
        assert np.array_equal(r["converged"], g[f"{v}_converged"])
    if "brute_idx" in g:
        for j, i in enumerate(g["brute_idx"]):
            beta, obj, nv = oracle.solve_brute(g["x"][i], g["y"][i], max(float(g["lam"][i]), 1e-9))
            assert obj == g["brute_objective"][j] and np.array_equal(beta, g["brute_beta"][j])


def test_bench_fixture_distributions():
    """The fixtures carry the BASELINE config distributions (sanity, not parity)."""
    g0 = load_golden("bench_cfg0")
    assert g0["x"].shape[1:] == (30, 5) and np.all(g0["lam"] == 1.0)
    assert np.all((np.abs(g0["beta_true"]) > 0).sum(axis=1) == 2)
    g1 = load_golden("bench_cfg1")
    assert g1["x"].shape[1:] == (10, 2) and np.all(np.abs(g1["x"]) < 1) and np.all((g1["lam"] >= 0.1) & (g1["lam"] < 2))
    g4 = load_golden("bench_cfg4")
    assert g4["x"].shape[1:] == (31, 8) and np.all((np.abs(g4["beta_true"]) > 0).sum(axis=1) == 3)


def test_oracle_objective_matches_reference(oracle):
    g = load_golden("objective")
    for m, d in g["shapes"]:
        X, Y, b, lam = g[f"x_{m}_{d}"], g[f"y_{m}_{d}"], g[f"beta_{m}_{d}"], g[f"lam_{m}_{d}"]
        got = np.array([oracle.objective(X[i], Y[i], max(float(lam[i]), 1e-9), b[i]) for i in range(len(lam))])
        assert np.array_equal(got, g[f"objective_{m}_{d}"]), (m, d)


@pytest.mark.parametrize("variant", ["ternary", "quadrature"])
def test_oracle_warm_path_matches_reference(oracle, variant):
    """The warm-started lambda path (paper_2510_15649_b200/path.py's rule, every stage a reference
    solve_locus with initial_bracket) replayed on the oracle == the reference (warm_path.npz)."""
    g = load_golden("warm_path")
    X = np.concatenate([oracle.generate(2, 1, int(g["seed"]), int(f))[0] for f in g["dataset_index"]])
    assert np.array_equal(X, g["x"])
    r = oracle.solve_warm_path(g["x"], g["y"], g["lambdas"], outer_search=variant, nthreads=4)
    assert np.array_equal(r["beta"], g[f"{variant}_beta"])
    assert np.array_equal(r["objective"], g[f"{variant}_objective"])
    assert np.array_equal(r["iterations"], g[f"{variant}_iterations"])
    assert np.array_equal(r["objective_evals"], g[f"{variant}_objective_evals"])
    assert np.array_equal(r["converged"], g[f"{variant}_converged"])


def test_oracle_per_problem_brackets_equal_single_solves(oracle):
    g = load_golden("bench_cfg0")
    X, Y, L = g["x"][:6], g["y"][:6], g["lam"][:6]
    bk = np.array([[-3.0, 3.0], [-1.0, 2.0], [-0.5, 0.5], [2.0, 2.0], [-np.inf, 1.0], [-10.0, 10.0]])
    r = oracle.solve_locus_batch(X, Y, L, brackets=bk, nthreads=2)
    assert list(r["status"]) == [0, 0, 0, 2, 2, 0]
    for i in (0, 1, 2, 5):
        s = oracle.solve_locus(X[i], Y[i], 1.0, initial_bracket=tuple(bk[i]))
        assert s.objective == r["objective"][i] and np.array_equal(s.beta, r["beta"][i])
