"""Pin the CPU oracle against the reference's own outputs (tests/golden).

The goldens were produced by oracle/gen_golden.py running the unmodified
reference (/root/reference/pkg/src/ladlasso, numpy 2.3.5 + OpenBLAS 0.3.30).
The oracle restates the reference's evaluation order, so everything here is
checked bit-for-bit, counters included.
"""

import numpy as np
import pytest

from conftest import load_golden
from parity import locus_report


def test_pcg32_golden(oracle):
    k = load_golden("kat")
    # test_datagen.py:19-24 first six outputs
    assert oracle.pcg32_sequence(42, 6) == [0xA15C02B7, 0x7B47F409, 0xBA1D3330, 0x83D2F293, 0xBFA4784B, 0xCBED606E]
    assert oracle.pcg32_sequence(42, 200) == k["pcg32_seed42"].tolist()
    for a in range(8):
        assert oracle.pcg32_sequence(0x5EED + a, 64) == k["pcg32_fan"][a].tolist()


def test_weighted_median_kats(oracle):
    k = load_golden("kat")
    for loc, w, t, v, tc in zip(k["median_loc"], k["median_w"], k["median_t"], k["median_v"], k["median_loc_ccd"]):
        n = int(np.sum(~np.isnan(loc)))
        t2, v2 = oracle.weighted_median_min(loc[:n], w[:n])
        assert t2 == t and v2 == v
        assert oracle.median_location(loc[:n], w[:n]) == tc
    # test_linesearch.py:33-54 literal KATs
    assert oracle.weighted_median_min([3.0], [0.7]) == (3.0, 0.0)
    assert oracle.weighted_median_min([1.0, 2.0, 9.0], [1.0, 1.0, 1.0])[0] == 2.0
    assert oracle.weighted_median_min([0.0, 5.0], [10.0, 1.0])[0] == 0.0
    assert oracle.weighted_median_min([0.0, 1.0], [1.0, 1.0])[0] == 0.5


def test_linear_system_kats(oracle):
    k = load_golden("kat")
    for a, b, s, ok in zip(k["ls_a"], k["ls_b"], k["ls_sol"], k["ls_ok"]):
        n = int(np.sum(~np.isnan(b)))
        got = oracle.solve_linear_system(a[:n, :n], b[:n])
        assert (got is not None) == bool(ok)
        if ok:
            assert np.array_equal(got, s[:n])
    assert oracle.solve_linear_system(np.eye(2), [3.0, 4.0]).tolist() == [3.0, 4.0]
    assert oracle.solve_linear_system([[1.0, 1.0], [2.0, 2.0]], [1.0, 2.0]) is None
    assert oracle.solve_linear_system([[0.0, 0.0], [1.0, 2.0]], [0.0, 1.0]) is None


def test_ccd_descend_bit_exact(oracle):
    g = load_golden("ccd_cases")
    for i in range(len(g["m"])):
        m, d = int(g["m"][i]), int(g["d"][i])
        lam = max(float(g["lam"][i]), 1e-9)
        fr = int(g["frozen"][i])
        r = oracle.ccd_descend(g["x"][i, :m, :d], g["y"][i, :m], lam, g["start"][i, :d], None if fr < 0 else fr,
                               float(g["tol"][i]), int(g["sweeps"][i]), trace=True)
        assert np.array_equal(r.beta, g["beta"][i, :d]), i
        assert r.objective == g["objective"][i], i
        assert r.iterations == g["iterations"][i] and r.objective_evals == g["objective_evals"][i], i
        assert r.converged == bool(g["converged"][i]), i
        assert len(r.trace) == g["trace_len"][i]
        assert np.all(np.diff(r.trace) <= 0)  # acceptance criterion 3: monotone descent


def _run_locus_fixture(oracle, g, variant, rows=None, **kw):
    rows = range(len(g["lam"])) if rows is None else rows
    out = dict(beta=[], objective=[], iterations=[], objective_evals=[], converged=[], D=[], S=[])
    for i in rows:
        m = int(g["m"][i]) if "m" in g else g["x"].shape[1]
        d = int(g["d"][i]) if "d" in g else g["x"].shape[2]
        r = oracle.solve_locus(g["x"][i, :m, :d], g["y"][i, :m], max(float(g["lam"][i]), 1e-9),
                               outer_search=variant, **kw)
        b = np.full(g["x"].shape[2], np.nan)
        b[:d] = r.beta
        out["beta"].append(b)
        out["objective"].append(r.objective)
        out["iterations"].append(r.iterations)
        out["objective_evals"].append(r.objective_evals)
        out["converged"].append(r.converged)
        out["D"].append(r.descents)
        out["S"].append(r.steps)
    return {k: np.array(v) for k, v in out.items()}


@pytest.mark.parametrize("variant", ["ternary", "quadrature"])
def test_acceptance_grid_bit_exact(oracle, variant):
    g = load_golden("acceptance")
    r = _run_locus_fixture(oracle, g, variant)
    rep = locus_report(r["beta"], r["objective"], g[f"{variant}_beta"], g[f"{variant}_objective"],
                       {k: r[k] for k in ("iterations", "objective_evals", "D", "S")},
                       {k: g[f"{variant}_{k}"] for k in ("iterations", "objective_evals", "D", "S")})
    n = rep["n"]
    assert rep["exact"] == n, rep
    assert rep["iterations_equal"] == n and rep["objective_evals_equal"] == n, rep
    assert rep["D_equal"] == n and rep["S_equal"] == n, rep
    assert np.array_equal(r["converged"], g[f"{variant}_converged"])
    # acceptance criterion 1 (test_acceptance.py:140-158): within 1e-5 of brute force
    gap = (r["objective"] - g["brute_objective"]) / np.abs(g["brute_objective"])
    assert gap.max() < 1e-5


def test_acceptance_brute_bit_exact(oracle):
    g = load_golden("acceptance")
    for i in range(len(g["lam"])):
        m, d = int(g["m"][i]), int(g["d"][i])
        beta, obj, nv = oracle.solve_brute(g["x"][i, :m, :d], g["y"][i, :m], max(float(g["lam"][i]), 1e-9))
        assert obj == g["brute_objective"][i]
        assert np.array_equal(beta, g["brute_beta"][i, :d])
        assert nv == g["brute_vertices"][i]


def test_locus_config_knobs_bit_exact(oracle):
    g = load_golden("params")
    for i in range(len(g["lam"])):
        m, d = int(g["m"][i]), int(g["d"][i])
        kw = dict(outer_search=("ternary", "quadrature")[int(g["outer_search"][i])],
                  outer_axis=None if g["outer_axis"][i] < 0 else int(g["outer_axis"][i]),
                  initial_bracket=tuple(g["bracket"][i]) if g["has_bracket"][i] else None,
                  outer_probes=int(g["outer_probes"][i]), outer_tolerance=float(g["outer_tolerance"][i]),
                  outer_max_iterations=int(g["outer_max_iterations"][i]),
                  inner_max_sweeps=int(g["inner_sweeps"][i]), inner_sweep_tol=float(g["inner_tol"][i]))
        r = oracle.solve_locus(g["x"][i, :m, :d], g["y"][i, :m], max(float(g["lam"][i]), 1e-9), **kw)
        assert r.objective == g["objective"][i], (i, kw)
        assert np.array_equal(r.beta, g["beta"][i, :d]), (i, kw)
        assert r.iterations == g["iterations"][i] and r.objective_evals == g["objective_evals"][i], (i, kw)
        assert r.converged == bool(g["converged"][i]), (i, kw)
        assert r.descents == g["D"][i] and r.steps == g["S"][i], (i, kw)


def test_stall_fixture(oracle):
    """fixtures.py:15-20: plain CCD stalls at 41.69174235002273, optimum 41.437510830005365."""
    k = load_golden("kat")
    x, y, lam = k["stall_x"], k["stall_y"], float(k["stall_lam"])
    plain = oracle.ccd_descend(x, y, lam, np.zeros(x.shape[1]))
    assert plain.converged and plain.objective == 41.69174235002273
    _, opt, _ = oracle.solve_brute(x, y, lam)
    assert opt == 41.437510830005365
    res = oracle.solve_locus(x, y, lam)
    assert abs(res.objective - opt) / opt < 1e-5


@pytest.mark.parametrize("name,variants", [("cfg0", ("ternary", "quadrature")), ("cfg1", ("ternary", "quadrature")),
                                           ("cfg2", ("ternary", "quadrature")), ("cfg3", ("quadrature",)),
                                           ("cfg4", ("ternary",))])
def test_config_shapes_bit_exact(oracle, name, variants):
    g = load_golden(name)
    B = len(g["lam"])
    for v in variants:
        r = oracle.solve_locus_batch(g["x"], g["y"], g["lam"], outer_search=v)
        rep = locus_report(r["beta"], r["objective"], g[f"{v}_beta"], g[f"{v}_objective"],
                           {"iterations": r["iterations"], "objective_evals": r["objective_evals"],
                            "D": r["descents"], "S": r["steps"]},
                           {k: g[f"{v}_{k}"] for k in ("iterations", "objective_evals", "D", "S")})
        assert rep["exact"] == B, (name, v, rep)
        assert rep["S_equal"] == B and rep["D_equal"] == B, (name, v, rep)
        assert np.array_equal(r["converged"], g[f"{v}_converged"])
    if "brute_idx" in g:
        for j, i in enumerate(g["brute_idx"]):
            beta, obj, nv = oracle.solve_brute(g["x"][i], g["y"][i], max(float(g["lam"][i]), 1e-9))
            assert obj == g["brute_objective"][j] and np.array_equal(beta, g["brute_beta"][j])
            assert nv == g["brute_vertices"][j]


def test_numerics_model_matches_live_numpy():
    """The restated numpy/OpenBLAS orders match this interpreter's numpy (SkylakeX OpenBLAS only)."""
    from oracle import probe_numerics as P

    if P.openblas_arch() != "SkylakeX":
        pytest.skip(f"order model measured for OpenBLAS SkylakeX kernels, host uses {P.openblas_arch()}")
    res = P.check(trials=10)
    assert all(v == 0 for v in res.values()), res


def test_certificate_oracle_matches_reference(oracle):
    """ccd.is_axiswise_minimum (ccd.py:214-237) restated: 360 certified / nudged / random vectors."""
    g = load_golden("curve")
    for i in range(len(g["lam"])):
        m, d = int(g["m"][i]), int(g["d"][i])
        sk = int(g["skip"][i])
        got = oracle.is_axiswise_minimum(g["x"][i, :m, :d], g["y"][i, :m], max(float(g["lam"][i]), 1e-9),
                                         g["beta"][i, :d], None if sk < 0 else sk)
        assert got == bool(g["certified"][i]), i


def test_large_problems_oracle_matches_reference(oracle):
    """m up to 1000 rows: numpy's pairwise-sum recursion (n > 128), OpenBLAS ddot's 32-element
    accumulator blocks (n >= 48) and dgemv_t rows, through ccd_descend and solve_locus."""
    g = load_golden("large")
    for i in range(len(g["ccd_lam"])):
        m, d = int(g["ccd_m"][i]), int(g["ccd_d"][i])
        fr = int(g["ccd_frozen"][i])
        r = oracle.ccd_descend(g["ccd_x"][i, :m, :d], g["ccd_y"][i, :m], max(float(g["ccd_lam"][i]), 1e-9),
                               g["ccd_start"][i, :d], None if fr < 0 else fr)
        assert np.array_equal(r.beta, g["ccd_beta"][i, :d]) and r.objective == g["ccd_objective"][i], i
        assert (r.iterations, r.objective_evals) == (g["ccd_iterations"][i], g["ccd_objective_evals"][i]), i
    for i in range(len(g["locus_lam"])):
        m, d = int(g["locus_m"][i]), int(g["locus_d"][i])
        r = oracle.solve_locus(g["locus_x"][i, :m, :d], g["locus_y"][i, :m], max(float(g["locus_lam"][i]), 1e-9),
                               outer_search="quadrature" if g["locus_variant"][i] else "ternary")
        assert np.array_equal(r.beta, g["locus_beta"][i, :d]) and r.objective == g["locus_objective"][i], i
        assert (r.iterations, r.objective_evals, r.descents, r.steps) == (
            g["locus_iterations"][i], g["locus_objective_evals"][i], g["locus_D"][i], g["locus_S"][i]), i
