"""LP recasting + dense simplex against the reference's lp.py.

Goldens: tests/golden/lp.npz (oracle/gen_golden.py gen_lp) from the unmodified reference:
240 problems (m 2..32, d 1..8, both pivot rules, pivot budgets) with solve_lp's beta and
objective and simplex_minimize's primal point, basis, pivots and objective trace; dump_lp text.
CPU tests pin the oracle and the host-side formulation; GPU tests pin the kernel, bit for bit.
"""

import numpy as np
import pytest

from conftest import load_golden
from paper_2510_15649_b200 import lp as LP
from paper_2510_15649_b200.errors import InvalidInputError
from paper_2510_15649_b200.solver import Dataset, ProblemSpec


def _case(g, i):
    m, d = int(g["m"][i]), int(g["d"][i])
    return m, d, g["x"][i, :m, :d], g["y"][i, :m], float(g["lam"][i])


def _cfg(g, i):
    mp = int(g["max_pivots"][i])
    return dict(max_pivots=mp or None, pivot_rule="bland" if g["rule"][i] else "dantzig_with_bland_fallback")


def test_oracle_lp_matches_reference(oracle):
    g = load_golden("lp")
    for i in range(len(g["lam"])):
        m, d, x, y, lam = _case(g, i)
        c = _cfg(g, i)
        o = oracle.lp_solve(x, y, max(lam, 1e-9), c["max_pivots"], c["pivot_rule"])
        n = 2 * d + 2 * m
        assert np.array_equal(o.x, g["xfull"][i, :n]), i
        assert list(o.basis) == list(g["basis"][i, :m]), i
        assert o.pivots == g["pivots"][i] and o.converged == bool(g["converged"][i]), i
        assert np.array_equal(o.beta, g["beta"][i, :d]) and o.objective == g["objective"][i], i


def test_formulation_host_side():
    """lp.py:82-103 restated; test_lp.py:20-49 properties."""
    spec = ProblemSpec(Dataset(np.array([[1.0]]), np.array([2.0])), 0.5)
    lp = LP.formulate(spec)
    assert list(lp.cost) == [0.5, 0.5, 1.0, 1.0]
    assert lp.constraint_matrix.tolist() == [[1.0, -1.0, 1.0, -1.0]]
    assert list(lp.rhs) == [2.0] and lp.variable_names == ("bp_0", "bn_0", "rp_0", "rn_0")
    rng = np.random.default_rng(0)
    spec = ProblemSpec(Dataset(rng.standard_normal((6, 3)), rng.standard_normal(6)), 0.2)
    lp = LP.formulate(spec)
    for _ in range(10):
        beta = rng.uniform(-5, 5, 3)
        v = LP.embed(lp, beta)
        assert (v >= 0).all() and np.allclose(lp.constraint_matrix @ v, lp.rhs, atol=1e-12)
    basis = LP.initial_basis(lp)
    v0 = LP.embed(lp, np.zeros(3))
    assert set(np.flatnonzero(v0 > 0)) <= set(basis)
    with pytest.raises(InvalidInputError):
        LP.SimplexConfig(max_pivots=0)
    with pytest.raises(InvalidInputError):
        LP.SimplexConfig(pivot_rule="steepest")


def test_dump_lp_bytes(tmp_path):
    g = load_golden("lp")
    for k, text in zip((0, 5), g["dump_text"]):
        spec = ProblemSpec(Dataset(g[f"dump{k}_x"], g[f"dump{k}_y"]), 0.25)
        path = tmp_path / "lp.txt"
        LP.dump_lp(LP.formulate(spec), path)
        assert path.read_text() == str(text)


@pytest.mark.gpu
def test_gpu_lp_batched_matches_reference():
    pytest.importorskip("torch")
    g = load_golden("lp")
    groups = {}
    for i in range(len(g["lam"])):
        groups.setdefault((int(g["m"][i]), int(g["d"][i]), int(g["rule"][i]), int(g["max_pivots"][i])), []).append(i)
    for (m, d, rule, mp), rows in groups.items():
        rows = np.array(rows)
        cfg = LP.SimplexConfig(max_pivots=mp or None, pivot_rule="bland" if rule else "dantzig_with_bland_fallback")
        r = LP.solve_lp_batched(np.ascontiguousarray(g["x"][rows][:, :m, :d]), np.ascontiguousarray(g["y"][rows][:, :m]),
                                g["lam"][rows], cfg, full=True, trace_cap=64)
        n = 2 * d + 2 * m
        assert (r.status == 0).all()
        assert np.array_equal(r.x, g["xfull"][rows][:, :n]), (m, d)
        assert np.array_equal(r.basis, g["basis"][rows][:, :m]), (m, d)
        assert np.array_equal(r.pivots, g["pivots"][rows]) and np.array_equal(r.converged, g["converged"][rows])
        assert np.array_equal(r.beta, g["beta"][rows][:, :d]) and np.array_equal(r.objective, g["objective"][rows])
        for k, i in enumerate(rows):
            nt = int(g["ntrace"][i])
            assert np.array_equal(r.trace[k, :nt], g["trace"][i, :nt]), i


@pytest.mark.gpu
def test_gpu_lp_single_problem_api():
    """test_lp.py:52-124 restated on the GPU mirrors."""
    pytest.importorskip("torch")
    spec = ProblemSpec(Dataset(np.array([[1.0]]), np.array([2.0])), 0.0001)
    res = LP.solve_lp(spec)
    assert res.converged and res.solver_id == "lp" and res.beta.beta[0] == pytest.approx(2.0, abs=1e-9)
    rng = np.random.default_rng(4)
    spec = ProblemSpec(Dataset(rng.standard_normal((10, 3)), rng.standard_normal(10)), 0.1)
    sol = LP.simplex_minimize(LP.formulate(spec))
    assert sol.converged and (np.diff(sol.objective_trace) <= 1e-12).all()
    bp, bn = sol.x[:3], sol.x[3:6]
    assert (np.minimum(bp, bn) == 0).all()
    bl = LP.solve_lp(spec, LP.SimplexConfig(pivot_rule="bland"))
    assert bl.objective == pytest.approx(LP.solve_lp(spec).objective, rel=1e-9)
    short = LP.solve_lp(spec, LP.SimplexConfig(max_pivots=1))
    assert not short.converged
