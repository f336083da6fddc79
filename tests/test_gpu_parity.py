"""GPU parity: the CUDA path (through the C ABI) against the reference goldens and the CPU oracle.

Bar: bit-exact beta and objective, identical iterations / objective_evals /
converged, and identical work counters (D descents, S coordinate steps) --
strictly stronger than the north-star contract (objective within 1e-9 rel,
same support, beta within 1e-6), which `locus_report` also records.
"""

import numpy as np
import pytest

from conftest import load_golden
from parity import locus_report

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_15649_b200 as lad  # noqa: E402
from paper_2510_15649_b200 import configgen as G  # noqa: E402


def _np(a):
    return a.cpu().numpy() if torch.is_tensor(a) else np.asarray(a)


def _locus_groups(g, variant, cfg_kw=None):
    """Run the GPU solver on a padded golden fixture, grouping rows by (m, d)."""
    B = len(g["lam"])
    ms = g["m"] if "m" in g else np.full(B, g["x"].shape[1])
    ds = g["d"] if "d" in g else np.full(B, g["x"].shape[2])
    Dx = g["x"].shape[2]
    out = dict(beta=np.full((B, Dx), np.nan), objective=np.zeros(B), iterations=np.zeros(B, int),
               objective_evals=np.zeros(B, int), converged=np.zeros(B, bool), D=np.zeros(B, int), S=np.zeros(B, int))
    for (m, d) in sorted(set(zip(ms.tolist(), ds.tolist()))):
        rows = np.nonzero((ms == m) & (ds == d))[0]
        X = np.ascontiguousarray(g["x"][rows][:, :m, :d])
        Y = np.ascontiguousarray(g["y"][rows][:, :m])
        r = lad.solve_locus_batched(X, Y, g["lam"][rows], lad.LocusConfig(outer_search=variant, **(cfg_kw or {})))
        assert (r.status == 0).all()
        out["beta"][rows, :d] = r.beta
        out["objective"][rows] = r.objective
        out["iterations"][rows] = r.iterations
        out["objective_evals"][rows] = r.objective_evals
        out["converged"][rows] = r.converged
        out["D"][rows] = r.descents
        out["S"][rows] = r.steps
    return out


def _assert_exact(r, g, prefix, n=None):
    ref = {k: g[f"{prefix}_{k}"] for k in ("iterations", "objective_evals", "D", "S")}
    rep = locus_report(r["beta"], r["objective"], g[f"{prefix}_beta"], g[f"{prefix}_objective"],
                       {k: r[k] for k in ref}, ref)
    n = rep["n"]
    assert rep["exact"] == n, rep
    for k in ("iterations", "objective_evals", "D", "S"):
        assert rep[f"{k}_equal"] == n, rep
    assert np.array_equal(np.asarray(r["converged"], bool), g[f"{prefix}_converged"].astype(bool))
    return rep


def test_library_loads_and_reports_version():
    from paper_2510_15649_b200 import _lib

    L = _lib.load()
    assert L.lad_version() >= 100


def test_ccd_descend_golden_bit_exact():
    g = load_golden("ccd_cases")
    for i in range(len(g["m"])):
        m, d = int(g["m"][i]), int(g["d"][i])
        fr = int(g["frozen"][i])
        cfg = lad.CcdConfig(sweep_tolerance=float(g["tol"][i]), max_sweeps=int(g["sweeps"][i]))
        r = lad.ccd_descend_batched(g["x"][i, :m, :d][None], g["y"][i, :m][None], np.array([g["lam"][i]]),
                                    g["start"][i, :d][None], cfg, frozen=None if fr < 0 else fr)
        assert np.array_equal(r.beta[0], g["beta"][i, :d]), i
        assert r.objective[0] == g["objective"][i], i
        assert r.iterations[0] == g["iterations"][i] and r.objective_evals[0] == g["objective_evals"][i], i
        assert bool(r.converged[0]) == bool(g["converged"][i]), i


@pytest.mark.parametrize("variant", ["ternary", "quadrature"])
def test_acceptance_grid_bit_exact(variant):
    g = load_golden("acceptance")
    r = _locus_groups(g, variant)
    _assert_exact(r, g, variant)
    gap = (r["objective"] - g["brute_objective"]) / np.abs(g["brute_objective"])
    assert gap.max() < 1e-5  # acceptance criterion 1


def test_locus_config_knobs_bit_exact():
    g = load_golden("params")
    for i in range(len(g["lam"])):
        m, d = int(g["m"][i]), int(g["d"][i])
        cfg = lad.LocusConfig(
            outer_search=("ternary", "quadrature")[int(g["outer_search"][i])],
            outer_axis=None if g["outer_axis"][i] < 0 else int(g["outer_axis"][i]),
            initial_bracket=lad.Bracket(*g["bracket"][i]) if g["has_bracket"][i] else None,
            outer_probes=int(g["outer_probes"][i]), outer_tolerance=float(g["outer_tolerance"][i]),
            outer_max_iterations=int(g["outer_max_iterations"][i]),
            inner=lad.CcdConfig(max_sweeps=int(g["inner_sweeps"][i]), sweep_tolerance=float(g["inner_tol"][i])))
        r = lad.solve_locus_batched(g["x"][i, :m, :d][None], g["y"][i, :m][None], np.array([g["lam"][i]]), cfg)
        assert r.objective[0] == g["objective"][i], i
        assert np.array_equal(r.beta[0], g["beta"][i, :d]), i
        assert r.iterations[0] == g["iterations"][i] and r.objective_evals[0] == g["objective_evals"][i], i
        assert bool(r.converged[0]) == bool(g["converged"][i]), i
        assert r.descents[0] == g["D"][i] and r.steps[0] == g["S"][i], i


@pytest.mark.parametrize("name,variants", [("cfg0", ("ternary", "quadrature")), ("cfg1", ("ternary", "quadrature")),
                                           ("cfg2", ("ternary", "quadrature")), ("cfg3", ("quadrature",)),
                                           ("cfg4", ("ternary",))])
def test_config_goldens_bit_exact(name, variants):
    g = load_golden(name)
    for v in variants:
        r = lad.solve_locus_batched(g["x"], g["y"], g["lam"], lad.LocusConfig(outer_search=v))
        assert (r.status == 0).all()
        rr = dict(beta=r.beta, objective=r.objective, iterations=r.iterations, objective_evals=r.objective_evals,
                  converged=r.converged, D=r.descents, S=r.steps)
        _assert_exact(rr, g, v)


def test_config_goldens_device_path_matches_host_path():
    g = load_golden("cfg0")
    X = torch.from_numpy(g["x"]).cuda()
    Y = torch.from_numpy(g["y"]).cuda()
    L = torch.from_numpy(g["lam"]).cuda()
    r = lad.solve_locus_batched(X, Y, L)
    torch.cuda.synchronize()
    assert np.array_equal(_np(r.beta), g["ternary_beta"])
    assert np.array_equal(_np(r.objective), g["ternary_objective"])


def test_brute_goldens_bit_exact():
    g = load_golden("acceptance")
    ms, ds = g["m"], g["d"]
    for (m, d) in sorted(set(zip(ms.tolist(), ds.tolist()))):
        rows = np.nonzero((ms == m) & (ds == d))[0]
        beta, obj, nv = lad.solve_brute_batched(np.ascontiguousarray(g["x"][rows][:, :m, :d]),
                                                np.ascontiguousarray(g["y"][rows][:, :m]), g["lam"][rows])
        assert np.array_equal(obj, g["brute_objective"][rows])
        assert np.array_equal(beta, g["brute_beta"][rows][:, :d])
        assert np.array_equal(nv, g["brute_vertices"][rows])
    for name in ("cfg0", "cfg1", "cfg2", "cfg3"):
        g = load_golden(name)
        idx = g["brute_idx"]
        beta, obj, nv = lad.solve_brute_batched(g["x"][idx], g["y"][idx], g["lam"][idx])
        assert np.array_equal(obj, g["brute_objective"]), name
        assert np.array_equal(beta, g["brute_beta"]), name
        assert np.array_equal(nv, g["brute_vertices"]), name


def test_brute_caps_raise_like_reference():
    x = np.random.default_rng(0).standard_normal((1, 6, 2))
    y = np.zeros((1, 6))
    with pytest.raises(lad.ProblemTooLargeError):
        lad.solve_brute_batched(x, y, [0.1], max_variables=1)
    with pytest.raises(lad.ProblemTooLargeError):
        lad.solve_brute_batched(x, y, [0.1], max_candidates=5)


def test_single_problem_kats():
    # test_brute.py:78-86 and fixtures.py:15-20 through the drop-in single-problem API
    spec = lad.ProblemSpec(lad.Dataset([[1.0]], [2.0]), 0.5)
    res = lad.solve_brute(spec)
    assert res.beta.beta[0] == 2.0 and res.objective == 1.0
    spec = lad.ProblemSpec(lad.Dataset([[1.0]], [2.0]), 1.5)
    res = lad.solve_brute(spec)
    assert res.beta.beta[0] == 0.0 and res.objective == 2.0
    k = load_golden("kat")
    spec = lad.ProblemSpec(lad.Dataset(k["stall_x"], k["stall_y"]), float(k["stall_lam"]))
    plain = lad.solve_ccd(spec)
    assert plain.converged and plain.objective == 41.69174235002273
    assert lad.solve_brute(spec).objective == 41.437510830005365
    res = lad.solve_locus(spec)
    assert abs(res.objective - 41.437510830005365) / 41.437510830005365 < 1e-5


def test_edge_cases(oracle):
    rng = np.random.default_rng(5)
    # empty batch
    r = lad.solve_locus_batched(np.zeros((0, 5, 2)), np.zeros((0, 5)), np.zeros(0))
    assert r.beta.shape == (0, 2)
    # non-finite input -> per-problem status 2, the rest of the batch is solved
    X = rng.standard_normal((3, 6, 2))
    Y = rng.standard_normal((3, 6))
    X[1, 2, 0] = np.nan
    r = lad.solve_locus_batched(X, Y, np.full(3, 0.1))
    assert list(r.status) == [0, 2, 0]
    with pytest.raises(lad.InvalidInputError):
        lad.solve_locus_batched(X, Y, np.full(3, 0.1), strict=True)
    # zero columns / exact zeros (sparse path), n = 1, p = 1, lambda = 0 (floor)
    cases = [np.diag([1.0, -2.0, 0.5]), np.array([[1.0]]), rng.standard_normal((7, 1)),
             np.where(rng.random((9, 3)) < 0.3, 0.0, rng.standard_normal((9, 3))),
             np.hstack([rng.standard_normal((8, 1)), np.zeros((8, 1))])]
    for x in cases:
        y = rng.standard_normal(x.shape[0])
        for lam in (0.0, 0.05, 1.0):
            for v in ("ternary", "quadrature"):
                r = lad.solve_locus_batched(x[None], y[None], np.array([lam]), lad.LocusConfig(outer_search=v))
                o = oracle.solve_locus(x, y, max(lam, 1e-9), outer_search=v)
                assert r.objective[0] == o.objective and np.array_equal(r.beta[0], o.beta), (x.shape, lam, v)
                assert r.descents[0] == o.descents and r.steps[0] == o.steps


@pytest.mark.parametrize("policy", ["thread", "warp"])
def test_data_index_out_of_range_is_per_problem_invalid(policy):
    """Device data_index is bounds-checked in the kernel (no host sync): bad rows get status 2."""
    from paper_2510_15649_b200 import _lib

    g = load_golden("cfg1" if policy == "thread" else "cfg0")
    X = torch.from_numpy(g["x"][:4]).cuda()
    Y = torch.from_numpy(g["y"][:4]).cuda()
    idx = torch.tensor([0, 3, -1, 4, 2, 1 << 40], device="cuda")
    L = torch.from_numpy(np.repeat(g["lam"][:1], 6)).cuda()
    _lib.set_kernel_policy({"thread": _lib.KERNEL_THREAD, "warp": _lib.KERNEL_WARP}[policy])
    try:
        r = lad.solve_locus_batched(X, Y, L, data_index=idx)
        torch.cuda.synchronize()
    finally:
        _lib.set_kernel_policy(_lib.KERNEL_AUTO)
    assert _np(r.status).tolist() == [0, 0, 2, 2, 0, 2]
    ref = lad.solve_locus_batched(g["x"][[0, 3, 2]], g["y"][[0, 3, 2]], np.repeat(g["lam"][:1], 3))
    assert np.array_equal(_np(r.objective)[[0, 1, 4]], ref.objective)
    with pytest.raises(lad.InvalidInputError):
        lad.solve_locus_batched(X, Y, L, data_index=idx, strict=True)


@pytest.mark.parametrize("axis_parallel", [True, False])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_extreme_magnitudes_bit_exact(oracle, dtype, axis_parallel):
    """Values outside the reciprocal-division range (|v| < 2^-450 or > 2^450 in binary64,
    2^+-50 in binary32) take the generic division: whole problems scaled up, single columns
    and single entries scaled down.  Rows exactly on the fit (residual 0) take the signed-zero
    branch.  Solved problems must equal the oracle bit for bit; problems where the reference
    raises UnboundedDirectionError (a huge column collapses the default bracket) must report
    status 1 like the oracle."""
    rng = np.random.default_rng(17)
    big, small = (1e140, 1e-140) if dtype == np.float64 else (1e16, 1e-16)
    for (n, p) in ((30, 5), (12, 3), (31, 8)):
        B = 15
        X = rng.standard_normal((B, n, p))
        beta = np.zeros(p)
        beta[0] = 2.0
        Y = X @ beta
        Y[:, ::4] += rng.laplace(0, 0.5, (B, (n + 3) // 4))  # most rows exactly on the fit: r == 0
        X[0::5, :, 1] *= small          # tiny column
        X[1::5, :, p - 1] *= big        # huge column (the reference reports an unbounded direction)
        X[2::5, 3, 0] = small * 0.5     # one tiny entry
        X[3::5] *= big                  # whole problem scaled up: every residual out of range
        Y[3::5] *= big
        X, Y = X.astype(dtype), Y.astype(dtype)
        L = np.full(B, 0.2, dtype)
        from paper_2510_15649_b200 import _lib

        _lib.set_axis_parallel(axis_parallel)
        try:
            r = lad.solve_locus_batched(X, Y, L)
        finally:
            _lib.set_axis_parallel(True)
        o = oracle.solve_locus_batch(X, Y, L)
        assert np.array_equal(r.status, o["status"]), (n, p, r.status, o["status"])
        # the work done up to the failing axis is the same as well
        assert np.array_equal(r.steps, o["steps"]) and np.array_equal(r.descents, o["descents"])
        ok = np.asarray(o["status"]) == 0
        assert ok.sum() >= 12
        assert np.array_equal(r.beta[ok], o["beta"][ok]) and np.array_equal(r.objective[ok], o["objective"][ok])
        assert np.array_equal(r.steps[ok], o["steps"][ok]) and np.array_equal(r.descents[ok], o["descents"][ok])


def test_device_generated_config2_against_oracle(oracle):
    """Config 2 shape at scale: device-generated bytes copied back, oracle on a sample."""
    X, Y, _ = G.generate(2, 512, seed=2024)
    lam_grid = torch.tensor(G.LAMBDA_GRID, dtype=torch.float64, device="cuda")
    B = 512 * 16
    data_index = torch.arange(512, device="cuda").repeat_interleave(16)
    lam = lam_grid.repeat(512)
    for v in ("ternary", "quadrature"):
        r = lad.solve_locus_batched(X, Y, lam, lad.LocusConfig(outer_search=v), data_index=data_index)
        torch.cuda.synchronize()
        sample = np.arange(0, B, 41)
        Xh, Yh = _np(X), _np(Y)
        o = oracle.solve_locus_batch(Xh[sample // 16], Yh[sample // 16], _np(lam)[sample], outer_search=v)
        assert np.array_equal(_np(r.objective)[sample], o["objective"]), v
        assert np.array_equal(_np(r.beta)[sample], o["beta"]), v
        assert np.array_equal(_np(r.steps)[sample], o["steps"]), v


def test_device_generated_config1_locus_matches_brute():
    """Config 1 property at scale: locus objective within 1e-9 of the brute-force optimum."""
    X, Y, L = G.generate(1, 1 << 16, seed=77)
    r = lad.solve_locus_batched(X, Y, L)
    _, obj, nv = lad.solve_brute_batched(X, Y, L)
    gap = ((r.objective - obj) / obj.abs()).cpu().numpy()
    assert (gap >= -1e-12).all()
    assert (gap <= 1e-9).mean() > 0.999
    assert (nv.cpu().numpy() <= 66).all()


def test_device_generated_subsets_match_host_combinations():
    import itertools

    X0, Y0 = G.config3_dataset()
    ks = [0, 1, 17, 142505]
    for k in ks:
        Xs, Ys = G.subsets(X0, Y0, 25, k, 1)
        rows = list(itertools.combinations(range(30), 25))[k]
        assert torch.equal(Xs[0], X0[list(rows)]) and torch.equal(Ys[0], Y0[list(rows)])


@pytest.mark.parametrize("policy", ["thread", "warp"])
def test_both_kernel_mappings_bit_exact(policy):
    """The thread-per-problem and warp-per-problem kernels both reproduce the reference."""
    from paper_2510_15649_b200 import _lib

    _lib.set_kernel_policy(_lib.KERNEL_THREAD if policy == "thread" else _lib.KERNEL_WARP)
    try:
        g = load_golden("acceptance")
        for v in ("ternary", "quadrature"):
            _assert_exact(_locus_groups(g, v), g, v)
        for name, v in (("cfg0", "ternary"), ("cfg1", "quadrature"), ("cfg3", "quadrature"), ("cfg4", "ternary")):
            g = load_golden(name)
            idx = np.arange(0, len(g["lam"]), 4)
            r = lad.solve_locus_batched(g["x"][idx], g["y"][idx], g["lam"][idx], lad.LocusConfig(outer_search=v))
            sub = {k: (g[k][idx] if g[k].shape[:1] == g["lam"].shape else g[k]) for k in g}
            rr = dict(beta=r.beta, objective=r.objective, iterations=r.iterations, objective_evals=r.objective_evals,
                      converged=r.converged, D=r.descents, S=r.steps)
            _assert_exact(rr, sub, v)
        g = load_golden("params")
        for i in range(len(g["lam"])):
            m, d = int(g["m"][i]), int(g["d"][i])
            cfg = lad.LocusConfig(
                outer_search=("ternary", "quadrature")[int(g["outer_search"][i])],
                outer_axis=None if g["outer_axis"][i] < 0 else int(g["outer_axis"][i]),
                initial_bracket=lad.Bracket(*g["bracket"][i]) if g["has_bracket"][i] else None,
                outer_probes=int(g["outer_probes"][i]), outer_tolerance=float(g["outer_tolerance"][i]),
                outer_max_iterations=int(g["outer_max_iterations"][i]),
                inner=lad.CcdConfig(max_sweeps=int(g["inner_sweeps"][i]), sweep_tolerance=float(g["inner_tol"][i])))
            r = lad.solve_locus_batched(g["x"][i, :m, :d][None], g["y"][i, :m][None], np.array([g["lam"][i]]), cfg)
            assert r.objective[0] == g["objective"][i] and r.steps[0] == g["S"][i], (policy, i)
    finally:
        _lib.set_kernel_policy(_lib.KERNEL_AUTO)


def _oracle_sample_exact(oracle, X, Y, L, r, idx, variant):
    o = oracle.solve_locus_batch(_np(X)[idx], _np(Y)[idx], _np(L)[idx], outer_search=variant)
    assert np.array_equal(_np(r.objective)[idx], o["objective"])
    assert np.array_equal(_np(r.beta)[idx], o["beta"])
    assert np.array_equal(_np(r.steps)[idx], o["steps"])
    assert np.array_equal(_np(r.descents)[idx], o["descents"])
    assert np.array_equal(_np(r.converged)[idx], o["converged"])


def test_config3_all_subsets_against_oracle(oracle):
    """Config 3 in full on the GPU (142,506 subsets, quadrature); oracle on a spread sample."""
    X0, Y0 = G.config3_dataset()
    total = G.CONFIG_BATCH[3]
    Xs, Ys = G.subsets(X0, Y0, 25, 0, total)
    L = torch.full((total,), 0.5, dtype=torch.float64, device="cuda")
    r = lad.solve_locus_batched(Xs, Ys, L, lad.LocusConfig(outer_search="quadrature"))
    torch.cuda.synchronize()
    assert bool((r.status == 0).all())
    idx = np.linspace(0, total - 1, 48).astype(np.int64)
    _oracle_sample_exact(oracle, Xs, Ys, L, r, idx, "quadrature")
    # brute force on two subsets: the reference is best effort at p=5, never below the optimum
    _, opt, _ = lad.solve_brute_batched(_np(Xs)[idx[:2]], _np(Ys)[idx[:2]], _np(L)[idx[:2]])
    assert np.all(_np(r.objective)[idx[:2]] >= opt * (1 - 1e-12))


def test_config4_shard_against_oracle(oracle):
    """Config 4 shape (n=31, p=8, heavy tails) on a device-generated shard; oracle on a sample."""
    X, Y, L = G.generate(4, 4096, seed=404, first=123456)
    r = lad.solve_locus_batched(X, Y, L)
    torch.cuda.synchronize()
    assert bool((r.status == 0).all())
    _oracle_sample_exact(oracle, X, Y, L, r, np.arange(0, 4096, 128), "ternary")


def test_config0_full_batch_against_oracle(oracle):
    """Config 0 in full (B=256) on device-generated data, both variants, all 256 checked."""
    X, Y, L = G.generate(0, 256, seed=15649)
    for v in ("ternary", "quadrature"):
        r = lad.solve_locus_batched(X, Y, L, lad.LocusConfig(outer_search=v))
        torch.cuda.synchronize()
        _oracle_sample_exact(oracle, X, Y, L, r, np.arange(256), v)


@pytest.mark.parametrize("axis_parallel", [False, True])
def test_axis_parallel_small_batch_mode_bit_exact(axis_parallel):
    """Small batches may split each solve into independent per-axis work items
    (locus.py:223-225) recombined in order; both modes must equal the reference."""
    from paper_2510_15649_b200 import _lib

    _lib.set_axis_parallel(axis_parallel)
    try:
        for name, v in (("cfg0", "ternary"), ("cfg0", "quadrature"), ("cfg4", "ternary"), ("cfg2", "ternary")):
            g = load_golden(name)
            r = lad.solve_locus_batched(g["x"], g["y"], g["lam"], lad.LocusConfig(outer_search=v))
            rr = dict(beta=r.beta, objective=r.objective, iterations=r.iterations, objective_evals=r.objective_evals,
                      converged=r.converged, D=r.descents, S=r.steps)
            _assert_exact(rr, g, v)
        g = load_golden("acceptance")
        _assert_exact(_locus_groups(g, "ternary"), g, "ternary")
    finally:
        _lib.set_axis_parallel(True)


def test_generator_shards_are_reproducible():
    """Problem i depends only on (seed, i): shards generated separately equal one big generation."""
    for config in (0, 1, 2, 4):
        Xa, Ya, La = G.generate(config, 300, seed=9, first=1000)
        Xb, Yb, Lb = G.generate(config, 100, seed=9, first=1200)
        assert torch.equal(Xa[200:], Xb) and torch.equal(Ya[200:], Yb) and torch.equal(La[200:], Lb)
