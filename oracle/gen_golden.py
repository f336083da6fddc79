"""Generate tests/golden/*.npz by running the UNMODIFIED reference in this container.

TEST INFRASTRUCTURE ONLY.  Requires /root/reference (read-only) importable as
``ladlasso``; it does not exist on the GPU box, so the fixtures are committed
and the tests read only the .npz files.

    python oracle/gen_golden.py [--procs 8]

Every fixture stores the exact input bytes and the reference's outputs
(beta, objective, iterations, objective_evals, converged) plus the work
counters D (ccd_descend calls) and S (coordinate steps) obtained by wrapping
``ladlasso.locus.ccd_descend``.
"""

from __future__ import annotations

import argparse
import itertools
import math
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")
sys.path.insert(0, HERE)
import configs_np  # noqa: E402


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import ladlasso  # noqa: F401

    return ladlasso


def _task(args):
    kind, payload = args
    L = _ref()
    from ladlasso.model import Coefficients, Dataset, ProblemSpec

    x, y, lam = payload["x"], payload["y"], payload["lam"]
    spec = ProblemSpec(Dataset(x, y), lam)
    if kind == "ccd":
        from ladlasso.ccd import CcdConfig, ccd_descend

        trace = []
        r = ccd_descend(spec, Coefficients(payload["start"]),
                        CcdConfig(frozen_axis=payload["frozen"], sweep_tolerance=payload["tol"],
                                  max_sweeps=payload["sweeps"]), trace=trace)
        return dict(beta=r.beta.beta.copy(), objective=r.objective, iterations=r.iterations,
                    objective_evals=r.objective_evals, converged=r.converged, trace_len=len(trace),
                    trace_monotone=bool(np.all(np.diff(np.array(trace)) <= 0)) if len(trace) > 1 else True)
    if kind == "locus":
        import ladlasso.locus as LL
        from ladlasso.ccd import CcdConfig
        from ladlasso.errors import UnboundedDirectionError
        from ladlasso.linesearch import Bracket

        counts = {"D": 0, "S": 0}
        orig = LL.ccd_descend

        def counted(spec_, start, cfg=None, trace=None):
            res = orig(spec_, start, cfg, trace)
            counts["D"] += 1
            counts["S"] += res.objective_evals
            return res

        LL.ccd_descend = counted
        try:
            kw = dict(payload.get("cfg", {}))
            inner = CcdConfig(sweep_tolerance=kw.pop("inner_tol", 1e-10), max_sweeps=kw.pop("inner_sweeps", 500))
            br = kw.pop("bracket", None)
            cfg = LL.LocusConfig(inner=inner, initial_bracket=Bracket(*br) if br is not None else None, **kw)
            t0 = time.perf_counter()
            try:
                r = LL.solve_locus(spec, cfg)
            except UnboundedDirectionError:
                return dict(status=1, D=counts["D"], S=counts["S"])
            wall = time.perf_counter() - t0
        finally:
            LL.ccd_descend = orig
        return dict(beta=r.beta.beta.copy(), objective=r.objective, iterations=r.iterations,
                    objective_evals=r.objective_evals, converged=r.converged, status=0,
                    D=counts["D"], S=counts["S"], wall=wall)
    if kind == "brute":
        from ladlasso.brute import solve_brute
        from ladlasso.errors import ProblemTooLargeError

        try:
            r = solve_brute(spec, **payload.get("caps", {}))
        except ProblemTooLargeError:
            return dict(status=2)
        return dict(beta=r.beta.beta.copy(), objective=r.objective, vertices=r.iterations, status=0)
    raise ValueError(kind)


def _stack(results, d):
    out = {}
    B = len(results)
    out["beta"] = np.array([r.get("beta", np.full(d, np.nan)) for r in results]).reshape(B, d)
    for key in ("objective", "wall"):
        if any(key in r for r in results):
            out[key] = np.array([r.get(key, np.nan) for r in results], dtype=np.float64)
    for key in ("iterations", "objective_evals", "status", "D", "S", "vertices", "trace_len"):
        if any(key in r for r in results):
            out[key] = np.array([r.get(key, -1) for r in results], dtype=np.int64)
    for key in ("converged", "trace_monotone"):
        if any(key in r for r in results):
            out[key] = np.array([bool(r.get(key, False)) for r in results])
    return out


def _run(pool, kind, payloads, d):
    res = pool.map(_task, [(kind, p) for p in payloads], chunksize=1)
    return _stack(res, d)


def gen_kat(pool):
    L = _ref()
    from ladlasso.fixtures import CCD_STALL_LAMBDA, ccd_stall_problem
    from ladlasso.linesearch import PiecewiseLinear1D, weighted_median_min
    from ladlasso.rng import Pcg32

    out = {}
    # PCG32 golden (test_datagen.py:19-24) and a longer stream for the fan seeds
    g42 = Pcg32(42, stream=54)
    out["pcg32_seed42"] = np.array([g42._next_u32() for _ in range(200)], dtype=np.uint32)
    fans = [Pcg32(0x5EED + a) for a in range(8)]
    out["pcg32_fan"] = np.array([[g._next_u32() for _ in range(64)] for g in fans], dtype=np.uint32)
    # weighted-median KATs (test_linesearch.py:33-54) + random cases with ties
    med_loc, med_w, med_t, med_v = [], [], [], []
    rng = np.random.default_rng(1234)
    cases = [([3.0], [0.7]), ([1.0, 2.0, 9.0], [1.0, 1.0, 1.0]), ([0.0, 5.0], [10.0, 1.0]),
             ([0.0, 1.0], [1.0, 1.0])]
    for _ in range(300):
        n = int(rng.integers(1, 33))
        loc = np.round(rng.standard_normal(n) * 3, int(rng.integers(0, 3)))  # rounding -> exact ties
        w = rng.uniform(0.1, 2.0, n)
        if rng.random() < 0.3:
            w = np.round(w * 4) / 4 + 0.25  # dyadic weights -> exact half-sum ties
        cases.append((loc.tolist(), w.tolist()))
    for loc, w in cases:
        g = PiecewiseLinear1D(np.array(loc), np.array(w), 0.0)
        t, v = weighted_median_min(g)
        med_loc.append(np.pad(np.array(loc, float), (0, 33 - len(loc)), constant_values=np.nan))
        med_w.append(np.pad(np.array(w, float), (0, 33 - len(w)), constant_values=np.nan))
        med_t.append(t)
        med_v.append(v)
    out["median_loc"] = np.array(med_loc)
    out["median_w"] = np.array(med_w)
    out["median_t"] = np.array(med_t)
    out["median_v"] = np.array(med_v)
    # ccd._median_location on the same cases (total = cum[-1])
    from ladlasso.ccd import _median_location

    out["median_loc_ccd"] = np.array([_median_location(np.array(l, float), np.array(w, float)) for l, w in cases])
    # stall fixture (fixtures.py:15-20)
    spec = ccd_stall_problem()
    out["stall_x"] = spec.data.x.copy()
    out["stall_y"] = spec.data.y.copy()
    out["stall_lam"] = np.array(CCD_STALL_LAMBDA)
    # linear-system KATs (test_brute.py:17-38) + random systems
    from ladlasso.brute import solve_linear_system

    A, Bv, S, ok = [], [], [], []
    for _ in range(200):
        n = int(rng.integers(1, 7))
        a = rng.uniform(-2, 2, (n, n))
        if rng.random() < 0.15:
            a[int(rng.integers(0, n))] = 0.0
        if rng.random() < 0.15 and n > 1:
            a[1] = a[0] * 2.0
        b = rng.uniform(-2, 2, n)
        s = solve_linear_system(a, b)
        A.append(np.pad(a, ((0, 6 - n), (0, 6 - n)), constant_values=np.nan))
        Bv.append(np.pad(b, (0, 6 - n), constant_values=np.nan))
        S.append(np.pad(s if s is not None else np.full(n, np.nan), (0, 6 - n), constant_values=np.nan))
        ok.append(s is not None)
    out["ls_a"], out["ls_b"], out["ls_sol"], out["ls_ok"] = np.array(A), np.array(Bv), np.array(S), np.array(ok)
    np.savez_compressed(os.path.join(GOLDEN, "kat.npz"), **out)
    print("kat.npz", flush=True)


def gen_ccd(pool):
    rng = np.random.default_rng(4321)
    payloads = []
    for i in range(240):
        m = int(rng.integers(2, 32))
        d = int(rng.integers(1, 9))
        x = rng.standard_normal((m, d))
        if i % 5 == 0:  # sparse columns exercise the zero-row path (ccd.py:167-169, :178-179)
            x[rng.random((m, d)) < 0.3] = 0.0
        y = rng.standard_normal(m) * 3
        lam = float(rng.choice([0.0, 0.01, 0.1, 1.0, 5.0]))
        start = rng.standard_normal(d) * (rng.random() < 0.6)
        frozen = int(rng.integers(-1, d))
        payloads.append(dict(x=x, y=y, lam=lam, start=start, frozen=None if frozen < 0 else frozen,
                             tol=float(rng.choice([1e-10, 1e-7])), sweeps=int(rng.choice([500, 40, 3, 1]))))
    # orthogonal-columns KAT (test_ccd.py:22-36)
    payloads.append(dict(x=np.diag([1.0, -2.0, 0.5]), y=np.array([3.0, 4.0, -1.0]), lam=0.05,
                         start=np.zeros(3), frozen=None, tol=1e-10, sweeps=500))
    res = pool.map(_task, [("ccd", p) for p in payloads], chunksize=4)
    B = len(payloads)
    Mx, Dx = 32, 8
    X = np.full((B, Mx, Dx), np.nan)
    Y = np.full((B, Mx), np.nan)
    out = dict(m=np.array([p["x"].shape[0] for p in payloads]), d=np.array([p["x"].shape[1] for p in payloads]),
               lam=np.array([p["lam"] for p in payloads]),
               frozen=np.array([-1 if p["frozen"] is None else p["frozen"] for p in payloads]),
               tol=np.array([p["tol"] for p in payloads]), sweeps=np.array([p["sweeps"] for p in payloads]))
    S0 = np.full((B, Dx), np.nan)
    for k, p in enumerate(payloads):
        m, d = p["x"].shape
        X[k, :m, :d] = p["x"]
        Y[k, :m] = p["y"]
        S0[k, :d] = p["start"]
    beta = np.full((B, Dx), np.nan)
    for k, r in enumerate(res):
        beta[k, : len(r["beta"])] = r["beta"]
    out.update(x=X, y=Y, start=S0, beta=beta, objective=np.array([r["objective"] for r in res]),
               iterations=np.array([r["iterations"] for r in res]),
               objective_evals=np.array([r["objective_evals"] for r in res]),
               converged=np.array([r["converged"] for r in res]),
               trace_len=np.array([r["trace_len"] for r in res]),
               trace_monotone=np.array([r["trace_monotone"] for r in res]))
    np.savez_compressed(os.path.join(GOLDEN, "ccd_cases.npz"), **out)
    print("ccd_cases.npz", flush=True)


def gen_acceptance(pool):
    """The reference's 200-instance oracle sweep (test_acceptance.py:96-137)."""
    _ref()
    from ladlasso.datagen import GenSpec, generate

    grid = list(itertools.product((1, 2, 3), range(4, 13), (0.01, 0.1, 1.0)))
    probs = []
    for i in range(200):
        d, m, lam = grid[i % len(grid)]
        data, _ = generate(GenSpec(m=m, d=d, noise_sigma=1.0, outlier_fraction=0.2, seed=9000 + i))
        probs.append(dict(x=data.x.copy(), y=data.y.copy(), lam=lam))
    out = {}
    Mx, Dx = 12, 3
    B = len(probs)
    X = np.full((B, Mx, Dx), np.nan)
    Y = np.full((B, Mx), np.nan)
    for k, p in enumerate(probs):
        m, d = p["x"].shape
        X[k, :m, :d] = p["x"]
        Y[k, :m] = p["y"]
    out["x"], out["y"] = X, Y
    out["m"] = np.array([p["x"].shape[0] for p in probs])
    out["d"] = np.array([p["x"].shape[1] for p in probs])
    out["lam"] = np.array([p["lam"] for p in probs])
    for tag, cfg in (("ternary", dict(outer_search="ternary")), ("quadrature", dict(outer_search="quadrature"))):
        r = pool.map(_task, [("locus", dict(p, cfg=cfg)) for p in probs], chunksize=2)
        beta = np.full((B, Dx), np.nan)
        for k, rr in enumerate(r):
            beta[k, : len(rr["beta"])] = rr["beta"]
        st = _stack([dict(rr, beta=np.zeros(1)) for rr in r], 1)
        for key, v in st.items():
            if key != "beta":
                out[f"{tag}_{key}"] = v
        out[f"{tag}_beta"] = beta
    r = pool.map(_task, [("brute", p) for p in probs], chunksize=4)
    beta = np.full((B, Dx), np.nan)
    for k, rr in enumerate(r):
        beta[k, : len(rr["beta"])] = rr["beta"]
    out["brute_beta"] = beta
    out["brute_objective"] = np.array([rr["objective"] for rr in r])
    out["brute_vertices"] = np.array([rr["vertices"] for rr in r])
    np.savez_compressed(os.path.join(GOLDEN, "acceptance.npz"), **out)
    print("acceptance.npz", flush=True)


def gen_params(pool):
    """LocusConfig knobs: outer_axis, initial_bracket, probes, round caps, inner caps."""
    _ref()
    from ladlasso.datagen import GenSpec, generate

    rng = np.random.default_rng(777)
    probs, cfgs = [], []
    for i in range(48):
        d = 1 + i % 4
        m = 5 + i % 8
        data, _ = generate(GenSpec(m=m, d=d, noise_sigma=1.0, outlier_fraction=0.2, seed=7000 + i))
        c = dict(outer_search=("ternary", "quadrature")[i % 2])
        k = i % 6
        if k == 1:
            c["outer_axis"] = int(rng.integers(0, d))
        elif k == 2:
            c["bracket"] = (-0.5, 0.25)
        elif k == 3:
            c["outer_probes"] = 4
            c["outer_tolerance"] = 1e-6
        elif k == 4:
            c["outer_max_iterations"] = 5
        elif k == 5:
            c["inner_sweeps"] = 2
            c["inner_tol"] = 1e-12
        probs.append(dict(x=data.x.copy(), y=data.y.copy(), lam=(0.01, 0.1, 1.0)[i % 3], cfg=c))
        cfgs.append(c)
    r = pool.map(_task, [("locus", p) for p in probs], chunksize=2)
    B, Mx, Dx = len(probs), 12, 4
    X = np.full((B, Mx, Dx), np.nan)
    Y = np.full((B, Mx), np.nan)
    beta = np.full((B, Dx), np.nan)
    for k, p in enumerate(probs):
        m, d = p["x"].shape
        X[k, :m, :d] = p["x"]
        Y[k, :m] = p["y"]
        beta[k, :d] = r[k]["beta"]
    st = _stack([dict(rr, beta=np.zeros(1)) for rr in r], 1)
    out = dict(x=X, y=Y, m=np.array([p["x"].shape[0] for p in probs]), d=np.array([p["x"].shape[1] for p in probs]),
               lam=np.array([p["lam"] for p in probs]), beta=beta,
               outer_search=np.array([0 if c["outer_search"] == "ternary" else 1 for c in cfgs]),
               outer_axis=np.array([c.get("outer_axis", -1) for c in cfgs]),
               has_bracket=np.array([1 if "bracket" in c else 0 for c in cfgs]),
               bracket=np.array([c.get("bracket", (0.0, 0.0)) for c in cfgs], dtype=float),
               outer_probes=np.array([c.get("outer_probes", 8) for c in cfgs]),
               outer_tolerance=np.array([c.get("outer_tolerance", 1e-9) for c in cfgs]),
               outer_max_iterations=np.array([c.get("outer_max_iterations", 200) for c in cfgs]),
               inner_sweeps=np.array([c.get("inner_sweeps", 500) for c in cfgs]),
               inner_tol=np.array([c.get("inner_tol", 1e-10) for c in cfgs]))
    for key, v in st.items():
        if key != "beta":
            out[key] = v
    np.savez_compressed(os.path.join(GOLDEN, "params.npz"), **out)
    print("params.npz", flush=True)


def _locus_fixture(pool, name, X, Y, lam, variants, brute_idx=(), extra=None):
    B, n, p = X.shape
    out = dict(x=X, y=Y, lam=np.broadcast_to(np.asarray(lam, float), (B,)).copy())
    if extra:
        out.update(extra)
    for v in variants:
        t0 = time.time()
        payloads = [dict(x=X[b], y=Y[b], lam=float(out["lam"][b]), cfg=dict(outer_search=v)) for b in range(B)]
        st = _run(pool, "locus", payloads, p)
        for key, val in st.items():
            out[f"{v}_{key}"] = val
        print(f"  {name} {v}: {B} solves in {time.time() - t0:.1f}s", flush=True)
    if len(brute_idx):
        payloads = [dict(x=X[b], y=Y[b], lam=float(out["lam"][b])) for b in brute_idx]
        st = _run(pool, "brute", payloads, p)
        out["brute_idx"] = np.asarray(brute_idx)
        for key, val in st.items():
            out[f"brute_{key}"] = val
    np.savez_compressed(os.path.join(GOLDEN, f"{name}.npz"), **out)
    print(f"{name}.npz", flush=True)


def gen_configs(pool, quick=False):
    rng = np.random.default_rng(15649)
    X, Y, bt = configs_np.cfg0(rng, 32 if quick else 256)
    _locus_fixture(pool, "cfg0", X, Y, 1.0, ("ternary", "quadrature"), brute_idx=range(2 if quick else 8),
                   extra=dict(beta_true=bt))
    rng = np.random.default_rng(15650)
    X, Y, lam = configs_np.cfg1(rng, 64 if quick else 512)
    _locus_fixture(pool, "cfg1", X, Y, lam, ("ternary", "quadrature"), brute_idx=range(X.shape[0]))
    rng = np.random.default_rng(15651)
    X0, Y0, _ = configs_np.cfg0(rng, 8)
    Xr = np.repeat(X0, 16, axis=0)
    Yr = np.repeat(Y0, 16, axis=0)
    lam = np.tile(configs_np.LAMBDA_GRID, 8)
    _locus_fixture(pool, "cfg2", Xr, Yr, lam, ("ternary", "quadrature"), brute_idx=(0, 15))
    rng = np.random.default_rng(15652)
    Xd, Yd, _ = configs_np.cfg0(rng, 1)
    total = math.comb(30, 25)
    ks = np.unique(np.concatenate([np.arange(8), np.linspace(0, total - 1, 40).astype(np.int64)]))
    Xs, Ys = configs_np.cfg3_subsets(Xd[0], Yd[0], ks)
    _locus_fixture(pool, "cfg3", Xs, Ys, 0.5, ("quadrature",), brute_idx=(0, 1),
                   extra=dict(dataset_x=Xd[0], dataset_y=Yd[0], subset_index=ks))
    rng = np.random.default_rng(15653)
    X, Y, bt = configs_np.cfg4(rng, 8 if quick else 32)
    _locus_fixture(pool, "cfg4", X, Y, 1.0, ("ternary",), extra=dict(beta_true=bt))


def gen_bench(pool, quick=False):
    """The bench's ACTUAL inputs (bench.py seeds and block offsets, produced by the host
    restatement of the device generator, oracle/gen_host.c, which tests/test_gpu_generator.py
    pins byte-for-byte to lad_generate_f64) solved by the unmodified reference."""
    import oracle as O  # oracle/oracle.py (this directory is on sys.path)

    O.build()
    k = 4 if quick else 1
    # config 0: bench step 0 is problems [0, 256) of seed 15649, ternary
    X, Y, lam, bt = O.generate(0, 256 // k, 15649, 0, with_beta=True)
    _locus_fixture(pool, "bench_cfg0", X, Y, lam, ("ternary", "quadrature"), brute_idx=range(2),
                   extra=dict(beta_true=bt, seed=15649, first=0))
    # config 1: problems of the first and of a late bench step (seed 15650), both variants + brute
    X1, Y1, L1 = O.generate(1, 192 // k, 15650, 0)
    X2, Y2, L2 = O.generate(1, 64 // k, 15650, 7 << 20)
    X, Y, lam = np.concatenate([X1, X2]), np.concatenate([Y1, Y2]), np.concatenate([L1, L2])
    index = np.concatenate([np.arange(len(L1)), (7 << 20) + np.arange(len(L2))])
    _locus_fixture(pool, "bench_cfg1", X, Y, lam, ("ternary", "quadrature"), brute_idx=range(len(lam)),
                   extra=dict(seed=15650, problem_index=index))
    # config 2: datasets of the first and the last bench block (16384 datasets each), all 16 lambdas
    firsts = [0, 63 * 16384] if quick else [*range(8), *range(63 * 16384, 63 * 16384 + 4), 64 * 16384 - 4, 64 * 16384 - 3, 64 * 16384 - 2, 64 * 16384 - 1]
    Xd = np.concatenate([O.generate(2, 1, 15651, f)[0] for f in firsts])
    Yd = np.concatenate([O.generate(2, 1, 15651, f)[1] for f in firsts])
    Xr, Yr = np.repeat(Xd, 16, axis=0), np.repeat(Yd, 16, axis=0)
    lam = np.tile(configs_np.LAMBDA_GRID, len(firsts))
    _locus_fixture(pool, "bench_cfg2", Xr, Yr, lam, ("ternary", "quadrature"),
                   extra=dict(seed=15651, dataset_index=np.asarray(firsts)))
    # config 3: the bench's dataset (seed 15652, problem 0) and subsets spread over all 142,506
    X0, Y0 = O.config3_dataset(15652)
    total = math.comb(30, 25)
    ks = np.unique(np.concatenate([np.arange(4), np.linspace(0, total - 1, 44 // k).astype(np.int64)]))
    Xs = np.concatenate([O.subsets(X0, Y0, 25, int(q), 1)[0] for q in ks])
    Ys = np.concatenate([O.subsets(X0, Y0, 25, int(q), 1)[1] for q in ks])
    _locus_fixture(pool, "bench_cfg3", Xs, Ys, 0.5, ("quadrature",), brute_idx=(0,),
                   extra=dict(dataset_x=X0, dataset_y=Y0, subset_index=ks, seed=15652))
    # config 4: bench step 0 problems (seed 15653), ternary
    X, Y, lam, bt = O.generate(4, 64 // k, 15653, 0, with_beta=True)
    _locus_fixture(pool, "bench_cfg4", X, Y, lam, ("ternary",), extra=dict(beta_true=bt, seed=15653, first=0))


def _warm_task(args):
    """One dataset's warm lambda path on the reference (the rule of paper_2510_15649_b200/path.py)."""
    L = _ref()
    import ladlasso.locus as LL
    from ladlasso.linesearch import Bracket
    from ladlasso.model import Dataset, ProblemSpec

    x, y, lams, variant = args
    res = [None] * len(lams)
    prev = None
    for k in np.argsort(-np.asarray(lams), kind="stable"):
        br = None
        if prev is not None:
            R = max(1.0, 2.0 * float(np.abs(prev).max()))
            br = Bracket(-R, R)
        r = LL.solve_locus(ProblemSpec(Dataset(x, y), float(lams[k])),
                           LL.LocusConfig(outer_search=variant, initial_bracket=br))
        res[k] = (r.beta.beta.copy(), r.objective, r.iterations, r.objective_evals, r.converged)
        prev = r.beta.beta
    return res


def gen_warm(pool):
    """The warm-started lambda path (bench.py --warm) on bench config-2 datasets, both variants."""
    import oracle as O

    O.build()
    firsts = [0, 1, 2, 63 * 16384 + 5]
    X = np.concatenate([O.generate(2, 1, 15651, f)[0] for f in firsts])
    Y = np.concatenate([O.generate(2, 1, 15651, f)[1] for f in firsts])
    lams = configs_np.LAMBDA_GRID
    out = dict(x=X, y=Y, lambdas=lams, dataset_index=np.asarray(firsts), seed=15651)
    for v in ("ternary", "quadrature"):
        t0 = time.time()
        rs = pool.map(_warm_task, [(X[b], Y[b], lams, v) for b in range(len(firsts))], chunksize=1)
        out[f"{v}_beta"] = np.array([[q[0] for q in r] for r in rs])
        out[f"{v}_objective"] = np.array([[q[1] for q in r] for r in rs])
        out[f"{v}_iterations"] = np.array([[q[2] for q in r] for r in rs])
        out[f"{v}_objective_evals"] = np.array([[q[3] for q in r] for r in rs])
        out[f"{v}_converged"] = np.array([[q[4] for q in r] for r in rs])
        print(f"  warm {v}: {len(firsts)} datasets x {len(lams)} lambdas in {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(GOLDEN, "warm_path.npz"), **out)
    print("warm_path.npz", flush=True)


def gen_genspec(pool):
    """datagen.generate (datagen.py:63-80) on specs beyond the acceptance grid: up to 1000 rows,
    d = 8, informative subsets, fixed true coefficients, sigma 0, odd draw counts (the Box-Muller
    spare crossing phases), large seeds."""
    _ref()
    from ladlasso.datagen import GenSpec, generate

    rng = np.random.default_rng(2510)
    specs = []
    for k in range(40):
        m = int(rng.choice([1, 3, 7, 30, 31, 64, 129, 300, 1000]))
        d = int(rng.integers(1, 9))
        has_truth = k % 5 == 3
        truth = tuple(float(v) for v in rng.standard_normal(d)) if has_truth else None
        specs.append(dict(m=m, d=d, n_informative=int(rng.integers(1, d + 1)), true_coefficients=truth,
                          noise_sigma=float(rng.choice([0.0, 0.5, 1.0, 3.0])),
                          outlier_fraction=float(rng.choice([0.0, 0.1, 0.25, 0.5])),
                          outlier_scale=float(rng.choice([1.0, 10.0, 50.0])),
                          seed=int(rng.integers(0, 2 ** 63)) if k % 3 else k))
    Mx, Dx = 1000, 8
    B = len(specs)
    out = dict(x=np.full((B, Mx, Dx), np.nan), y=np.full((B, Mx), np.nan), beta=np.full((B, Dx), np.nan),
               truth=np.zeros((B, Dx)), has_truth=np.zeros(B, bool))
    for key in ("m", "d", "n_informative", "seed"):
        out[key] = np.array([s[key] for s in specs], dtype=np.uint64 if key == "seed" else np.int64)
    for key, src in (("sigma", "noise_sigma"), ("fraction", "outlier_fraction"), ("scale", "outlier_scale")):
        out[key] = np.array([s[src] for s in specs])
    for k, sp in enumerate(specs):
        data, beta = generate(GenSpec(**sp))
        m, d = sp["m"], sp["d"]
        out["x"][k, :m, :d] = data.x
        out["y"][k, :m] = data.y
        out["beta"][k, :d] = beta.beta
        if sp["true_coefficients"] is not None:
            out["truth"][k, :d] = sp["true_coefficients"]
            out["has_truth"][k] = True
    np.savez_compressed(os.path.join(GOLDEN, "genspec.npz"), **out)
    print("genspec.npz", flush=True)


def _objective_task(args):
    _ref()
    from ladlasso.model import Coefficients, Dataset, ProblemSpec, evaluate_objective

    x, y, lam, b = args
    return evaluate_objective(ProblemSpec(Dataset(x, y), lam), Coefficients(b))


def gen_objective(pool):
    """model.evaluate_objective (model.py:151-154) on random coefficients, every p <= 8 and
    row counts on both sides of numpy's 128-term pairwise block (up to 1000 rows)."""
    rng = np.random.default_rng(151)
    out = {}
    for m, d in ((1, 1), (7, 2), (30, 5), (31, 8), (128, 3), (129, 4), (200, 6), (257, 7), (1000, 8), (1023, 1)):
        B = 16 if m <= 257 else 4
        X = rng.standard_normal((B, m, d)) * rng.choice([1e-3, 1.0, 1e3], size=(B, 1, 1))
        Y = rng.standard_normal((B, m)) * 10
        beta = rng.standard_normal((B, d))
        beta[rng.random((B, d)) < 0.3] = 0.0
        lam = rng.uniform(0.0, 3.0, B)
        lam[0] = 0.0  # the 1e-9 floor
        vals = pool.map(_objective_task, [(X[b], Y[b], float(lam[b]), beta[b]) for b in range(B)])
        out[f"x_{m}_{d}"], out[f"y_{m}_{d}"], out[f"beta_{m}_{d}"] = X, Y, beta
        out[f"lam_{m}_{d}"], out[f"objective_{m}_{d}"] = lam, np.array(vals)
    out["shapes"] = np.array([[int(k.split("_")[1]), int(k.split("_")[2])] for k in out if k.startswith("x_")])
    np.savez_compressed(os.path.join(GOLDEN, "objective.npz"), **out)
    print("objective.npz", flush=True)


def _run_ref_cli(argv):
    """Run the reference CLI in-process; return (exit code, stdout, stderr)."""
    import contextlib
    import io

    _ref()
    from ladlasso import cli

    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = cli.main(argv)
    return code, out.getvalue(), err.getvalue()


def gen_cli(pool):
    """Reference CLI transcripts (cli.py) for tests/test_cli.py: gen files, solve RESULT
    lines, check/bench CSVs.  Wall-time fields are kept verbatim; the tests drop them."""
    import json
    import tempfile

    _ref()
    from ladlasso.rng import Pcg32

    fx = {}
    with tempfile.TemporaryDirectory() as tmp:
        # gen: CSV + sidecar bytes for a few specs
        fx["gen"] = []
        for spec in (["--m", "7", "--d", "3", "--seed", "11"],
                     ["--m", "12", "--d", "2", "--n-informative", "1", "--noise-sigma", "0.5",
                      "--outlier-fraction", "0.25", "--outlier-scale", "20", "--seed", "3"],
                     ["--m", "30", "--d", "5", "--outlier-fraction", "0.1", "--seed", "123456789"]):
            path = os.path.join(tmp, "g.csv")
            code, so, _ = _run_ref_cli(["gen", path] + spec)
            with open(path) as fh, open(path + ".meta.json") as fm:
                fx["gen"].append(dict(argv=spec, code=code, stdout=so, csv=fh.read(), meta=fm.read()))
        # solve: every in-scope solver on one generated dataset
        path = os.path.join(tmp, "s.csv")
        _run_ref_cli(["gen", path, "--m", "11", "--d", "3", "--outlier-fraction", "0.2", "--seed", "77"])
        with open(path) as fh:
            fx["solve_csv"] = fh.read()
        fx["solve"] = []
        for solver in ("locus_ternary", "locus_quadrature", "brute", "ccd_plain", "lp"):
            for lam in ("0.05", "1.5"):
                argv = ["solve", path, "--lambda", lam, "--solver", solver]
                code, so, _ = _run_ref_cli(argv)
                fx["solve"].append(dict(argv=argv[2:], code=code, stdout=so))
        # solve --dump-lp: the exported standard form
        lp_path = os.path.join(tmp, "s.lp")
        _run_ref_cli(["solve", path, "--lambda", "0.3", "--solver", "lp", "--dump-lp", lp_path])
        with open(lp_path) as fh:
            fx["dump_lp"] = fh.read()
        # check: per-instance CSV of a small seeded sweep
        fx["check"] = []
        for argv in (["--n-instances", "16", "--seed", "5"],
                     ["--n-instances", "12", "--seed", "2", "--d", "1-2", "--m", "5,8", "--lambda", "0.3,2"]):
            out = os.path.join(tmp, "c.csv")
            code, so, _ = _run_ref_cli(["check"] + argv + ["--out", out])
            with open(out) as fh:
                fx["check"].append(dict(argv=argv, code=code, stdout=so, csv=fh.read()))
        # check task picker for the default 50-instance sweep (d, m, lambda, seed)
        picker = Pcg32(0)
        d_set, m_set, l_set = [1, 2, 3], list(range(4, 13)), [0.01, 0.1, 1.0]
        fx["check_tasks_seed0"] = [[d_set[picker.below(3)], m_set[picker.below(9)], l_set[picker.below(3)],
                                    0 + 1_000_003 * (i + 1)] for i in range(50)]
        # bench: runs + medians CSVs (no lp)
        out = os.path.join(tmp, "b.csv")
        argv = ["--d", "1,2,3", "--m", "6,10", "--repeats", "2", "--seed", "4",
                "--solvers", "lp,brute,locus_ternary,locus_quadrature,ccd_plain"]
        code, so, _ = _run_ref_cli(["bench"] + argv + ["--out", out])
        with open(out) as fh, open(os.path.join(tmp, "b_medians.csv")) as fm:
            fx["bench"] = dict(argv=argv, code=code, csv=fh.read(), medians=fm.read())
    with open(os.path.join(GOLDEN, "cli.json"), "w") as fh:
        json.dump(fx, fh, indent=1)
        fh.write("\n")
    print("wrote cli.json")


def gen_curve(pool):
    """Certificate and locus-sampling goldens: ccd.is_axiswise_minimum (ccd.py:214-237) on certified,
    nudged and random coefficient vectors (with and without skip); locus.sample_locus (locus.py:126-147)."""
    _ref()
    from ladlasso.ccd import is_axiswise_minimum, solve_ccd
    from ladlasso.datagen import GenSpec, generate
    from ladlasso.linesearch import Bracket
    from ladlasso.locus import default_bracket, default_outer_axis, locus_value, sample_locus
    from ladlasso.model import ProblemSpec

    rng = np.random.default_rng(2024)
    Mx, Dx = 30, 5
    cx, cy, cl, cb, cs, cok = [], [], [], [], [], []
    for k in range(60):
        d = 1 + k % Dx
        m = 4 + (k * 7) % (Mx - 3)
        data, _ = generate(GenSpec(m=m, d=d, noise_sigma=1.0, outlier_fraction=0.2, seed=7000 + k))
        lam = (0.01, 0.1, 1.0)[k % 3]
        spec = ProblemSpec(data, lam)
        base = solve_ccd(spec).beta.beta
        axis = default_outer_axis(data)
        lp = locus_value(spec, axis, float(base[axis]) + 0.3).beta.beta
        cands = [(base, -1), (base + np.where(np.arange(d) == k % d, 1e-5 * (1 + abs(base[k % d])), 0.0), -1),
                 (base + np.where(np.arange(d) == k % d, 1e-12, 0.0), -1), (lp, axis), (lp, -1),
                 (rng.standard_normal(d), -1)]
        for b, sk in cands:
            X = np.zeros((Mx, Dx)); X[:m, :d] = data.x
            Y = np.zeros(Mx); Y[:m] = data.y
            B = np.zeros(Dx); B[:d] = b
            cx.append(X); cy.append(Y); cl.append(lam); cb.append(B); cs.append(sk)
            cok.append(bool(is_axiswise_minimum(spec, b, skip=None if sk < 0 else sk)))
    nm = [4 + (k * 7) % (Mx - 3) for k in range(60) for _ in range(6)]
    nd = [1 + k % Dx for k in range(60) for _ in range(6)]
    out = dict(x=np.array(cx), y=np.array(cy), lam=np.array(cl), beta=np.array(cb), skip=np.array(cs),
               m=np.array(nm), d=np.array(nd), certified=np.array(cok))
    # sample_locus on 16 problems (d = 2..4), 9 or 33 points, over the default bracket or a window
    sx, sy, sl, sm, sd, sa, sbr, sn = [], [], [], [], [], [], [], []
    st, sbeta, sval, sconv, sev = [], [], [], [], []
    for k in range(16):
        d = 2 + k % 3
        m = 6 + k % 9
        data, _ = generate(GenSpec(m=m, d=d, noise_sigma=1.0, outlier_fraction=0.2, seed=8000 + k))
        spec = ProblemSpec(data, (0.01, 0.1, 1.0)[k % 3])
        axis = default_outer_axis(data)
        br = default_bracket(data) if k % 2 == 0 else Bracket(-0.5, 1.5)
        npts = 9 if k % 2 else 33
        pts = sample_locus(spec, axis, br, npts)
        X = np.zeros((16, 4)); X[:m, :d] = data.x
        Y = np.zeros(16); Y[:m] = data.y
        sx.append(X); sy.append(Y); sl.append(spec.lam); sm.append(m); sd.append(d); sa.append(axis)
        sbr.append((br.lo, br.hi)); sn.append(npts)
        T = np.full(33, np.nan); T[:npts] = [pt.t for pt in pts]
        Bt = np.full((33, 4), np.nan); Bt[:npts, :d] = [pt.beta.beta for pt in pts]
        V = np.full(33, np.nan); V[:npts] = [pt.value for pt in pts]
        Cv = np.zeros(33, bool); Cv[:npts] = [pt.inner_converged for pt in pts]
        Ev = np.zeros(33, int); Ev[:npts] = [pt.inner_evals for pt in pts]
        st.append(T); sbeta.append(Bt); sval.append(V); sconv.append(Cv); sev.append(Ev)
    out.update(s_x=np.array(sx), s_y=np.array(sy), s_lam=np.array(sl), s_m=np.array(sm), s_d=np.array(sd),
               s_axis=np.array(sa), s_bracket=np.array(sbr), s_n=np.array(sn), s_t=np.array(st),
               s_beta=np.array(sbeta), s_value=np.array(sval), s_conv=np.array(sconv), s_evals=np.array(sev))
    np.savez_compressed(os.path.join(GOLDEN, "curve.npz"), **out)
    print("wrote curve.npz", int(np.sum(out["certified"])), "of", len(out["certified"]), "certified")


def gen_lp(pool):
    """lp.solve_lp / simplex_minimize goldens (lp.py:106-215): shapes m 2..32, d 1..8, both pivot rules,
    pivot budgets, the objective trace; dump_lp text (lp.py:218-251)."""
    import tempfile

    _ref()
    from ladlasso.datagen import GenSpec, generate
    from ladlasso.lp import SimplexConfig, dump_lp, formulate, simplex_minimize, solve_lp
    from ladlasso.model import ProblemSpec

    rng = np.random.default_rng(77)
    Mx, Dx, Nx, Tx = 32, 8, 80, 64
    rec = {k: [] for k in ("x", "y", "lam", "m", "d", "rule", "max_pivots", "beta", "objective", "pivots",
                           "converged", "xfull", "basis", "trace", "ntrace")}
    for k in range(240):
        d = 1 + k % Dx
        m = 2 + (k * 5) % (Mx - 1)
        data, _ = generate(GenSpec(m=m, d=d, noise_sigma=1.0, outlier_fraction=0.2, seed=11000 + k))
        lam = float(rng.choice([0.0, 0.01, 0.1, 1.0, 5.0]))
        rule = "bland" if k % 6 == 0 else "dantzig_with_bland_fallback"
        mp = int(rng.integers(1, 12)) if k % 9 == 0 else None
        spec = ProblemSpec(data, lam)
        cfg = SimplexConfig(max_pivots=mp, pivot_rule=rule)
        sol = simplex_minimize(formulate(spec), cfg)
        res = solve_lp(spec, cfg)
        X = np.zeros((Mx, Dx)); X[:m, :d] = data.x
        Y = np.zeros(Mx); Y[:m] = data.y
        xf = np.full(Nx, np.nan); xf[: 2 * d + 2 * m] = sol.x
        bs = np.full(Mx, -1); bs[:m] = sol.basis
        tr = np.full(Tx, np.nan); nt = min(Tx, len(sol.objective_trace)); tr[:nt] = sol.objective_trace[:nt]
        B = np.zeros(Dx); B[:d] = res.beta.beta
        for key, v in (("x", X), ("y", Y), ("lam", lam), ("m", m), ("d", d), ("rule", int(rule == "bland")),
                       ("max_pivots", 0 if mp is None else mp), ("beta", B), ("objective", res.objective),
                       ("pivots", sol.pivots), ("converged", sol.converged), ("xfull", xf), ("basis", bs),
                       ("trace", tr), ("ntrace", nt)):
            rec[key].append(v)
    out = {k: np.array(v) for k, v in rec.items()}
    dumps = []
    with tempfile.TemporaryDirectory() as tmp:
        for k in (0, 5):
            data, _ = generate(GenSpec(m=5 + k, d=2 + k % 3, seed=12000 + k))
            path = os.path.join(tmp, "lp.txt")
            dump_lp(formulate(ProblemSpec(data, 0.25)), path)
            dumps.append(open(path).read())
            out[f"dump{k}_x"], out[f"dump{k}_y"] = data.x.copy(), data.y.copy()
    out["dump_text"] = np.array(dumps)
    np.savez_compressed(os.path.join(GOLDEN, "lp.npz"), **out)
    print("wrote lp.npz", int(out["converged"].sum()), "converged of", len(out["lam"]))


def gen_large(pool):
    """Problems beyond 46 rows (block-per-problem path): ccd_descend with m up to 1000 (sparse columns
    included) and solve_locus (both variants, work counters) with m up to 256."""
    _ref()
    from ladlasso.datagen import GenSpec, generate

    rng = np.random.default_rng(9090)
    cp = []
    for i in range(48):
        m = int((47, 48, 64, 100, 127, 129, 200, 333, 500, 1000)[i % 10])
        d = 1 + i % 8
        x = rng.standard_normal((m, d)) * rng.choice([1.0, 3.0])
        if i % 4 == 0:
            x[rng.random((m, d)) < 0.1] = 0.0
        y = x @ np.where(rng.random(d) < 0.5, rng.uniform(1, 3, d), 0.0) + rng.laplace(0, 0.5, m)
        cp.append(dict(x=x, y=y, lam=float(rng.choice([0.01, 0.1, 1.0])), start=rng.standard_normal(d) * (i % 2),
                       frozen=None if i % 3 else int(rng.integers(0, d)), tol=1e-10, sweeps=500))
    cres = pool.map(_task, [("ccd", q) for q in cp], chunksize=1)
    lp_ = []
    for i in range(24):
        m = int((47, 60, 100, 150, 256, 64)[i % 6])
        d = (2, 3, 5, 8)[i % 4]
        data, _ = generate(GenSpec(m=m, d=d, noise_sigma=1.0, outlier_fraction=0.1, seed=21000 + i))
        lp_.append(dict(x=data.x, y=data.y, lam=float((0.05, 0.5, 2.0)[i % 3]),
                        cfg=dict(outer_search=("ternary", "quadrature")[(i // 4) % 2])))
    lres = pool.map(_task, [("locus", q) for q in lp_], chunksize=1)
    out = {}
    for tag, items, res in (("ccd", cp, cres), ("locus", lp_, lres)):
        Mx = max(q["x"].shape[0] for q in items)
        X = np.zeros((len(items), Mx, 8)); Y = np.zeros((len(items), Mx)); Bt = np.full((len(items), 8), np.nan)
        for k, q in enumerate(items):
            m, d = q["x"].shape
            X[k, :m, :d] = q["x"]; Y[k, :m] = q["y"]
            Bt[k, : len(res[k]["beta"])] = res[k]["beta"]
        out[f"{tag}_x"], out[f"{tag}_y"], out[f"{tag}_beta"] = X, Y, Bt
        out[f"{tag}_m"] = np.array([q["x"].shape[0] for q in items])
        out[f"{tag}_d"] = np.array([q["x"].shape[1] for q in items])
        out[f"{tag}_lam"] = np.array([q["lam"] for q in items])
        out[f"{tag}_objective"] = np.array([r["objective"] for r in res])
        for key in ("iterations", "objective_evals", "converged"):
            out[f"{tag}_{key}"] = np.array([r[key] for r in res])
    S0 = np.zeros((len(cp), 8))
    for k, q in enumerate(cp):
        S0[k, : len(q["start"])] = q["start"]
    out["ccd_start"] = S0
    out["ccd_frozen"] = np.array([-1 if q["frozen"] is None else q["frozen"] for q in cp])
    out["locus_variant"] = np.array([q["cfg"]["outer_search"] == "quadrature" for q in lp_])
    out["locus_D"] = np.array([r["D"] for r in lres]); out["locus_S"] = np.array([r["S"] for r in lres])
    out["locus_status"] = np.array([r["status"] for r in lres])
    np.savez_compressed(os.path.join(GOLDEN, "large.npz"), **out)
    print("large.npz", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--only", default="")
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    os.makedirs(GOLDEN, exist_ok=True)
    only = set(a.only.split(",")) if a.only else None
    with Pool(a.procs) as pool:
        for name, fn in (("kat", gen_kat), ("ccd", gen_ccd), ("acceptance", gen_acceptance),
                         ("params", gen_params), ("configs", lambda p: gen_configs(p, a.quick)),
                         ("cli", gen_cli), ("curve", gen_curve), ("lp", gen_lp), ("large", gen_large),
                         ("bench", lambda p: gen_bench(p, a.quick)), ("objective", gen_objective),
                         ("warm", gen_warm), ("genspec", gen_genspec)):
            if only is None or name in only:
                fn(pool)


if __name__ == "__main__":
    main()
