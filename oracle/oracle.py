"""ctypes wrapper over the CPU oracle (oracle/ladlasso_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's cpu_baseline / ``--impl reference`` legs as the parity checker and
the CPU baseline.  The product package (paper_2510_15649_b200) never imports
this module.

The oracle restates /root/reference/pkg/src/ladlasso (``solve_locus``,
``ccd_descend``, ``solve_brute``) with numpy 2.3.5 / OpenBLAS 0.3.30
(SkylakeX) reduction orders; it is pinned bit-exact against the reference's own
outputs in tests/golden (see oracle/gen_golden.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

MAX_M = 64
MAX_D = 8


class LocusParams(C.Structure):
    """Mirror of orc_locus_params (LocusConfig fields, locus.py:52-58)."""

    _fields_ = [
        ("outer_axis", C.c_int),
        ("outer_search", C.c_int),
        ("outer_tolerance", C.c_double),
        ("outer_probes", C.c_int),
        ("outer_max_iterations", C.c_int),
        ("has_bracket", C.c_int),
        ("bracket_lo", C.c_double),
        ("bracket_hi", C.c_double),
        ("inner_sweep_tol", C.c_double),
        ("inner_max_sweeps", C.c_int),
    ]


def build(force: bool = False) -> str:
    newest = max(os.path.getmtime(os.path.join(_HERE, f)) for f in ("ladlasso_oracle.c", "orc_descent.inc", "gen_host.c", "Makefile"))
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < newest:
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        lp = C.POINTER(C.c_longlong)
        L.orc_np_sum.restype = C.c_double
        L.orc_np_sum.argtypes = [dp, C.c_int]
        L.orc_ddot.restype = C.c_double
        L.orc_ddot.argtypes = [dp, dp, C.c_int]
        L.orc_gemv_row.restype = C.c_double
        L.orc_gemv_row.argtypes = [dp, dp, C.c_int, C.c_int, C.c_int]
        L.orc_objective.restype = C.c_double
        L.orc_objective.argtypes = [dp, dp, C.c_int, C.c_int, C.c_double, dp]
        L.orc_median_location.restype = C.c_double
        L.orc_median_location.argtypes = [dp, dp, C.c_int]
        L.orc_weighted_median_min.restype = C.c_double
        L.orc_weighted_median_min.argtypes = [dp, dp, C.c_int, C.c_double, dp]
        L.orc_ccd_descend.restype = C.c_int
        L.orc_ccd_descend.argtypes = [dp, dp, C.c_int, C.c_int, C.c_double, dp, C.c_int, C.c_double, C.c_int,
                                      dp, dp, ip, ip, ip, dp, ip]
        fp = C.POINTER(C.c_float)
        L.orc_ccd_descend_f32.restype = C.c_int
        L.orc_ccd_descend_f32.argtypes = [fp, fp, C.c_int, C.c_int, C.c_double, dp, C.c_int, C.c_double, C.c_int,
                                          dp, dp, ip, ip, ip, dp, ip]
        L.orc_solve_locus_batch_f32.restype = C.c_int
        L.orc_solve_locus_batch_f32.argtypes = [fp, fp, fp, C.c_longlong, C.c_int, C.c_int, C.c_double,
                                                C.POINTER(LocusParams), C.c_int, dp, dp, ip, ip, ip, ip, lp, lp]
        L.orc_lp_solve.restype = C.c_int
        L.orc_lp_solve.argtypes = [dp, dp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, dp, dp, ip,
                                   ip, dp, ip]
        L.orc_is_axiswise_minimum.restype = C.c_int
        L.orc_is_axiswise_minimum.argtypes = [dp, dp, C.c_int, C.c_int, C.c_double, dp, C.c_int, C.c_double]
        L.orc_pcg32_sequence.restype = None
        L.orc_pcg32_sequence.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_uint32)]
        L.orc_solve_locus.restype = C.c_int
        L.orc_solve_locus.argtypes = [dp, dp, C.c_int, C.c_int, C.c_double, C.POINTER(LocusParams),
                                      dp, dp, ip, ip, ip, ip, lp, lp]
        L.orc_solve_locus_batch.restype = C.c_int
        L.orc_solve_locus_batch.argtypes = [dp, dp, dp, C.c_longlong, C.c_int, C.c_int, C.c_double,
                                            C.POINTER(LocusParams), C.c_int, dp, dp, ip, ip, ip, ip, lp, lp]
        L.orc_solve_locus_batch_brackets.restype = C.c_int
        L.orc_solve_locus_batch_brackets.argtypes = [dp, dp, dp, C.c_longlong, C.c_int, C.c_int, C.c_double,
                                                     C.POINTER(LocusParams), dp, C.c_int, dp, dp, ip, ip, ip, ip, lp,
                                                     lp]
        L.orc_solve_linear_system.restype = C.c_int
        L.orc_solve_linear_system.argtypes = [dp, dp, C.c_int, C.c_double, dp]
        L.orc_candidate_count.restype = C.c_longlong
        L.orc_candidate_count.argtypes = [C.c_int, C.c_int]
        L.orc_solve_brute.restype = C.c_int
        L.orc_solve_brute.argtypes = [dp, dp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_longlong, dp, dp, lp]
        L.orc_generate.restype = C.c_int
        L.orc_generate.argtypes = [C.c_int, C.c_uint64, C.c_longlong, C.c_longlong, C.c_int, C.c_int, dp, dp, dp, dp]
        L.orc_subsets.restype = C.c_int
        L.orc_subsets.argtypes = [dp, dp, C.c_int, C.c_int, C.c_int, C.c_longlong, C.c_longlong, dp, dp]
        _lib = L
    return _lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def _f(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(C.POINTER(C.c_float))


def _is_f32(*arrays):
    return any(getattr(a, "dtype", None) == np.float32 for a in arrays)


def np_sum(a) -> float:
    a, p = _d(a)
    return lib().orc_np_sum(p, a.size)


def ddot(x, y) -> float:
    x, px = _d(x)
    y, py = _d(y)
    return lib().orc_ddot(px, py, x.size)


def gemv(x, b) -> np.ndarray:
    x, px = _d(x)
    b, pb = _d(b)
    m, d = x.shape
    out = np.empty(m)
    for i in range(m):
        out[i] = lib().orc_gemv_row(C.cast(C.addressof(px.contents) + 8 * i * d, C.POINTER(C.c_double)),
                                    pb, d, i, m)
    return out


def objective(x, y, lam_eff, b) -> float:
    x, px = _d(x)
    y, py = _d(y)
    b, pb = _d(b)
    return lib().orc_objective(px, py, x.shape[0], x.shape[1], lam_eff, pb)


def median_location(loc, w) -> float:
    loc, pl = _d(loc)
    w, pw = _d(w)
    return lib().orc_median_location(pl, pw, loc.size)


def weighted_median_min(loc, w, constant=0.0):
    loc, pl = _d(loc)
    w, pw = _d(w)
    v = C.c_double()
    t = lib().orc_weighted_median_min(pl, pw, loc.size, constant, C.byref(v))
    return t, v.value


@dataclass
class Descent:
    beta: np.ndarray
    objective: float
    iterations: int
    objective_evals: int
    converged: bool
    trace: np.ndarray | None = None


def ccd_descend(x, y, lam_eff, start, frozen_axis=None, sweep_tolerance=1e-10, max_sweeps=500, trace=False):
    """float32 x/y select the fp32 mode (binary32 descent; start and outputs stay binary64)."""
    f32 = _is_f32(x, y)
    x, px = (_f if f32 else _d)(x)
    y, py = (_f if f32 else _d)(y)
    s, ps = _d(start)
    m, d = x.shape
    beta = np.empty(d)
    obj = C.c_double()
    sw, st, cv, tl = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    tbuf = np.empty(max_sweeps * d + 1) if trace else None
    fn = lib().orc_ccd_descend_f32 if f32 else lib().orc_ccd_descend
    rc = fn(px, py, m, d, lam_eff, ps, -1 if frozen_axis is None else int(frozen_axis),
                               sweep_tolerance, max_sweeps, beta.ctypes.data_as(C.POINTER(C.c_double)),
                               C.byref(obj), C.byref(sw), C.byref(st), C.byref(cv),
                               None if tbuf is None else tbuf.ctypes.data_as(C.POINTER(C.c_double)),
                               C.byref(tl))
    if rc:
        raise ValueError("problem shape outside oracle limits")
    return Descent(beta, obj.value, sw.value, st.value, bool(cv.value),
                   None if tbuf is None else tbuf[: tl.value].copy())


def is_axiswise_minimum(x, y, lam_eff, beta, skip=None, tol=1e-9) -> bool:
    x, px = _d(x)
    y, py = _d(y)
    b, pb = _d(beta)
    rc = lib().orc_is_axiswise_minimum(px, py, x.shape[0], x.shape[1], lam_eff, pb, -1 if skip is None else int(skip),
                                       tol)
    if rc < 0:
        raise ValueError("problem shape outside oracle limits")
    return bool(rc)


@dataclass
class LpResult:
    beta: np.ndarray
    objective: float
    pivots: int
    converged: bool
    status: int          # 0 ok, 1 unbounded, 3 objective mismatch
    x: np.ndarray
    basis: np.ndarray


def lp_solve(x, y, lam_eff, max_pivots=None, pivot_rule="dantzig_with_bland_fallback", tol=1e-9) -> LpResult:
    """lp.solve_lp restated (lp.py:106-215)."""
    x, px = _d(x)
    y, py = _d(y)
    m, d = x.shape
    beta = np.empty(d)
    xf = np.empty(2 * d + 2 * m)
    bs = np.empty(m, np.int32)
    obj = C.c_double()
    pv, cv = C.c_int(), C.c_int()
    rc = lib().orc_lp_solve(px, py, m, d, lam_eff, 0 if max_pivots is None else int(max_pivots),
                            1 if pivot_rule == "bland" else 0, tol, beta.ctypes.data_as(C.POINTER(C.c_double)),
                            C.byref(obj), C.byref(pv), C.byref(cv), xf.ctypes.data_as(C.POINTER(C.c_double)),
                            bs.ctypes.data_as(C.POINTER(C.c_int)))
    if rc < 0:
        raise ValueError("problem shape outside oracle limits")
    return LpResult(beta, obj.value, pv.value, bool(cv.value), rc, xf, bs)


def pcg32_sequence(seed, n, stream=54):
    out = (C.c_uint32 * n)()
    lib().orc_pcg32_sequence(seed, stream, n, out)
    return [int(v) for v in out]


def make_params(outer_axis=None, outer_search="ternary", outer_tolerance=1e-9, outer_probes=8,
                outer_max_iterations=200, initial_bracket=None, inner_sweep_tol=1e-10, inner_max_sweeps=500):
    p = LocusParams()
    p.outer_axis = -1 if outer_axis is None else int(outer_axis)
    p.outer_search = {"ternary": 0, "quadrature": 1}[outer_search]
    p.outer_tolerance = outer_tolerance
    p.outer_probes = outer_probes
    p.outer_max_iterations = outer_max_iterations
    if initial_bracket is not None:
        p.has_bracket = 1
        p.bracket_lo, p.bracket_hi = float(initial_bracket[0]), float(initial_bracket[1])
    p.inner_sweep_tol = inner_sweep_tol
    p.inner_max_sweeps = inner_max_sweeps
    return p


@dataclass
class LocusResult:
    beta: np.ndarray
    objective: float
    iterations: int
    objective_evals: int
    converged: bool
    status: int
    descents: int
    steps: int


def solve_locus(x, y, lam_eff, **kw) -> LocusResult:
    x, px = _d(x)
    y, py = _d(y)
    m, d = x.shape
    prm = make_params(**kw)
    beta = np.empty(d)
    obj = C.c_double()
    it, ev, cv, stt = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    dsc, stp = C.c_longlong(), C.c_longlong()
    rc = lib().orc_solve_locus(px, py, m, d, lam_eff, C.byref(prm), beta.ctypes.data_as(C.POINTER(C.c_double)),
                               C.byref(obj), C.byref(it), C.byref(ev), C.byref(cv), C.byref(stt), C.byref(dsc),
                               C.byref(stp))
    if rc:
        raise ValueError("problem shape outside oracle limits")
    return LocusResult(beta, obj.value, it.value, ev.value, bool(cv.value), stt.value, dsc.value, stp.value)


def solve_locus_batch(X, Y, L, lambda_floor=1e-9, nthreads=None, brackets=None, **kw):
    """Batched oracle solve over host threads; X (B,m,d), Y (B,m), L (B,) raw lambdas.
    float32 X/Y select the fp32 mode (then L is taken as float32 too).  brackets (B, 2):
    a per-problem LocusConfig.initial_bracket (fp64 only)."""
    f32 = _is_f32(X, Y)
    cv_ = _f if f32 else _d
    X, pX = cv_(X)
    Y, pY = cv_(Y)
    L, pL = cv_(L)
    B, m, d = X.shape
    prm = make_params(**kw)
    nthreads = nthreads or os.cpu_count() or 1
    beta = np.empty((B, d))
    obj = np.empty(B)
    it = np.empty(B, np.int32)
    ev = np.empty(B, np.int32)
    cv = np.empty(B, np.int32)
    stt = np.empty(B, np.int32)
    dsc = np.empty(B, np.int64)
    stp = np.empty(B, np.int64)
    ip = C.POINTER(C.c_int)
    lp = C.POINTER(C.c_longlong)
    if brackets is not None:
        if f32:
            raise ValueError("per-problem brackets: fp64 only")
        bk, pk = _d(np.asarray(brackets, dtype=np.float64).reshape(B, 2))
        rc = lib().orc_solve_locus_batch_brackets(pX, pY, pL, B, m, d, lambda_floor, C.byref(prm), pk, nthreads,
                                                  beta.ctypes.data_as(C.POINTER(C.c_double)),
                                                  obj.ctypes.data_as(C.POINTER(C.c_double)), it.ctypes.data_as(ip),
                                                  ev.ctypes.data_as(ip), cv.ctypes.data_as(ip), stt.ctypes.data_as(ip),
                                                  dsc.ctypes.data_as(lp), stp.ctypes.data_as(lp))
        if rc:
            raise ValueError("problem shape outside oracle limits")
        return dict(beta=beta, objective=obj, iterations=it, objective_evals=ev, converged=cv.astype(bool),
                    status=stt, descents=dsc, steps=stp)
    fn = lib().orc_solve_locus_batch_f32 if f32 else lib().orc_solve_locus_batch
    rc = fn(pX, pY, pL, B, m, d, lambda_floor, C.byref(prm), nthreads,
                                     beta.ctypes.data_as(C.POINTER(C.c_double)),
                                     obj.ctypes.data_as(C.POINTER(C.c_double)), it.ctypes.data_as(ip),
                                     ev.ctypes.data_as(ip), cv.ctypes.data_as(ip), stt.ctypes.data_as(ip),
                                     dsc.ctypes.data_as(lp), stp.ctypes.data_as(lp))
    if rc:
        raise ValueError("problem shape outside oracle limits")
    return dict(beta=beta, objective=obj, iterations=it, objective_evals=ev, converged=cv.astype(bool),
                status=stt, descents=dsc, steps=stp)


def solve_linear_system(a, b, pivot_rtol=1e-12):
    a, pa = _d(a)
    b, pb = _d(b)
    n = b.size
    sol = np.empty(n)
    ok = lib().orc_solve_linear_system(pa, pb, n, pivot_rtol, sol.ctypes.data_as(C.POINTER(C.c_double)))
    return sol if ok else None


def candidate_count(m, d) -> int:
    return int(lib().orc_candidate_count(m, d))


def solve_brute(x, y, lam_eff, max_variables=6, max_candidates=2_000_000):
    """Returns (beta, objective, vertices) or raises ValueError('too large')."""
    x, px = _d(x)
    y, py = _d(y)
    m, d = x.shape
    beta = np.empty(d)
    obj = C.c_double()
    ev = C.c_longlong()
    rc = lib().orc_solve_brute(px, py, m, d, lam_eff, max_variables, max_candidates,
                               beta.ctypes.data_as(C.POINTER(C.c_double)), C.byref(obj), C.byref(ev))
    if rc in (2, 3):
        raise OverflowError("enumeration too large")
    if rc:
        raise ValueError(f"brute failed rc={rc}")
    return beta, obj.value, ev.value


# ---- host restatement of the device config generator (oracle/gen_host.c) ----

CONFIG_SHAPES = {0: (30, 5), 1: (10, 2), 2: (30, 5), 3: (25, 5), 4: (31, 8)}


def generate(config: int, B: int, seed: int, first: int = 0, with_beta: bool = False):
    """Problems [first, first + B) of BASELINE config 0/1/2/4, byte-identical to lad_generate_f64."""
    n, p = CONFIG_SHAPES[config]
    X = np.empty((B, n, p))
    Y = np.empty((B, n))
    lam = np.empty(B)
    bt = np.empty((B, p))
    dp = C.POINTER(C.c_double)
    rc = lib().orc_generate(config, seed, first, B, n, p, X.ctypes.data_as(dp), Y.ctypes.data_as(dp),
                            lam.ctypes.data_as(dp), bt.ctypes.data_as(dp))
    if rc != 0:
        raise ValueError(f"orc_generate: bad arguments (config {config})")
    return (X, Y, lam, bt) if with_beta else (X, Y, lam)


def subsets(X0, Y0, keep: int, first: int, B: int):
    """Config 3: rows of the k-th keep-subsets (lexicographic), k in [first, first + B)."""
    X0, px = _d(X0)
    Y0, py = _d(Y0)
    n0, p = X0.shape
    X = np.empty((B, keep, p))
    Y = np.empty((B, keep))
    dp = C.POINTER(C.c_double)
    if lib().orc_subsets(px, py, n0, p, keep, first, B, X.ctypes.data_as(dp), Y.ctypes.data_as(dp)) != 0:
        raise ValueError("orc_subsets: bad arguments")
    return X, Y


def config3_dataset(seed: int = 15649 + 3):
    """The one n=30, p=5 dataset of config 3 (config-0 problem 0 under config 3's seed)."""
    X, Y, _ = generate(0, 1, seed)
    return X[0], Y[0]


# ---- the warm-started lambda path (paper_2510_15649_b200/path.py defines the rule) ----

def solve_warm_path(X, Y, lambdas, outer_search="ternary", nthreads=None):
    """Replay of path.solve_lambda_path_batched(warm=True): largest lambda first with the
    default bracket, then Bracket(-R, R), R = max(1, 2 max_j |beta_prev_j|) (1 after a failed
    solve); every stage a reference solve_locus call with initial_bracket.  Returns arrays
    shaped (B, L, ...) in the order of `lambdas`."""
    lam = np.asarray(lambdas, dtype=np.float64).reshape(-1)
    B, nl = X.shape[0], lam.size
    out, prev = {}, None
    for k in np.argsort(-lam, kind="stable"):
        L = np.full(B, float(lam[k]))
        if prev is None:
            r = solve_locus_batch(X, Y, L, nthreads=nthreads, outer_search=outer_search)
        else:
            R = np.maximum(1.0, 2.0 * np.abs(prev["beta"]).max(axis=1))
            R = np.where(prev["status"] == 0, R, 1.0)
            r = solve_locus_batch(X, Y, L, nthreads=nthreads, outer_search=outer_search,
                                  brackets=np.stack([-R, R], axis=1))
        out[k] = r
        prev = r
    return {f: np.stack([out[k][f] for k in range(nl)], axis=1) for f in out[0]}
