"""LP recasting and the batched dense simplex (mirror of the reference's lp.py).

``formulate`` / ``embed`` / ``initial_basis`` / ``dump_lp`` build and export the
standard form on the host exactly as the reference does (lp.py:82-103, :218-251;
they are data layout, not solves).  ``simplex_minimize`` / ``simplex_solve`` /
``solve_lp`` run the tableau simplex on the GPU (lad_lp.cuh through
``lad_lp_solve_f64``), bit-identical to the reference: same pivots, basis,
primal point and objective.  ``solve_lp_batched`` solves B problems at once.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import DEFAULT_LAMBDA_FLOOR
from .errors import InvalidInputError, SimplexError
from .solver import (Coefficients, SolveResult, _check, _is_torch, _spec_arrays, _to_device, _to_host,
                     _validate_device, _validate_host)

PIVOT_RULES = ("bland", "dantzig_with_bland_fallback")

__all__ = ["PIVOT_RULES", "LpStandardForm", "SimplexConfig", "SimplexSolution", "LpBatch", "formulate", "embed",
           "initial_basis", "simplex_minimize", "simplex_solve", "solve_lp", "solve_lp_batched", "dump_lp"]


@dataclass(frozen=True, eq=False)
class LpStandardForm:
    """min cost.v s.t. constraint_matrix @ v = rhs, v >= 0; columns bp (d), bn (d), rp (m), rn (m)."""

    cost: np.ndarray
    constraint_matrix: np.ndarray
    rhs: np.ndarray
    variable_names: tuple
    spec: object

    @property
    def d(self) -> int:
        return self.spec.d

    @property
    def m(self) -> int:
        return self.spec.m


@dataclass(frozen=True)
class SimplexConfig:
    max_pivots: int | None = None  # default 50 * (number of columns)
    pivot_rule: str = "dantzig_with_bland_fallback"
    feasibility_tolerance: float = 1e-9

    def __post_init__(self):
        if self.max_pivots is not None and self.max_pivots < 1:
            raise InvalidInputError("max_pivots must be at least 1")
        if self.pivot_rule not in PIVOT_RULES:
            raise InvalidInputError(f"unknown pivot rule {self.pivot_rule!r}")


@dataclass(eq=False)
class SimplexSolution:
    x: np.ndarray
    objective: float
    pivots: int
    converged: bool
    basis: np.ndarray
    objective_trace: list


def formulate(spec) -> LpStandardForm:
    x, y = np.asarray(spec.data.x), np.asarray(spec.data.y)
    m, d = x.shape
    lam = spec.lambda_eff
    cost = np.concatenate([np.full(2 * d, lam), np.ones(2 * m)])
    matrix = np.hstack([x, -x, np.eye(m), -np.eye(m)])
    names = tuple([f"bp_{j}" for j in range(d)] + [f"bn_{j}" for j in range(d)] + [f"rp_{i}" for i in range(m)]
                  + [f"rn_{i}" for i in range(m)])
    return LpStandardForm(cost, matrix, y.copy(), names, spec)


def embed(lp: LpStandardForm, beta) -> np.ndarray:
    """Feasible full-space point representing ``beta``; its cost equals the objective."""
    b = np.asarray(beta.beta if hasattr(beta, "beta") else beta, dtype=float)
    if b.shape != (lp.d,):
        raise InvalidInputError(f"beta has shape {b.shape}, problem has {lp.d} variables")
    r = np.asarray(lp.spec.data.y) - np.asarray(lp.spec.data.x) @ b
    return np.concatenate([np.maximum(b, 0.0), np.maximum(-b, 0.0), np.maximum(r, 0.0), np.maximum(-r, 0.0)])


def initial_basis(lp: LpStandardForm) -> np.ndarray:
    d, m = lp.d, lp.m
    return np.where(lp.rhs >= 0, 2 * d + np.arange(m), 2 * d + m + np.arange(m))


@dataclass
class LpBatch:
    """Per-problem outputs of ``solve_lp_batched``."""

    beta: object        # (B, d)
    objective: object   # (B,) evaluate_objective(beta)
    pivots: object      # (B,)
    converged: object   # (B,) bool
    status: object      # (B,) 0 ok, 1 unbounded, 2 invalid input, 3 objective mismatch
    x: object = None    # (B, 2d+2m) when requested
    basis: object = None
    trace: object = None

    def raise_for_status(self):
        st = np.asarray(self.status.cpu() if _is_torch(self.status) else self.status)
        if ((st == 1) | (st == 3)).any():
            raise SimplexError(f"problem {int(np.nonzero((st == 1) | (st == 3))[0][0])}: unbounded direction or "
                               "the LP optimum does not reproduce the objective")
        if (st == 2).any():
            raise InvalidInputError(f"problem {int(np.nonzero(st == 2)[0][0])}: non-finite data or invalid lambda")


def solve_lp_batched(X, y, lam, cfg: SimplexConfig | None = None, *, lambda_floor: float = DEFAULT_LAMBDA_FLOOR,
                     full: bool = False, trace_cap: int = 0) -> LpBatch:
    """Batched ``solve_lp`` on the device; numpy inputs give numpy outputs."""
    import torch

    cfg = cfg or SimplexConfig()
    L = _lib.load()
    host = not _is_torch(X)
    if host:
        X, y, lam = _validate_host(X, y, lam)
        dev = torch.device("cuda")
        Xt, yt, lt = (_to_device(a, dev) for a in (X, y, lam))
    else:
        Xt, yt, lt = _validate_device(X, y, lam)
        dev = Xt.device
    B, m, d = Xt.shape
    ncol = 2 * d + 2 * m
    beta = torch.empty((B, d), dtype=torch.float64, device=dev)
    obj = torch.empty(B, dtype=torch.float64, device=dev)
    piv = torch.empty(B, dtype=torch.int32, device=dev)
    cv = torch.empty(B, dtype=torch.uint8, device=dev)
    st = torch.empty(B, dtype=torch.uint8, device=dev)
    xf = torch.empty((B, ncol), dtype=torch.float64, device=dev) if full else None
    bs = torch.empty((B, m), dtype=torch.int32, device=dev) if full else None
    tr = torch.full((B, max(trace_cap, 1)), np.nan, dtype=torch.float64, device=dev) if trace_cap > 0 else None
    _check(L.lad_lp_solve_f64(Xt.data_ptr(), yt.data_ptr(), lt.data_ptr(), B, m, d,
                              0 if cfg.max_pivots is None else int(cfg.max_pivots),
                              1 if cfg.pivot_rule == "bland" else 0, float(cfg.feasibility_tolerance),
                              float(lambda_floor), beta.data_ptr(), obj.data_ptr(), piv.data_ptr(), cv.data_ptr(),
                              st.data_ptr(), None if xf is None else xf.data_ptr(),
                              None if bs is None else bs.data_ptr(), None if tr is None else tr.data_ptr(),
                              int(trace_cap), torch.cuda.current_stream(dev).cuda_stream))
    out = LpBatch(beta, obj, piv, cv.bool(), st, xf, bs, tr)
    if host:
        out = LpBatch(*[None if v is None else _to_host(v) for v in
                        (beta, obj, piv, cv.bool(), st, xf, bs, tr)])
    return out


def _one(lp_or_spec, cfg, full, trace):
    spec = lp_or_spec.spec if isinstance(lp_or_spec, LpStandardForm) else lp_or_spec
    X, y, lam, floor = _spec_arrays(spec)
    cfg = cfg or SimplexConfig()
    cap = 0
    if trace:
        cap = (cfg.max_pivots if cfg.max_pivots is not None else 50 * (2 * X.shape[2] + 2 * X.shape[1])) + 1
    return solve_lp_batched(X, y, lam, cfg, lambda_floor=floor, full=full, trace_cap=cap), cfg


def simplex_minimize(lp: LpStandardForm, cfg: SimplexConfig | None = None) -> SimplexSolution:
    """Primal simplex from the sign-split basis (lp.py:106-170), on the GPU."""
    r, cfg = _one(lp, cfg, True, True)
    if r.status[0] == 2:
        raise InvalidInputError("non-finite data or invalid lambda")
    x = r.x[0]
    npiv = int(r.pivots[0])
    if r.status[0] == 1:
        raise SimplexError("unbounded direction in a formulation that cannot be unbounded")
    return SimplexSolution(x, float(lp.cost @ x), npiv, bool(r.converged[0]), r.basis[0].astype(np.int64),
                           [float(v) for v in r.trace[0, : npiv + 1]])


def simplex_solve(lp: LpStandardForm, cfg: SimplexConfig | None = None) -> SolveResult:
    """Solve the LP and map back to coefficients, revalidating the objective (lp.py:173-193)."""
    t0 = time.perf_counter()
    r, _ = _one(lp, cfg, False, False)
    if r.status[0] == 1:
        raise SimplexError("unbounded direction in a formulation that cannot be unbounded")
    if r.status[0] == 3:
        raise SimplexError("LP optimum does not reproduce the objective")
    if r.status[0] == 2:
        raise InvalidInputError("non-finite data or invalid lambda")
    return SolveResult(Coefficients(r.beta[0]), float(r.objective[0]), "lp", int(r.pivots[0]), 1,
                       time.perf_counter() - t0, bool(r.converged[0]))


def solve_lp(spec, cfg: SimplexConfig | None = None) -> SolveResult:
    """Drop-in for ``ladlasso.lp.solve_lp`` (lp.py:196-215): formulate + solve on the GPU."""
    return simplex_solve(formulate(spec), cfg)


def dump_lp(lp: LpStandardForm, path) -> None:
    """The reference's text export of the standard form (lp.py:218-251), byte for byte."""
    num = "{:+25.17e}"

    def row(values) -> str:
        return " ".join(num.format(v) for v in values)

    m = lp.constraint_matrix.shape[0]
    lines = ["LADLASSO-LP 1", f"vars {lp.cost.size} rows {m}", " ".join(lp.variable_names), "minimize",
             row(lp.cost), "subject-to"]
    lines += [row(lp.constraint_matrix[i]) + " = " + num.format(lp.rhs[i]) for i in range(m)]
    lines.append("bounds all >= 0")
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join(lines) + "\n")
