"""The locus curve outside the solver: restricted descents, sampling, restarts.

Mirrors of the reference's ``locus.locus_value`` / ``locus.sample_locus``
(locus.py:104-147), ``ccd.perturb_restart`` (ccd.py:240-256) and the data
helpers ``default_outer_axis`` / ``axes_by_influence`` / ``default_bracket``
(locus.py:86-101).  Every descent runs on the GPU through the batched
``ccd_descend`` kernel; a sample of n points is n batched launches, each warm
started from the previous point's coefficients, exactly as the reference's
loop (the points of one problem are sequential by definition).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .config import DEFAULT_LAMBDA_FLOOR, Bracket, CcdConfig
from .errors import InvalidInputError
from .solver import Coefficients, _is_torch, _spec_arrays, ccd_descend, ccd_descend_batched

__all__ = ["LocusPoint", "default_outer_axis", "axes_by_influence", "default_bracket", "locus_value",
           "sample_locus", "sample_locus_batched", "perturb_restart"]


@dataclass(frozen=True, eq=False)
class LocusPoint:
    """locus.LocusPoint (locus.py:74-83)."""

    t: float
    beta: Coefficients
    value: float
    inner_converged: bool
    inner_evals: int


def default_outer_axis(data) -> int:
    return int(np.argmax(np.abs(data.x).sum(axis=0)))


def axes_by_influence(data) -> list[int]:
    influence = np.abs(data.x).sum(axis=0)
    return sorted(range(data.d), key=lambda j: (-influence[j], j))


def default_bracket(data) -> Bracket:
    column_scale = float(np.abs(data.x).mean(axis=0).max())
    radius = float(np.abs(data.y).max()) / column_scale if column_scale > 0 else np.inf
    if not np.isfinite(radius) or radius <= 0:
        radius = 1.0
    return Bracket(-radius, radius)


def locus_value(spec, axis: int, t: float, inner: CcdConfig | None = None, warm=None) -> LocusPoint:
    """Minimise over every coordinate but ``axis`` (held at t), from ``warm`` or zero (locus.py:104-123)."""
    if not 0 <= axis < spec.d:
        raise InvalidInputError(f"axis {axis} out of range for d={spec.d}")
    inner = inner or CcdConfig()
    start = np.array(warm.beta if hasattr(warm, "beta") else warm, dtype=float) if warm is not None \
        else np.zeros(spec.d)
    start[axis] = t
    res = ccd_descend(spec, Coefficients(start), replace(inner, frozen_axis=axis))
    return LocusPoint(t, res.beta, res.objective, res.converged, res.objective_evals)


def sample_locus_batched(X, y, lam, axis: int, bracket: Bracket, n: int, inner: CcdConfig | None = None, *,
                         lambda_floor: float = DEFAULT_LAMBDA_FLOOR):
    """``sample_locus`` over B problems sharing (axis, bracket): n batched restricted descents.

    Returns a dict of arrays: t (n,), beta (B, n, p), value / inner_converged /
    inner_evals (B, n).  Host inputs give numpy outputs, CUDA tensors give tensors."""
    import torch

    if n < 3:
        raise InvalidInputError("need at least 3 sample points")
    inner = inner or CcdConfig()
    host = not _is_torch(X)
    if host:
        dev = torch.device("cuda")
        X = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float64)).to(dev)
        y = torch.from_numpy(np.ascontiguousarray(y, dtype=np.float64)).to(dev)
        lam = torch.as_tensor(np.asarray(lam, dtype=np.float64), device=dev)
    B, m, p = X.shape
    if not 0 <= axis < p:
        raise InvalidInputError(f"axis {axis} out of range for d={p}")
    cfg = replace(inner, frozen_axis=axis)
    ts = np.linspace(bracket.lo, bracket.hi, n)
    warm = torch.zeros((B, p), dtype=torch.float64, device=X.device)
    betas, values, conv, evals = [], [], [], []
    for t in ts:
        start = warm.clone()
        start[:, axis] = float(t)
        r = ccd_descend_batched(X, y, lam, start, cfg, lambda_floor=lambda_floor)
        warm = r.beta
        betas.append(r.beta)
        values.append(r.objective)
        conv.append(r.converged)
        evals.append(r.objective_evals)
    out = dict(t=ts, beta=torch.stack(betas, 1), value=torch.stack(values, 1),
               inner_converged=torch.stack(conv, 1), inner_evals=torch.stack(evals, 1))
    if host:
        out = {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in out.items()}
    return out


def sample_locus(spec, axis: int, bracket: Bracket, n: int, inner: CcdConfig | None = None) -> list[LocusPoint]:
    """Drop-in for ``locus.sample_locus`` (locus.py:126-147) on one problem."""
    if not 0 <= axis < spec.d:
        raise InvalidInputError(f"axis {axis} out of range for d={spec.d}")
    X, y, lam, floor = _spec_arrays(spec)
    s = sample_locus_batched(X, y, lam, axis, bracket, n, inner, lambda_floor=floor)
    return [LocusPoint(float(s["t"][k]), Coefficients(s["beta"][0, k]), float(s["value"][0, k]),
                       bool(s["inner_converged"][0, k]), int(s["inner_evals"][0, k])) for k in range(n)]


def perturb_restart(spec, beta, axis: int, delta: float, cfg: CcdConfig | None = None):
    """Drop-in for ``ccd.perturb_restart`` (ccd.py:240-256): nudge one coordinate, descend again."""
    b = np.array(beta.beta if hasattr(beta, "beta") else beta, dtype=float)
    if not 0 <= axis < spec.d:
        raise InvalidInputError(f"axis {axis} out of range for d={spec.d}")
    b[axis] += delta
    return ccd_descend(spec, Coefficients(b), cfg)
