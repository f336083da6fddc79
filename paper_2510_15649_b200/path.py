"""The lambda path (BASELINE config 2): every dataset solved over a lambda grid.

Cold mode is 16 independent ``solve_locus`` calls per dataset (the reference's own
semantics: solve_locus has no state across calls, locus.py:300-409).  It runs as ONE
launch per outer search over all (dataset, lambda) pairs, the lambdas sharing each
dataset's X through ``data_index``.

Warm mode ("with warm starts", BASELINE config 2) is defined here, because the
reference has no warm start across problems.  It uses only the reference's own
knob, ``LocusConfig.initial_bracket`` (locus.py:56, consumed at :227 for every axis
search and at :364-365 for the dense-refine width), so every warm solve is still
exactly a reference ``solve_locus`` call and is replayable on the CPU oracle:

    the grid is walked from the largest lambda down (sparse to dense);
    the first lambda uses the default bracket (locus.py:96-101);
    lambda k >= 1 uses Bracket(-R, R) with R = max(1, 2 * max_j |beta_prev_j|),
    beta_prev = this dataset's solution at the previous (larger) lambda
    (R = 1 if that solve did not finish with status 0).

Each warm stage is one launch over all datasets (stages depend on each other).
"""

from __future__ import annotations

import numpy as np

from .config import DEFAULT_LAMBDA_FLOOR, LocusConfig
from .solver import _is_torch, solve_locus_batched

FIELDS = ("beta", "objective", "iterations", "objective_evals", "converged", "status", "descents", "steps")


def warm_radius(beta_prev, status_prev):
    """R = max(1, 2 max_j |beta_j|) per problem (exact IEEE ops; 1 where the previous solve failed)."""
    if _is_torch(beta_prev):
        import torch

        r = torch.clamp(2.0 * beta_prev.abs().amax(dim=1), min=1.0)
        return torch.where(status_prev == 0, r, torch.ones_like(r))
    r = np.maximum(1.0, 2.0 * np.abs(beta_prev).max(axis=1))
    return np.where(np.asarray(status_prev) == 0, r, 1.0)


def solve_lambda_path_batched(X, y, lambdas, cfg: LocusConfig | None = None, *, warm: bool = False,
                              lambda_floor: float = DEFAULT_LAMBDA_FLOOR) -> dict:
    """Solve every dataset of X (Bd, n, p), y (Bd, n) at every lambda of `lambdas` (L,).

    Returns a dict of per-(dataset, lambda) arrays shaped (Bd, L, ...) in the order of
    `lambdas` (numpy for host inputs, CUDA tensors for device inputs).  Cold: one launch;
    warm: one launch per lambda, largest lambda first (module docstring)."""
    cfg = cfg if cfg is not None else LocusConfig()
    on_dev = _is_torch(X)
    lam_host = np.asarray(lambdas.cpu() if _is_torch(lambdas) else lambdas, dtype=np.float64).reshape(-1)
    Bd, nl = X.shape[0], lam_host.size
    if on_dev:
        import torch

        dev = X.device
    if not warm:
        if on_dev:
            idx = torch.arange(Bd, device=dev, dtype=torch.int64).repeat_interleave(nl)
            lam = torch.as_tensor(lam_host, device=dev).repeat(Bd)
        else:
            idx = np.repeat(np.arange(Bd, dtype=np.int64), nl)
            lam = np.tile(lam_host, Bd)
        r = solve_locus_batched(X, y, lam, cfg, lambda_floor=lambda_floor, data_index=idx)
        return {k: getattr(r, k).reshape((Bd, nl) + tuple(getattr(r, k).shape[1:])) for k in FIELDS}
    order = np.argsort(-lam_host, kind="stable")
    stages = [None] * nl
    prev = None
    for k in order:
        lam_k = (torch.full((Bd,), float(lam_host[k]), device=dev, dtype=torch.float64) if on_dev
                 else np.full(Bd, float(lam_host[k])))
        if prev is None:
            r = solve_locus_batched(X, y, lam_k, cfg, lambda_floor=lambda_floor)
        else:
            R = warm_radius(prev.beta, prev.status)
            br = torch.stack([-R, R], dim=1) if on_dev else np.stack([-R, R], axis=1)
            r = solve_locus_batched(X, y, lam_k, cfg, lambda_floor=lambda_floor, brackets=br)
        stages[k] = r
        prev = r
    stack = (lambda vs: torch.stack(vs, dim=1)) if on_dev else (lambda vs: np.stack(vs, axis=1))
    return {f: stack([getattr(stages[k], f) for k in range(nl)]) for f in FIELDS}
