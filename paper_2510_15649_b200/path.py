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

A warm stage depends on the previous one, but only within a dataset.  The datasets are
therefore split into a few groups, each walking its own stages on its own CUDA stream: the
persistent solve kernel of one group fills the SMs that another group's launch leaves idle in
its tail (a 16,384-dataset stage is 3.5 waves of resident warps), and no stage waits on the host.
Host arrays are uploaded once per call, not once per stage; results come back once.
"""

from __future__ import annotations

import numpy as np

from .config import DEFAULT_LAMBDA_FLOOR, LocusConfig
from .solver import (STATUS_SCRATCH, _is_torch, _rerun_scratch, _validate_host, _worst_case_seen, locus_params,
                     solve_locus_batched)

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
                              lambda_floor: float = DEFAULT_LAMBDA_FLOOR, groups: int = 2) -> dict:
    """Solve every dataset of X (Bd, n, p), y (Bd, n) at every lambda of `lambdas` (L,).

    Returns a dict of per-(dataset, lambda) arrays shaped (Bd, L, ...) in the order of
    `lambdas` (numpy for host inputs, CUDA tensors for device inputs).  Cold: one launch;
    warm: one launch per lambda and dataset group, largest lambda first, the groups (at most
    `groups`, at least MIN_GROUP datasets each) on concurrent streams (module docstring)."""
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
    if not on_dev:  # one upload, the device path, one download
        import torch

        Xh, yh, _ = _validate_host(X, y, 0.0)
        dev = torch.device("cuda", torch.cuda.current_device())
        Xd = torch.from_numpy(Xh).to(dev, non_blocking=True)
        yd = torch.from_numpy(yh).to(dev, non_blocking=True)
        out = _warm_path_device(Xd, yd, lam_host, cfg, lambda_floor, groups)
        return {f: v.cpu().numpy() for f, v in out.items()}
    return _warm_path_device(X, y, lam_host, cfg, lambda_floor, groups)


# fewest datasets per stream group (a group's stage is one launch: about one wave of resident warps)
MIN_GROUP = 4096


def _warm_path_device(X, y, lam_host, cfg, lambda_floor, groups):
    """The warm path on device tensors: `groups` independent dataset ranges, each a chain of
    stage launches on its own stream (module docstring).  Results are tensors on X's device,
    ordered on the caller's current stream."""
    import torch

    dev = X.device
    Bd, nl = X.shape[0], lam_host.size
    order = np.argsort(-lam_host, kind="stable")
    # The curve-point scratch at its worst-case capacity, so no solve can end with status 3 and no
    # stage has to be inspected on the host; only a huge outer_max_iterations (where that scratch
    # would be large) keeps the tolerance-bounded capacity and re-runs status-3 problems per stage.
    cap = _worst_case_seen(locus_params(cfg, lambda_floor, X.shape[2]))
    cap = cap if cap <= 4096 else 0
    G = max(1, min(int(groups), Bd // MIN_GROUP))
    bounds = [(g * Bd // G, (g + 1) * Bd // G) for g in range(G)]
    cur = torch.cuda.current_stream(dev)
    streams = [cur] if G == 1 else [torch.cuda.Stream(dev) for _ in range(G)]
    for st in streams:
        if st is not cur:
            st.wait_stream(cur)
    stages = [[None] * G for _ in range(nl)]
    prev = [None] * G
    for k in order:
        for g, (a, b) in enumerate(bounds):
            with torch.cuda.stream(streams[g]):
                Xg, yg = X[a:b], y[a:b]
                lam_k = torch.full((b - a,), float(lam_host[k]), device=dev, dtype=torch.float64)
                br = None
                if prev[g] is not None:
                    R = warm_radius(prev[g].beta, prev[g].status)
                    br = torch.stack([-R, R], dim=1)
                r = solve_locus_batched(Xg, yg, lam_k, cfg, lambda_floor=lambda_floor, brackets=br, seen_capacity=cap)
                if cap == 0:
                    redo = np.nonzero(r.status.cpu().numpy() == STATUS_SCRATCH)[0]
                    if redo.size:
                        r = _rerun_scratch(r, redo, Xg, yg, lam_k, cfg, lambda_floor, None, br, None)
                stages[k][g] = r
                prev[g] = r
    for st in streams:
        if st is not cur:
            cur.wait_stream(st)
    out = {}
    for f in FIELDS:
        cols = []
        for k in range(nl):
            parts = [getattr(stages[k][g], f) for g in range(G)]
            for t in parts:  # allocated on a group's stream, consumed on the caller's
                t.record_stream(cur)
            cols.append(parts[0] if G == 1 else torch.cat(parts))
        out[f] = torch.stack(cols, dim=1)
    return out
