"""Parity metrics shared by the CPU (oracle vs reference golden) and GPU tests.

The contract (BASELINE.json north_star):
  * per problem |f - f_ref| <= 1e-9 * |f_ref|;
  * support {j : |beta_j| > 1e-6} identical;
  * ||beta - beta_ref||_inf <= 1e-6 where the minimiser is unique.
On top of that we track bit-exactness (beta, f) and equality of the work
counters (iterations, objective_evals, D = descents, S = coordinate steps),
which is what the oracle and the CUDA path actually achieve.
"""

from __future__ import annotations

import numpy as np

OBJ_RTOL = 1e-9
BETA_ATOL = 1e-6
SUPPORT_EPS = 1e-6


def locus_report(beta, obj, beta_ref, obj_ref, counters=None, counters_ref=None):
    beta = np.asarray(beta, float)
    beta_ref = np.asarray(beta_ref, float)
    obj = np.asarray(obj, float)
    obj_ref = np.asarray(obj_ref, float)
    rel = np.abs(obj - obj_ref) / np.maximum(np.abs(obj_ref), 1e-300)
    sup = (np.abs(beta) > SUPPORT_EPS) == (np.abs(beta_ref) > SUPPORT_EPS)
    sup_ok = np.all(sup | np.isnan(beta_ref), axis=-1)
    dbeta = np.nanmax(np.abs(beta - beta_ref), axis=-1)
    exact = np.all((beta == beta_ref) | np.isnan(beta_ref), axis=-1) & (obj == obj_ref)
    rep = dict(n=int(obj.size), exact=int(exact.sum()), obj_ok=int((rel <= OBJ_RTOL).sum()),
               support_ok=int(sup_ok.sum()), beta_ok=int((dbeta <= BETA_ATOL).sum()),
               worst_rel=float(rel.max()) if rel.size else 0.0, worst_dbeta=float(dbeta.max()) if dbeta.size else 0.0)
    if counters is not None:
        for k in counters:
            rep[f"{k}_equal"] = int((np.asarray(counters[k]) == np.asarray(counters_ref[k])).sum())
    rep["mismatch_idx"] = np.nonzero(~((rel <= OBJ_RTOL) & sup_ok))[0].tolist()
    return rep
