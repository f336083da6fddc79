"""Re-check the oracle's floating-point order model against the live numpy/OpenBLAS.

TEST INFRASTRUCTURE ONLY.  The reference's reductions (numpy pairwise sums,
OpenBLAS ddot / dgemv_t) have evaluation orders that depend on the numpy
build and on the OpenBLAS kernel DYNAMIC_ARCH picks for the host CPU.  The
oracle restates the orders measured in the build container (numpy 2.3.5,
OpenBLAS 0.3.30, SkylakeX).  This script checks them on random inputs with a
wide dynamic range, where any order difference shows up in the low bits.

    python oracle/probe_numerics.py        # exit 0 when every model matches
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402


def openblas_arch() -> str:
    try:
        from threadpoolctl import threadpool_info

        for info in threadpool_info():
            if info.get("internal_api") == "openblas":
                return str(info.get("architecture"))
    except Exception:  # pragma: no cover
        pass
    return "unknown"


def check(trials: int = 60, seed: int = 0) -> dict:
    rng = np.random.default_rng(seed)
    bad = {"np_sum": 0, "ddot": 0, "gemv": 0, "colsum": 0}
    for _ in range(trials):
        for n in (1, 5, 8, 10, 25, 30, 31):
            a = np.abs(rng.standard_normal(n) * np.exp(rng.uniform(-10, 10, n)))
            bad["np_sum"] += O.np_sum(a) != a.sum()
        for n in range(1, 34):
            x = rng.standard_normal(n) * np.exp(rng.uniform(-8, 8, n))
            y = np.abs(rng.standard_normal(n))
            bad["ddot"] += O.ddot(x, y) != x @ y
        for d in range(1, 9):
            for m in (4, 6, 10, 25, 30, 31):
                x = rng.standard_normal((m, d)) * np.exp(rng.uniform(-5, 5, (m, d)))
                b = rng.standard_normal(d) * np.exp(rng.uniform(-5, 5, d))
                bad["gemv"] += int(np.sum(O.gemv(x, b) != x @ b))
                xa = np.abs(x)
                seq = np.array([xa[:, j].sum() if d == 1 else sum(xa[i, j] for i in range(m)) for j in range(d)])
                if d == 1:
                    seq = np.array([O.np_sum(xa[:, 0])])
                bad["colsum"] += int(np.sum(seq != xa.sum(axis=0)))
    return bad


if __name__ == "__main__":
    arch = openblas_arch()
    res = check()
    print(f"OpenBLAS arch: {arch}; mismatches: {res}")
    sys.exit(0 if all(v == 0 for v in res.values()) else 1)
