"""Bucket rules (ncu_lines.py --buckets) for locus_warp_kernel, from the current source line numbers.

usage: python scripts/warp_buckets.py  -> prints name:file:first:last,... for ncu_lines.py
Buckets: the phases of a coordinate step (div = breakpoints, mhit = median guess test, walk = order-
neighbour walk, sort = ordering fallback, skip = skip test, ddot = v_new, accept), the descent loop
(dinit / dloop / dend), the objective, the controller and the per-problem fetch.
"""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W = "lad_locus_warp.cuh"
L = "lad_locus.cuh"
src = {f: open(os.path.join(ROOT, "paper_2510_15649_b200", "csrc", f)).read().splitlines() for f in (W, L)}


def find(f, pat, start=0):
    for i in range(start, len(src[f])):
        if re.search(pat, src[f][i]):
            return i
    raise SystemExit(f"{f}: no match for {pat!r} after line {start + 1}")


def func(f, pat, indent=""):
    """1-based [first, last] lines of the function whose signature matches pat (ends at `indent}`)."""
    a = find(f, pat)
    b = find(f, "^" + indent + "}$", a)
    return a + 1, b + 1


rules = []
rules.append(("nearest",) + func(W, r"__device__ int nearest\(const double \*seen", "    "))
rules.append(("fetch",) + func(W, r"__device__ int fetch\(Ctl<PMAX> &C", "    "))
rules.append(("colsum",) + func(W, r"__device__ double col_abs_sum", "    "))
rules.append(("sparse",) + func(W, r"void sparse_column\("))
s0 = find(W, r"uint32_t bitonic_inv_mask")
s1 = func(W, r"T median_by_order_call\(")[1]
rules.append(("sort", s0 + 1, s1))
mu0, mu1 = func(W, r"__forceinline__ void median_update\(")
h1 = find(W, r"if \(!hit\) \{", mu0)
h2 = find(W, r"if \(!hit\) \{", h1 + 1)
dd = find(W, r"const T a = fabs\(dsub\(t_new, loc\)\);", h2)
ac = find(W, r"if \(v_new < f_cur\) \{", dd)
rules += [("walk", h1 + 1, h2), ("skip", h2 + 1, dd), ("ddot", dd + 1, ac), ("accept", ac + 1, mu1),
          ("mhit", mu0, h1)]
rules.append(("sparse_step",) + func(W, r"StepState<T> sparse_step\("))
rules.append(("div",) + func(W, r"__forceinline__ void warp_step\("))
rules.append(("objective",) + func(W, r"T warp_objective\("))
d0, d1 = func(W, r"void warp_descent_body\(")
j0 = find(W, r"int j = j0;", d0)
ob = find(W, r"const T obj = warp_objective", j0)
rules += [("dinit", d0, j0 + 1), ("dend", ob + 1, d1), ("dloop", j0 + 2, ob)]
c0 = find(L, r"int controller_body\(")
c1 = find(L, r"^#undef ISSUE", c0)
rules.append(("controller", c0 + 1, c1 + 1))
rules.append(("kernel",) + func(W, r"__global__ void .*locus_warp_kernel"))
print(",".join(f"{n}:{W if n != 'controller' else L}:{a}:{b}" for n, a, b in rules))
