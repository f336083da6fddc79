"""One launch of one library kernel on a BASELINE-shaped workload, for ncu (and its work units).

usage: python scripts/prof_kernels.py WORKLOAD [--units OUT.json]
WORKLOAD: cfg0 cfg1 cfg2 bench2 cfg3 cfg4 cfg4f32 warm2 brute1 brute0 lp2 cert2 gen4 genspec
A warm-up launch of the same kernel on a few problems precedes the profiled one, so the
profiled launch is the LAST launch of that kernel (ncu -k regex:NAME --launch-skip ... or -c
with the kernel filter picks it via --launch-skip-before-match ... ; the driver script uses
`-k regex:NAME -s 1 -c 1`).  The work units of the profiled launch (coordinate steps,
vertices, pivots, problems) are written to --units for the per-unit counters.
"""
import argparse
import json
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import os  # noqa: E402

if os.environ.get("LAD_PROF_LIB"):  # profile another build of the library (A/B captures)
    from paper_2510_15649_b200 import _build  # noqa: E402

    _build.LIB = os.path.abspath(os.environ["LAD_PROF_LIB"])
import paper_2510_15649_b200 as lad  # noqa: E402
from paper_2510_15649_b200 import configgen as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--units", default=None)
a = ap.parse_args()
w = a.workload
units = {}


def locus(config, B, variant="ternary", f32=False, warmup=True):
    seed = 15649 + config
    if config == 3:
        X0, Y0 = G.config3_dataset(seed=seed)
        X, Y = G.subsets(X0, Y0, 25, 0, B)
        L = torch.full((B,), 0.5, device=X.device, dtype=torch.float64)
    else:
        X, Y, L = G.generate(config, B, seed=seed)
    if f32:
        X, Y, L = X.float(), Y.float(), L.float()
    cfg = lad.LocusConfig(outer_search=variant)
    if warmup:
        lad.solve_locus_batched(X[:64], Y[:64], L[:64], cfg)
    r = lad.solve_locus_batched(X, Y, L, cfg)
    torch.cuda.synchronize()
    units.update(kernel="locus", unit="coordinate step", units=float(r.steps.double().sum()),
                 descents=float(r.descents.double().sum()), solves=B, n=X.shape[1], p=X.shape[2])


if w == "cfg0":
    locus(0, 256)  # the whole config (axis-parallel mode: B < two waves)
elif w == "cfg1":
    locus(1, 262144)
elif w == "cfg2":
    locus(2, 8288)  # two waves of resident warps (config-2 shapes, independent problems)
elif w == "cfg3":
    locus(3, 8288, variant="quadrature")
elif w == "cfg4":
    locus(4, 8288)
elif w == "cfg4f32":
    locus(4, 8288, f32=True)
elif w == "bench2":  # the bench's own config-2 launch: 16,384 datasets x 16 lambdas (data_index), ternary
    X, Y, _ = G.generate(2, 16384, seed=15651)
    idx = torch.arange(16384, device=X.device).repeat_interleave(16)
    L = torch.tensor(G.LAMBDA_GRID, device=X.device, dtype=torch.float64).repeat(16384)
    lad.solve_locus_batched(X[:4], Y[:4], L[:64], data_index=idx[:64])
    r = lad.solve_locus_batched(X, Y, L, data_index=idx)
    torch.cuda.synchronize()
    units.update(kernel="locus", unit="coordinate step", units=float(r.steps.double().sum()),
                 descents=float(r.descents.double().sum()), solves=262144, n=30, p=5)
elif w == "warm2":  # one warm stage of the lambda path: per-problem brackets
    X, Y, _ = G.generate(2, 8288, seed=15651)
    br = torch.tensor([[-2.0, 2.0]], device=X.device, dtype=torch.float64).repeat(8288, 1)
    L = torch.full((8288,), 0.1, device=X.device, dtype=torch.float64)
    lad.solve_locus_batched(X[:64], Y[:64], L[:64], brackets=br[:64])
    r = lad.solve_locus_batched(X, Y, L, brackets=br)
    torch.cuda.synchronize()
    units.update(kernel="locus", unit="coordinate step", units=float(r.steps.double().sum()),
                 descents=float(r.descents.double().sum()), solves=8288, n=30, p=5)
elif w in ("brute1", "brute0"):
    config, B = (1, 1 << 18) if w == "brute1" else (0, 64)
    X, Y, L = G.generate(config, B, seed=15649 + config)
    lad.solve_brute_batched(X[:8], Y[:8], L[:8])
    bb, bo, bv = lad.solve_brute_batched(X, Y, L)
    torch.cuda.synchronize()
    units.update(kernel="brute", unit="nonsingular vertex", units=float(bv.double().sum()), solves=B,
                 n=X.shape[1], p=X.shape[2], candidates_per_problem=int(math.comb(X.shape[1] + X.shape[2],
                                                                                     X.shape[2])))
elif w == "lp2":
    X, Y, _ = G.generate(2, 65536, seed=15651)
    L = torch.tensor(G.LAMBDA_GRID, device=X.device).repeat(4096)
    lad.solve_lp_batched(X[:64], Y[:64], L[:64])
    r = lad.solve_lp_batched(X, Y, L)
    torch.cuda.synchronize()
    units.update(kernel="lp", unit="pivot", units=float(r.pivots.double().sum()), solves=65536, n=30, p=5)
elif w == "cert2":
    X, Y, L = G.generate(2, 65536, seed=15651)
    beta = torch.zeros((65536, 5), device=X.device, dtype=torch.float64)
    lad.axiswise_minimum_batched(X[:64], Y[:64], L[:64], beta[:64])
    lad.axiswise_minimum_batched(X, Y, L, beta)
    torch.cuda.synchronize()
    units.update(kernel="cert", unit="problem", units=65536.0, solves=65536, n=30, p=5)
elif w == "gen4":
    G.generate(4, 64, seed=1)
    G.generate(4, 1 << 16, seed=15653)
    torch.cuda.synchronize()
    units.update(kernel="gen", unit="problem", units=float(1 << 16), solves=1 << 16, n=31, p=8)
elif w == "genspec":
    from paper_2510_15649_b200.synth import GenSpec, generate_batched

    generate_batched([GenSpec(m=30, d=5, outlier_fraction=0.1, seed=s) for s in range(8)])
    generate_batched([GenSpec(m=30, d=5, outlier_fraction=0.1, seed=s) for s in range(1 << 16)])
    torch.cuda.synchronize()
    units.update(kernel="genspec", unit="problem", units=float(1 << 16), solves=1 << 16, n=30, p=5)
else:
    raise SystemExit(f"unknown workload {w}")
print(json.dumps(units))
if a.units:
    json.dump(units, open(a.units, "w"))
