"""Small launches of every library kernel, for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

usage: compute-sanitizer --tool racecheck python scripts/sanitize_workload.py [GROUP...]
GROUPs (default: all): warp (the warp-per-problem locus kernel: compile-time and runtime shapes, both
axis modes, sparse columns, fp32, per-problem brackets, data_index), thread (config-1 shape), block (32 <= n),
descent (ccd_descend), brute, lp, cert, gen.  Batches are a few problems each: the sanitizer runs the
kernels 10-100x slower.  Every result is also compared with the CPU oracle where one exists, so a
sanitizer-clean run is a correct run.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_15649_b200 as lad  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2510_15649_b200 import _lib, configgen as G  # noqa: E402
from paper_2510_15649_b200.synth import GenSpec, generate_batched  # noqa: E402

groups = sys.argv[1:] or ["warp", "thread", "block", "descent", "brute", "lp", "cert", "gen"]
dev = "cuda"
checked = 0


def same(r, X, Y, L, f32=False, **kw):
    """GPU result r against the oracle on the same bytes (beta, objective, steps bit-identical)."""
    global checked
    Xh, Yh, Lh = (t.cpu().numpy() for t in (X, Y, L))
    o = O.solve_locus_batch(Xh, Yh, Lh, nthreads=4, **kw)
    ok = (np.array_equal(r.beta.cpu().numpy(), o["beta"]) and np.array_equal(r.objective.cpu().numpy(), o["objective"])
          and np.array_equal(r.steps.cpu().numpy(), o["steps"]))
    if not ok:
        raise SystemExit(f"parity failure under the sanitizer: {kw} f32={f32}")
    checked += len(Lh)


if "warp" in groups:
    for config, B in ((0, 6), (3, 4), (4, 3)):
        if config == 3:
            X0, Y0 = G.config3_dataset(seed=15652)
            X, Y = G.subsets(X0, Y0, 25, 0, B)
            L = torch.full((B,), 0.5, device=dev, dtype=torch.float64)
        else:
            X, Y, L = G.generate(config, B, seed=15649 + config)
        for variant in ("ternary", "quadrature"):
            r = lad.solve_locus_batched(X, Y, L, lad.LocusConfig(outer_search=variant))  # axis-parallel (small B)
            same(r, X, Y, L, outer_search=variant)
        _lib.set_axis_parallel(0)  # the serial axis scan (what large batches run)
        r = lad.solve_locus_batched(X[:2], Y[:2], L[:2])
        same(r, X[:2], Y[:2], L[:2])
        _lib.set_axis_parallel(1)
    # fp32 mode (config-4 shape) and a runtime-shape problem with a sparse column
    X, Y, L = G.generate(4, 3, seed=15653)
    r = lad.solve_locus_batched(X.float(), Y.float(), L.float())
    same(r, X.float(), Y.float(), L.float())
    rng = np.random.default_rng(7)
    Xs = rng.standard_normal((4, 17, 3))
    Xs[:, ::3, 1] = 0.0
    Ys = rng.standard_normal((4, 17))
    Xs, Ys = torch.tensor(Xs, device=dev), torch.tensor(Ys, device=dev)
    Ls = torch.full((4,), 0.7, device=dev, dtype=torch.float64)
    r = lad.solve_locus_batched(Xs, Ys, Ls)
    same(r, Xs, Ys, Ls)
    # lambda grid through data_index and per-problem brackets (the warm stage's inputs)
    X, Y, _ = G.generate(2, 2, seed=15651)
    idx = torch.arange(2, device=dev).repeat_interleave(3)
    L = torch.tensor([0.01, 1.0, 10.0], device=dev, dtype=torch.float64).repeat(2)
    br = torch.tensor([[-2.0, 2.0]], device=dev, dtype=torch.float64).repeat(6, 1)
    lad.solve_locus_batched(X, Y, L, data_index=idx)
    lad.solve_locus_batched(X, Y, L, data_index=idx, brackets=br)
    print("warp ok")

if "thread" in groups:
    X, Y, L = G.generate(1, 96, seed=15650)
    for variant in ("ternary", "quadrature"):
        r = lad.solve_locus_batched(X, Y, L, lad.LocusConfig(outer_search=variant))
        same(r, X, Y, L, outer_search=variant)
    print("thread ok")

if "block" in groups:
    rng = np.random.default_rng(11)
    for n, p in ((40, 3), (63, 2)):
        Xb = torch.tensor(rng.standard_normal((2, n, p)), device=dev)
        Yb = torch.tensor(rng.standard_normal((2, n)), device=dev)
        Lb = torch.full((2,), 1.0, device=dev, dtype=torch.float64)
        r = lad.solve_locus_batched(Xb, Yb, Lb)
        same(r, Xb, Yb, Lb)
    print("block ok")

if "descent" in groups:
    X, Y, L = G.generate(0, 8, seed=3)
    st = torch.zeros((8, 5), device=dev, dtype=torch.float64)
    lad.ccd_descend_batched(X, Y, L, st)
    X1, Y1, L1 = G.generate(1, 64, seed=4)
    lad.ccd_descend_batched(X1, Y1, L1, torch.zeros((64, 2), device=dev, dtype=torch.float64))
    print("descent ok")

if "brute" in groups:
    X1, Y1, L1 = G.generate(1, 64, seed=15650)
    lad.solve_brute_batched(X1, Y1, L1)  # thread per problem (66 vertices)
    rng = np.random.default_rng(5)
    Xc = torch.tensor(rng.standard_normal((2, 12, 4)), device=dev)  # C(16,4) = 1820: thread kernel
    Yc = torch.tensor(rng.standard_normal((2, 12)), device=dev)
    lad.solve_brute_batched(Xc, Yc, torch.ones(2, device=dev, dtype=torch.float64))
    Xc = torch.tensor(rng.standard_normal((2, 16, 5)), device=dev)  # C(21,5) = 20349: chunked kernel
    Yc = torch.tensor(rng.standard_normal((2, 16)), device=dev)
    lad.solve_brute_batched(Xc, Yc, torch.ones(2, device=dev, dtype=torch.float64))
    print("brute ok")

if "lp" in groups:
    X, Y, L = G.generate(0, 8, seed=9)
    lad.solve_lp_batched(X, Y, L)
    print("lp ok")

if "cert" in groups:
    X, Y, L = G.generate(0, 64, seed=9)
    r = lad.solve_locus_batched(X[:4], Y[:4], L[:4])
    beta = torch.zeros((64, 5), device=dev, dtype=torch.float64)
    beta[:4] = r.beta
    lad.axiswise_minimum_batched(X, Y, L, beta)
    lad.evaluate_objective_batched(X, Y, L, beta)
    print("cert ok")

if "gen" in groups:
    for c in (0, 1, 2, 4):
        G.generate(c, 64, seed=1)
    X0, Y0 = G.config3_dataset(seed=15652)
    G.subsets(X0, Y0, 25, 100, 64)
    generate_batched([GenSpec(m=30, d=5, outlier_fraction=0.1, seed=s) for s in range(64)])
    print("gen ok")

torch.cuda.synchronize()
print(f"done: {checked} solves checked bit-exact against the oracle")
