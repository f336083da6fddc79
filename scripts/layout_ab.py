"""Same-box A/B of the config-2 problem layout: the bench step's 16,384 datasets x 16 lambdas in
dataset-major order (problem = dataset * 16 + k) against lambda-major orders (problem = k * D +
dataset, lambdas ascending or descending).  The persistent kernel fetches problems in index order,
so the layout decides which problems form each launch's tail.

usage: python scripts/layout_ab.py [reps] [datasets]
"""
import sys
import torch
sys.path.insert(0, '.')
import numpy as np
import paper_2510_15649_b200 as lad
from paper_2510_15649_b200 import configgen as G

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
D = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
dev = torch.device('cuda:0')
grid = np.logspace(-2, 1, 16)
X, Y, _ = G.generate(2, D, seed=15651, device=dev)
g = torch.tensor(grid, device=dev, dtype=torch.float64)
lays = {
    'dataset_major': (torch.arange(D, device=dev).repeat_interleave(16), g.repeat(D)),
    'lambda_major_asc': (torch.arange(D, device=dev).repeat(16), g.repeat_interleave(D)),
    'lambda_major_desc': (torch.arange(D, device=dev).repeat(16), g.flip(0).repeat_interleave(D)),
}
cfgs = {v: lad.LocusConfig(outer_search=v) for v in ('ternary', 'quadrature')}
lad.solve_locus_batched(X, Y, lays['dataset_major'][1][:4096], cfgs['ternary'], data_index=lays['dataset_major'][0][:4096])
torch.cuda.synchronize()
best = {}
sums = {}
for r in range(reps):
    for name, (idx, lam) in lays.items():
        for v, c in cfgs.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = lad.solve_locus_batched(X, Y, lam, c, data_index=idx)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            best[(name, v)] = min(best.get((name, v), 1e9), t)
            sums[(name, v)] = res.objective.double().sum().item()
for name in lays:
    tt = sum(best[(name, v)] for v in cfgs)
    print(f"{name:18s} ternary {best[(name, 'ternary')]:.4f}s quadrature {best[(name, 'quadrature')]:.4f}s "
          f"step {tt:.4f}s {32 * D / tt:,.0f} solves/s  objsum {sums[(name, 'ternary')]:.10g} {sums[(name, 'quadrature')]:.10g}",
          flush=True)
