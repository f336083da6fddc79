"""Serial vs axis-parallel locus solves across batch sizes (config 2 or 4 problems): where to switch.

usage: python scripts/axis_threshold.py [config]
"""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2510_15649_b200 as lad
from paper_2510_15649_b200 import configgen as G, _lib
CFG = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for B in ((256, 1024, 2048, 4096, 8192, 16384) if CFG != 4 else (256, 1024, 2048, 4096, 8192)):
    X, Y, L = G.generate(CFG, B, seed=3)
    row = []
    for mode in (0, 2):  # 0: serial scan; 2: axis-parallel forced
        _lib.set_axis_parallel(mode)
        lad.solve_locus_batched(X[:64], Y[:64], L[:64]); torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            lad.solve_locus_batched(X, Y, L); torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        row.append(B / best)
    _lib.set_axis_parallel(1)
    print(f"B={B:6d} serial {row[0]:10,.0f}  axis-parallel {row[1]:10,.0f}  ratio {row[1] / row[0]:.2f}", flush=True)
