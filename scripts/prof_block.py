"""One block-kernel launch (n rows, default 100; p=5) for ncu: python scripts/prof_block.py [n]."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2510_15649_b200 as lad
n, p, B = (int(sys.argv[1]) if len(sys.argv) > 1 else 100), 5, 1184
rng = np.random.default_rng(1)
X = rng.standard_normal((B, n, p))
Y = X @ np.array([2.0, -1.5, 0, 0, 0]) + rng.laplace(0, 0.5, (B, n))
r = lad.solve_locus_batched(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(),
                            torch.full((B,), 0.5, dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
print("steps", int(r.steps.sum()), "ok", bool((r.status == 0).all()))
