"""Throughput of the locus solve at a given (n, p) on random problems; kernel policy selectable.

usage: python scripts/shape_timing.py n p B [policy: auto|thread]
"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2510_15649_b200 as lad
from paper_2510_15649_b200 import _lib
n, p, B = (int(a) for a in sys.argv[1:4])
pol = sys.argv[4] if len(sys.argv) > 4 else "auto"
rng = np.random.default_rng(1)
X = rng.standard_normal((B, n, p))
beta = np.zeros(p); beta[:2] = (2.0, -1.5)
Y = X @ beta + rng.laplace(0, 0.5, (B, n))
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
L = torch.full((B,), 0.5, dtype=torch.float64, device="cuda")
if pol == "thread":
    _lib.set_kernel_policy(_lib.KERNEL_THREAD)
lad.solve_locus_batched(Xd[:8], Yd[:8], L[:8])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); r = lad.solve_locus_batched(Xd, Yd, L); e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 1e3
S = r.steps.double().sum().item()
print(f"n={n} p={p} B={B} {pol}: {t:.3f}s {B/t:,.0f} solves/s {S/t/1e9:.3f} Gsteps/s steps/solve={S/B:.0f} "
      f"status_ok={bool((r.status == 0).all())} obj_sum={r.objective.double().sum().item():.17g}", flush=True)
