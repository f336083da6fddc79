"""Where the host-buffer brute-force call spends its time (config 1, 2^20 problems)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_15649_b200 as lad
from paper_2510_15649_b200 import configgen as G, solver as S
B = 1 << 20
X, Y, L = G.generate(1, B, seed=1)
torch.cuda.synchronize()
hp = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t).numpy() for t in (X, Y, L)]
lad.solve_brute_batched(*hp); torch.cuda.synchronize()
def tm(name, f, k=3):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(name, [round(t * 1e3, 2) for t in ts], flush=True)
tm("device call", lambda: lad.solve_brute_batched(X, Y, L))
tm("host call", lambda: lad.solve_brute_batched(*hp))
tm("validate_host", lambda: S._validate_host(*hp))
tm("to_device x3", lambda: [S._to_device(a, torch.device('cuda')) for a in hp])
r = lad.solve_brute_batched(X, Y, L)
tm("results .cpu()", lambda: [t.cpu().numpy() for t in r])
