import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_15649_b200 as lad
from paper_2510_15649_b200 import configgen as G
B = 1 << 20
X, Y, L = G.generate(1, B, seed=1)
torch.cuda.synchronize()
pin = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t) for t in (X, Y, L)]
hp = [t.numpy() for t in pin]
hn = [np.array(t.cpu().numpy()) for t in (X, Y, L)]  # pageable copies
lad.solve_locus_batched(X[:1024], Y[:1024], L[:1024]); torch.cuda.synchronize()
def tm(f, k=3):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return [round(t * 1e3, 1) for t in ts]
print("device ms", tm(lambda: lad.solve_locus_batched(X, Y, L)))
print("host pinned ms", tm(lambda: lad.solve_locus_batched(*hp)))
print("host pageable ms", tm(lambda: lad.solve_locus_batched(*hn)))
t0 = time.perf_counter(); d = torch.from_numpy(hp[0]).cuda(); torch.cuda.synchronize(); print("H2D X pinned via torch ms", round((time.perf_counter() - t0) * 1e3, 1), hp[0].nbytes / 1e6, "MB")
