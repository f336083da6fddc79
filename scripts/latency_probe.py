import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2510_15649_b200 as lad
from paper_2510_15649_b200 import configgen as G, _lib
X, Y, L = G.generate(0, 256, seed=15649)
cfg = lad.LocusConfig()
# warm clocks
for _ in range(3): lad.solve_locus_batched(X, Y, L, cfg); torch.cuda.synchronize()
def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best, r
for ap in (False, True):
    _lib.set_axis_parallel(ap)
    dt, r = t(lambda: lad.solve_locus_batched(X, Y, L, cfg))
    S = r.steps.cpu().numpy()
    print(f"axis_parallel={ap}: B=256 {dt*1e3:.1f} ms; steps/solve median {np.median(S):.0f} max {S.max()} (argmax {S.argmax()})")
    i = int(S.argmax())
    dt1, r1 = t(lambda: lad.solve_locus_batched(X[i:i+1], Y[i:i+1], L[i:i+1], cfg))
    j = int(np.argsort(S)[128])
    dt2, r2 = t(lambda: lad.solve_locus_batched(X[j:j+1], Y[j:j+1], L[j:j+1], cfg))
    print(f"   single worst problem {dt1*1e3:.1f} ms ({S[i]} steps, {dt1/S[i]*1.9e9:.0f} cyc/step);  median problem {dt2*1e3:.1f} ms ({S[j]} steps)")
