"""Quick GPU timing of the locus kernel on device-generated config problems."""
import sys, time
import torch
sys.path.insert(0, '.')
import paper_2510_15649_b200 as lad
from paper_2510_15649_b200 import configgen as G

def run(config, B, variant="ternary", lam=None):
    X, Y, L = G.generate(config, B, seed=1)
    if lam is not None:
        L = torch.full_like(L, lam)
    cfg = lad.LocusConfig(outer_search=variant)
    r = lad.solve_locus_batched(X[:256], Y[:256], L[:256], cfg)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = lad.solve_locus_batched(X, Y, L, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    S = r.steps.double().sum().item(); D = r.descents.double().sum().item()
    print(f"cfg{config} {variant} B={B}: {dt:.3f}s  {B/dt:,.0f} solves/s  steps/solve={S/B:.0f} descents/solve={D/B:.0f}  "
          f"{S/dt/1e9:.2f} Gsteps/s status_ok={(r.status==0).float().mean().item():.4f}", flush=True)

for (c, B, v) in [(0, 256, "ternary"), (2, 1 << 14, "ternary"), (2, 1 << 16, "ternary"), (2, 1 << 16, "quadrature"),
                  (1, 1 << 18, "ternary"), (4, 1 << 13, "ternary")]:
    run(c, B, v)
X0, Y0 = G.config3_dataset()
Xs, Ys = G.subsets(X0, Y0, 25, 0, 1 << 15)
t0 = time.perf_counter(); r = lad.solve_locus_batched(Xs, Ys, torch.full((1 << 15,), 0.5, device='cuda', dtype=torch.float64), lad.LocusConfig(outer_search="quadrature")); torch.cuda.synchronize()
print(f"cfg3 quadrature B=32768: {time.perf_counter()-t0:.3f}s")
