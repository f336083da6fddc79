"""One locus launch on device-generated config problems (for ncu)."""
import sys, argparse
import torch
sys.path.insert(0, '.')
import paper_2510_15649_b200 as lad
from paper_2510_15649_b200 import configgen as G
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--B", type=int, default=4096)
ap.add_argument("--variant", default="ternary")
a = ap.parse_args()
X, Y, L = G.generate(a.config, a.B, seed=1)
r = lad.solve_locus_batched(X, Y, L, lad.LocusConfig(outer_search=a.variant))
torch.cuda.synchronize()
print("steps", r.steps.sum().item(), "status_ok", (r.status == 0).all().item())
