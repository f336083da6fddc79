"""A/B timing of two builds of the library on the same inputs (run each in its own process).

usage: python scripts/ab_timing.py LIBPATH [config] [B] [reps] [f64|f32]
"""
import sys, time
import torch
sys.path.insert(0, '.')
from paper_2510_15649_b200 import _build, _lib
_build.LIB = sys.argv[1]
import paper_2510_15649_b200 as lad
from paper_2510_15649_b200 import configgen as G
config = int(sys.argv[2]) if len(sys.argv) > 2 else 2
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 16
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
X, Y, L = G.generate(config, B, seed=1)
if len(sys.argv) > 5 and sys.argv[5] == "f32":  # the fp32 mode on the same problems rounded once
    X, Y, L = X.float(), Y.float(), L.float()
cfg = lad.LocusConfig()
lad.solve_locus_batched(X[:1024], Y[:1024], L[:1024], cfg)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r = lad.solve_locus_batched(X, Y, L, cfg); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
S = r.steps.double().sum().item()
print(f"{sys.argv[1].split('/')[-1]} cfg{config}{'f32' if len(sys.argv) > 5 and sys.argv[5] == 'f32' else ''} B={B}: best {min(ts):.4f}s {B/min(ts):,.0f} solves/s "
      f"{S/min(ts)/1e9:.3f} Gsteps/s  obj_sum={r.objective.double().sum().item():.17g}", flush=True)
