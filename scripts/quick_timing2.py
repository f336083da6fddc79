import sys, time, subprocess
import torch
sys.path.insert(0, '.')
import paper_2510_15649_b200 as lad
from paper_2510_15649_b200 import configgen as G, _lib
print(subprocess.run(["nvidia-smi","--query-gpu=clocks.sm,clocks.max.sm,power.draw","--format=csv,noheader"],capture_output=True,text=True).stdout.strip())
def run(config, B, variant="ternary", policy=0, reps=2):
    _lib.set_kernel_policy(policy)
    X, Y, L = G.generate(config, B, seed=1)
    cfg = lad.LocusConfig(outer_search=variant)
    lad.solve_locus_batched(X[:512], Y[:512], L[:512], cfg); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter(); r = lad.solve_locus_batched(X, Y, L, cfg); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    S = r.steps.double().sum().item()
    print(f"cfg{config} {variant} B={B} policy={policy}: {best:.3f}s {B/best:,.0f} solves/s {S/best/1e9:.2f} Gsteps/s", flush=True)
run(1, 1 << 18, policy=0); run(1, 1 << 18, policy=1); run(1, 1 << 18, policy=2)
run(2, 1 << 16, policy=0); run(2, 1 << 16, policy=0)
run(4, 1 << 13, policy=0)
print(subprocess.run(["nvidia-smi","--query-gpu=clocks.sm,clocks.max.sm,power.draw","--format=csv,noheader"],capture_output=True,text=True).stdout.strip())
