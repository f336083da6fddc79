"""Straggler probe: per-problem work distribution of a config-2 bench block, serial vs axis-parallel."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2510_15649_b200 as lad
from paper_2510_15649_b200 import _lib, configgen as G
from paper_2510_15649_b200.distributed import block_for_step
LAMBDA_GRID = 10.0 ** np.linspace(-2.0, 1.0, 16)
blk = 1 << 14
dev = torch.device('cuda')
for s in [int(a) for a in sys.argv[1:]] or [3, 6]:
    first = block_for_step(s, 1, 0, (1 << 20) // blk) * blk
    X, Y, _ = G.generate(2, blk, seed=15649 + 2, first=first, device=dev)
    idx = torch.arange(blk, device=dev).repeat_interleave(16)
    lam = torch.tensor(LAMBDA_GRID, device=dev).repeat(blk)
    for mode in (1, 2):
        _lib.set_axis_parallel(mode)
        lad.solve_locus_batched(X[:64], Y[:64], lam[:1024], data_index=idx[:1024])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = lad.solve_locus_batched(X, Y, lam, data_index=idx); e1.record(); torch.cuda.synchronize()
        st = r.steps.cpu().numpy()
        print(f"step {s} mode {mode}: {e0.elapsed_time(e1):.1f} ms; steps/solve median {np.median(st):.0f} "
              f"p99 {np.percentile(st, 99):.0f} max {st.max()} (solve {int(st.argmax())}, x{st.max() / np.median(st):.1f}); "
              f"obj_sum {r.objective.double().sum().item():.17g}", flush=True)
    _lib.set_axis_parallel(1)
