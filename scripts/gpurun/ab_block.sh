# Block-kernel timing (n >= 32) of two library builds: ab_block.sh TAG_A TAG_B
for v in "$@"; do
  for np in "40 5" "100 5" "256 4" "1000 3"; do
    set -- $np
    python - "$v" $1 $2 <<'PY'
import sys, time
sys.path.insert(0, '.')
from paper_2510_15649_b200 import _build
_build.LIB = f"paper_2510_15649_b200/libladlasso_b200_{sys.argv[1]}.so"
import numpy as np, torch
import paper_2510_15649_b200 as lad
n, p = int(sys.argv[2]), int(sys.argv[3])
B = {40: 8192, 100: 4096, 256: 2048, 1000: 592}[n]
rng = np.random.default_rng(1)
X = rng.standard_normal((B, n, p)); beta = np.zeros(p); beta[:2] = (2.0, -1.5)
Y = X @ beta + rng.laplace(0, 0.5, (B, n))
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
L = torch.full((B,), 0.5, dtype=torch.float64, device="cuda")
lad.solve_locus_batched(Xd[:64], Yd[:64], L[:64]); torch.cuda.synchronize()
t0 = time.perf_counter(); r = lad.solve_locus_batched(Xd, Yd, L); torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"{sys.argv[1]} n={n} p={p} B={B}: {B/dt:,.0f} solves/s  obj_sum={float(r.objective.sum()):.17g} steps={int(r.steps.sum())}")
PY
  done
done
