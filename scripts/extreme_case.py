"""Debug helper: the extreme-magnitude parity case on a given library build."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2510_15649_b200 import _build
_build.LIB = sys.argv[1]
import paper_2510_15649_b200 as lad
from oracle import oracle as O
dtype = np.float64
rng = np.random.default_rng(17)
big, small = 1e140, 1e-140
for (n, p) in ((30, 5), (12, 3), (31, 8)):
    B = 12
    X = rng.standard_normal((B, n, p))
    X[0::3, :, 1] *= small
    X[1::3, :, p - 1] *= big
    X[2::3, 3, 0] = small * 0.5
    beta = np.zeros(p); beta[0] = 2.0
    Y = X @ beta
    Y[:, ::4] += rng.laplace(0, 0.5, (B, (n + 3) // 4))
    Y[3] *= small
    L = np.full(B, 0.2)
    r = lad.solve_locus_batched(X, Y, L)
    o = O.solve_locus_batch(X, Y, L)
    bad = [i for i in range(B) if not (np.array_equal(r.beta[i], o["beta"][i]) and r.objective[i] == o["objective"][i]
                                        and r.steps[i] == o["steps"][i])]
    print(sys.argv[1].split('/')[-1], (n, p), "mismatches", bad)
    for i in bad[:3]:
        print("  ", i, r.objective[i], o["objective"][i], r.steps[i], o["steps"][i], r.descents[i], o["descents"][i])
