"""The bench's ACTUAL device inputs, solved on the GPU, against the unmodified reference.

Each problem is generated on the device exactly as bench.py does (lad_generate_f64 /
lad_subsets_f64 at the bench's seeds and offsets), solved through the C ABI (config 2
with the bench's data_index lambda replication), and compared bit for bit with the
reference outputs in tests/golden/bench_cfg*.npz (beta, objective, iterations,
objective_evals, converged, D, S).  Also lad_objective_f64 against the reference's
evaluate_objective (model.py:151-154) up to 1023 rows.
"""

import numpy as np
import pytest

from conftest import load_golden
from parity import locus_report

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_15649_b200 as lad  # noqa: E402
from paper_2510_15649_b200 import configgen as G  # noqa: E402


def _device_inputs(g, config):
    seed = int(g["seed"])
    if config in (0, 4):
        X, Y, L = G.generate(config, len(g["lam"]), seed=seed, first=int(g["first"]))
        return X, Y, L, None
    if config == 1:
        parts = [G.generate(1, 1, seed=seed, first=int(i)) for i in g["problem_index"]]
        return (*(torch.cat([p[k] for p in parts]) for k in range(3)), None)
    if config == 2:
        parts = [G.generate(2, 1, seed=seed, first=int(f)) for f in g["dataset_index"]]
        X = torch.cat([p[0] for p in parts])
        Y = torch.cat([p[1] for p in parts])
        idx = torch.arange(X.shape[0], device=X.device).repeat_interleave(16)
        L = torch.tensor(G.LAMBDA_GRID, device=X.device, dtype=torch.float64).repeat(X.shape[0])
        return X, Y, L, idx
    X0, Y0 = G.config3_dataset(seed=seed)
    parts = [G.subsets(X0, Y0, 25, int(k), 1) for k in g["subset_index"]]
    X = torch.cat([p[0] for p in parts])
    Y = torch.cat([p[1] for p in parts])
    return X, Y, torch.full((X.shape[0],), 0.5, device=X.device, dtype=torch.float64), None


@pytest.mark.parametrize("name,config,variants", [
    ("bench_cfg0", 0, ("ternary", "quadrature")), ("bench_cfg1", 1, ("ternary", "quadrature")),
    ("bench_cfg2", 2, ("ternary", "quadrature")), ("bench_cfg3", 3, ("quadrature",)),
    ("bench_cfg4", 4, ("ternary",))])
def test_device_generated_bench_problems_match_reference(name, config, variants):
    g = load_golden(name)
    X, Y, L, idx = _device_inputs(g, config)
    Xe = X[idx] if idx is not None else X
    assert np.array_equal(Xe.cpu().numpy(), g["x"]) and np.array_equal(L.cpu().numpy(), g["lam"])
    B = len(g["lam"])
    for v in variants:
        r = lad.solve_locus_batched(X, Y, L, lad.LocusConfig(outer_search=v), data_index=idx)
        assert bool((r.status == 0).all())
        got = {k: getattr(r, a).cpu().numpy() for k, a in (("iterations", "iterations"),
                                                             ("objective_evals", "objective_evals"),
                                                             ("D", "descents"), ("S", "steps"))}
        rep = locus_report(r.beta.cpu().numpy(), r.objective.cpu().numpy(), g[f"{v}_beta"], g[f"{v}_objective"],
                           got, {k: g[f"{v}_{k}"] for k in got})
        assert rep["exact"] == B, (name, v, rep)
        for k in got:
            assert rep[f"{k}_equal"] == B, (name, v, k, rep)
        assert np.array_equal(r.converged.cpu().numpy().astype(bool), g[f"{v}_converged"])
    if "brute_idx" in g and config != 3:
        bi = np.asarray(g["brute_idx"])
        bb, bo, bv = lad.solve_brute_batched(g["x"][bi], g["y"][bi], g["lam"][bi])
        assert np.array_equal(np.asarray(bo), g["brute_objective"])
        assert np.array_equal(np.asarray(bb), g["brute_beta"])


def test_objective_matches_reference_up_to_1023_rows():
    g = load_golden("objective")
    for m, d in g["shapes"]:
        got = lad.evaluate_objective_batched(g[f"x_{m}_{d}"], g[f"y_{m}_{d}"], g[f"lam_{m}_{d}"],
                                             g[f"beta_{m}_{d}"])
        assert np.array_equal(np.asarray(got), g[f"objective_{m}_{d}"]), (m, d)
