"""The lambda path on the GPU: cold (one launch, data_index) and warm (per-lambda launches with
per-problem initial_bracket) against the reference (warm_path.npz) and the oracle replay;
per-problem brackets and the curve-point scratch status (3) with its automatic re-run."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_15649_b200 as lad  # noqa: E402
from paper_2510_15649_b200 import configgen as G  # noqa: E402


@pytest.mark.parametrize("variant", ["ternary", "quadrature"])
@pytest.mark.parametrize("on_device", [True, False])
def test_warm_path_matches_reference(variant, on_device):
    g = load_golden("warm_path")
    X, Y = g["x"], g["y"]
    if on_device:
        X, Y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    r = lad.solve_lambda_path_batched(X, Y, g["lambdas"], lad.LocusConfig(outer_search=variant), warm=True)
    get = (lambda a: a.cpu().numpy()) if on_device else np.asarray
    assert np.array_equal(get(r["beta"]), g[f"{variant}_beta"])
    assert np.array_equal(get(r["objective"]), g[f"{variant}_objective"])
    assert np.array_equal(get(r["iterations"]), g[f"{variant}_iterations"])
    assert np.array_equal(get(r["objective_evals"]), g[f"{variant}_objective_evals"])
    assert np.array_equal(get(r["converged"]).astype(bool), g[f"{variant}_converged"])


def test_warm_path_matches_oracle_replay_at_scale(oracle):
    X, Y, _ = G.generate(2, 256, seed=15651, first=12345)
    lams = G.LAMBDA_GRID
    for variant in ("ternary", "quadrature"):
        r = lad.solve_lambda_path_batched(X, Y, lams, lad.LocusConfig(outer_search=variant), warm=True)
        o = oracle.solve_warm_path(X.cpu().numpy(), Y.cpu().numpy(), lams, outer_search=variant)
        assert np.array_equal(r["objective"].cpu().numpy(), o["objective"])
        assert np.array_equal(r["beta"].cpu().numpy(), o["beta"])
        assert np.array_equal(r["steps"].cpu().numpy(), o["steps"])


@pytest.mark.parametrize("on_device", [True, False])
def test_warm_path_stream_groups_equal_one_group(monkeypatch, on_device):
    """Dataset groups walking their stages on concurrent streams (path.py) give the single-stream
    result, bit for bit, for device tensors and for host arrays (one upload, one download)."""
    from paper_2510_15649_b200 import path

    X, Y, _ = G.generate(2, 96, seed=15651, first=777)
    lams = G.LAMBDA_GRID[::3]
    cfg = lad.LocusConfig(outer_search="quadrature")
    one = lad.solve_lambda_path_batched(X, Y, lams, cfg, warm=True, groups=1)
    monkeypatch.setattr(path, "MIN_GROUP", 16)
    args = (X, Y) if on_device else (X.cpu().numpy(), Y.cpu().numpy())
    for groups in (2, 5):
        r = lad.solve_lambda_path_batched(*args, lams, cfg, warm=True, groups=groups)
        for f in path.FIELDS:
            got = r[f].cpu().numpy() if on_device else np.asarray(r[f])
            assert got.shape == tuple(one[f].shape)
            assert np.array_equal(got, one[f].cpu().numpy()), f


def test_warm_path_large_max_iterations_keeps_bounded_scratch():
    """outer_max_iterations large enough that the worst-case scratch is not used: the per-stage
    status-3 inspection path gives the same results as the default."""
    X, Y, _ = G.generate(2, 24, seed=15651, first=99)
    lams = G.LAMBDA_GRID[::5]
    ref = lad.solve_lambda_path_batched(X, Y, lams, lad.LocusConfig(), warm=True)
    r = lad.solve_lambda_path_batched(X, Y, lams, lad.LocusConfig(outer_max_iterations=5000), warm=True)
    assert torch.equal(r["objective"], ref["objective"])
    assert torch.equal(r["beta"], ref["beta"])


def test_cold_path_equals_independent_solves():
    X, Y, _ = G.generate(2, 64, seed=15651)
    lams = G.LAMBDA_GRID
    r = lad.solve_lambda_path_batched(X, Y, lams)
    Xr, Yr = X.repeat_interleave(16, 0), Y.repeat_interleave(16, 0)
    s = lad.solve_locus_batched(Xr, Yr, torch.tensor(lams, device=X.device).repeat(64))
    assert torch.equal(r["objective"].reshape(-1), s.objective)


def test_per_problem_brackets_device_and_host(oracle):
    g = load_golden("bench_cfg0")
    X, Y, L = g["x"][:6], g["y"][:6], g["lam"][:6]
    bk = np.array([[-3.0, 3.0], [-1.0, 2.0], [-0.5, 0.5], [2.0, 2.0], [-np.inf, 1.0], [-10.0, 10.0]])
    o = oracle.solve_locus_batch(X, Y, L, brackets=bk, nthreads=2)
    for host in (True, False):
        args = (X, Y, L) if host else tuple(torch.from_numpy(a).cuda() for a in (X, Y, L))
        r = lad.solve_locus_batched(*args, brackets=bk)
        st = np.asarray(r.status if host else r.status.cpu())
        assert list(st) == [0, 0, 0, 2, 2, 0]
        ok = st == 0
        ob = np.asarray(r.objective if host else r.objective.cpu())
        assert np.array_equal(ob[ok], o["objective"][ok])


def test_scratch_capacity_status_and_rerun(oracle):
    """A capacity below what the search needs ends the problem with status 3; the default
    (tolerance-bounded) capacity and the automatic worst-case re-run give the reference's result."""
    X, Y, L = G.generate(0, 32, seed=15649)
    r = lad.solve_locus_batched(X, Y, L, seen_capacity=40)
    assert bool((r.status == 3).all())
    o = oracle.solve_locus_batch(X.cpu().numpy(), Y.cpu().numpy(), L.cpu().numpy())
    r = lad.solve_locus_batched(X.cpu().numpy(), Y.cpu().numpy(), L.cpu().numpy())
    assert np.array_equal(np.asarray(r.objective), o["objective"])
    # a stalled search (relative tolerance below the bracket's resolution) runs all max_iterations
    cfg = lad.LocusConfig(outer_tolerance=1e-17, outer_max_iterations=400)
    rs = lad.solve_locus_batched(X[:4].cpu().numpy(), Y[:4].cpu().numpy(), L[:4].cpu().numpy(), cfg)
    os_ = oracle.solve_locus_batch(X[:4].cpu().numpy(), Y[:4].cpu().numpy(), L[:4].cpu().numpy(),
                                   outer_tolerance=1e-17, outer_max_iterations=400)
    assert list(np.asarray(rs.status)) == [0, 0, 0, 0]
    assert np.array_equal(np.asarray(rs.objective), os_["objective"])
