"""Edge inputs through every batched entry point: empty batches, read-only and non-contiguous
host arrays, device tensors, and agreement between the host-array and device-tensor paths.

The reference's datasets are frozen read-only float64 arrays (model.py:32-39); host arrays go
through lad_copy_h2d (a copy from the caller's own pointer) and come back in page-locked
arrays, so both must be exercised for every call, as must B = 0 (a shard of an empty range in
the multi-GPU split, distributed.shard_range).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_15649_b200 as lad  # noqa: E402


def _problems(B, n=12, p=3, seed=3):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((B, n, p))
    Y = X @ np.array([1.5, 0.0, -2.0][:p]) + rng.laplace(0, 0.4, (B, n))
    L = rng.uniform(0.1, 1.5, B)
    return X, Y, L


CALLS = {
    "locus": lambda X, Y, L, b: lad.solve_locus_batched(X, Y, L).objective,
    "ccd": lambda X, Y, L, b: lad.ccd_descend_batched(X, Y, L, b).objective,
    "brute": lambda X, Y, L, b: lad.solve_brute_batched(X, Y, L)[1],
    "lp": lambda X, Y, L, b: lad.solve_lp_batched(X, Y, L).objective,
    "objective": lambda X, Y, L, b: lad.evaluate_objective_batched(X, Y, L, b),
    "certificate": lambda X, Y, L, b: lad.axiswise_minimum_batched(X, Y, L, b),
}


def _np(a):
    return a.cpu().numpy() if torch.is_tensor(a) else np.asarray(a)


@pytest.mark.parametrize("name", sorted(CALLS))
def test_empty_batch_host_and_device(name):
    X, Y, L = _problems(0)
    b = np.zeros((0, 3))
    out = CALLS[name](X, Y, L, b)
    assert _np(out).shape[0] == 0
    dev = [torch.from_numpy(a).cuda() for a in (X, Y, L, b)]
    out = CALLS[name](*dev)
    assert _np(out).shape[0] == 0


@pytest.mark.parametrize("name", sorted(CALLS))
def test_read_only_and_strided_host_arrays_match_device(name):
    X, Y, L = _problems(64)
    b = np.random.default_rng(5).standard_normal((64, 3))
    ref = _np(CALLS[name](*[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (X, Y, L, b)]))
    ro = [a.copy() for a in (X, Y, L, b)]
    for a in ro:
        a.setflags(write=False)
    assert np.array_equal(_np(CALLS[name](*ro)), ref), "read-only host arrays"
    # the same values through non-contiguous views (column-reversed storage, every other row of a wider array)
    Xw = np.empty((64, 12, 6))
    Xw[:, :, ::2] = X
    Yw = np.empty((128, 12))
    Yw[::2] = Y
    Lw = np.empty(192)
    Lw[::3] = L
    bw = np.empty((64, 6))
    bw[:, 1::2] = b
    assert not (Xw[:, :, ::2].flags.c_contiguous or Lw[::3].flags.c_contiguous or bw[:, 1::2].flags.c_contiguous)
    out = CALLS[name](Xw[:, :, ::2], Yw[::2], Lw[::3], bw[:, 1::2])
    assert np.array_equal(_np(out), ref), "strided host arrays"


def test_host_results_are_ordinary_writable_arrays():
    X, Y, L = _problems(8)
    r = lad.solve_locus_batched(X, Y, L)
    beta, obj, nv = lad.solve_brute_batched(X, Y, L)
    for a in (r.beta, r.objective, beta, obj, nv):
        assert isinstance(a, np.ndarray) and a.flags.writeable and a.flags.c_contiguous
    r.beta[0, 0] = 1.0  # results own their (page-locked) memory
    beta[0, 0] = 1.0


def test_float32_host_arrays_go_to_the_fp32_mode_and_float64_stays_exact(oracle):
    """dtype selects the path: float64 in -> reference arithmetic, float32 in -> fp32 mode."""
    X, Y, L = _problems(16)
    r64 = lad.solve_locus_batched(X, Y, L)
    o64 = oracle.solve_locus_batch(X, Y, L)
    assert np.array_equal(r64.objective, o64["objective"])
    Xf, Yf, Lf = (a.astype(np.float32) for a in (X, Y, L))
    r32 = lad.solve_locus_batched(Xf, Yf, Lf)
    o32 = oracle.solve_locus_batch(Xf, Yf, Lf)
    assert r32.objective.dtype == np.float64 and np.array_equal(r32.objective, o32["objective"])


def _degenerate_cases():
    rng = np.random.default_rng(21)
    n, p = 10, 3
    base_X = rng.standard_normal((n, p))
    base_y = base_X @ np.array([1.0, -2.0, 0.5]) + rng.laplace(0, 0.3, n)
    cases = []
    cases.append(("all-zero design", np.zeros((n, p)), base_y, 0.5))
    cases.append(("lambda 0 (floor 1e-9)", base_X, base_y, 0.0))
    cases.append(("lambda above max column sum", base_X, base_y, 2.0 * np.abs(base_X).sum(axis=0).max()))
    cases.append(("duplicated rows", np.repeat(base_X[:5], 2, axis=0), np.repeat(base_y[:5], 2), 0.3))
    cases.append(("y identically zero", base_X, np.zeros(n), 0.3))
    cases.append(("one row", base_X[:1], base_y[:1], 0.3))
    cases.append(("one column", base_X[:, :1], base_y, 0.3))
    Xc = base_X.copy()
    Xc[:, 1] = 1.0  # a constant column
    cases.append(("constant column", Xc, base_y, 0.3))
    return cases


@pytest.mark.parametrize("case", range(8))
@pytest.mark.parametrize("variant", ["ternary", "quadrature"])
def test_degenerate_problems_bit_exact(oracle, case, variant):
    name, x, y, lam = _degenerate_cases()[case]
    X, Y, L = x[None].copy(), y[None].copy(), np.array([lam])
    r = lad.solve_locus_batched(X, Y, L, lad.LocusConfig(outer_search=variant))
    o = oracle.solve_locus_batch(X, Y, L, outer_search=variant)
    assert np.array_equal(r.status, o["status"]), name
    if o["status"][0] == 0:
        assert np.array_equal(r.beta, o["beta"]) and np.array_equal(r.objective, o["objective"]), name
        assert (r.steps[0], r.descents[0], r.iterations[0]) == (o["steps"][0], o["descents"][0], o["iterations"][0])
    d = lad.ccd_descend_batched(X, Y, L, np.zeros((1, x.shape[1])))
    od = oracle.ccd_descend(x, y, max(lam, 1e-9), np.zeros(x.shape[1]))
    assert np.array_equal(d.beta[0], od.beta) and d.objective[0] == od.objective, name


def test_big_endian_host_arrays():
    X, Y, L = _problems(16)
    ref = lad.solve_brute_batched(X, Y, L)[1]
    be = [a.astype(a.dtype.newbyteorder(">")) for a in (X, Y, L)]
    assert np.array_equal(lad.solve_brute_batched(*be)[1], ref)
    assert np.array_equal(lad.solve_locus_batched(*be).objective, lad.solve_locus_batched(X, Y, L).objective)


def test_brute_chunked_path_beyond_65535_problems(oracle):
    """C(33,3) = 5456 > 4096 vertices takes the block-per-(problem, chunk) path, whose grid.y holds
    at most 65535 problems: larger batches run in slices."""
    B = 65535 + 77
    rng = np.random.default_rng(11)
    X = rng.standard_normal((B, 30, 3))
    Y = rng.standard_normal((B, 30))
    L = rng.uniform(0.1, 2.0, B)
    bb, bo, bv = lad.solve_brute_batched(X, Y, L)
    for i in (0, 65534, 65535, 65536, B - 1):
        ob, oo, on = oracle.solve_brute(X[i], Y[i], float(L[i]))
        assert float(bo[i]) == oo and np.array_equal(np.asarray(bb[i]), ob) and int(bv[i]) == on, i


def test_large_host_batch_pipelined_equals_device_solve(oracle):
    """Host arrays of >= 2^19 independent problems take the chunked two-stream path of
    lad_locus_solve_host_f64 (copies overlapping solves); its results equal the device-tensor solve
    of the same problems bit for bit, including a ragged last chunk, and the oracle on a sample."""
    from paper_2510_15649_b200 import configgen as G

    B = (1 << 19) + 12345
    X, Y, L = G.generate(1, B, seed=15650, first=4242)
    dev = lad.solve_locus_batched(X, Y, L)
    Xh, Yh, Lh = (t.cpu().numpy() for t in (X, Y, L))
    host = lad.solve_locus_batched(Xh, Yh, Lh)
    for f in ("beta", "objective", "iterations", "objective_evals", "converged", "status", "descents", "steps"):
        assert np.array_equal(np.asarray(getattr(host, f)), getattr(dev, f).cpu().numpy()), f
    idx = np.concatenate([np.arange(0, 64), np.arange((1 << 18) - 32, (1 << 18) + 32), np.arange(B - 64, B)])
    o = oracle.solve_locus_batch(Xh[idx], Yh[idx], Lh[idx], nthreads=4)
    assert np.array_equal(np.asarray(host.objective)[idx], o["objective"])
    assert np.array_equal(np.asarray(host.beta)[idx], o["beta"])


@pytest.mark.parametrize("shape", [(10, 2), (30, 5), (40, 3)])
def test_tiny_weight_totals_with_a_lowered_lambda_floor(oracle, shape):
    """Weights so small that the fixed-point scale 2^30 / total would overflow (possible only with a
    lambda_floor far below the default): the median tests must accept nothing there and the exact
    order decides, on the thread, warp and block kernels alike."""
    n, p = shape
    rng = np.random.default_rng(31)
    X = rng.standard_normal((24, n, p)) * 1e-304
    Y = rng.standard_normal((24, n)) * 1e-304
    L = np.full(24, 1e-306)
    o = oracle.solve_locus_batch(X, Y, L, lambda_floor=1e-310, nthreads=4)
    r = lad.solve_locus_batched(X, Y, L, lambda_floor=1e-310)
    assert np.array_equal(np.asarray(r.status), o["status"])
    assert np.array_equal(np.asarray(r.objective), o["objective"])
    assert np.array_equal(np.asarray(r.beta), o["beta"])
    assert np.array_equal(np.asarray(r.steps), o["steps"])
