"""GPU: the axis-wise-minimum certificate and locus sampling against reference goldens.

Goldens (tests/golden/curve.npz, oracle/gen_golden.py gen_curve) come from the unmodified
reference: ccd.is_axiswise_minimum on 360 certified / nudged / random vectors (with and
without skip) and locus.sample_locus on 16 problems.  Bar: identical booleans; sampled
points bit-exact (t, beta, value, convergence, evaluation counts).
"""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2510_15649_b200 as lad  # noqa: E402


def test_certificate_batched_matches_reference():
    g = load_golden("curve")
    ms, ds = g["m"], g["d"]
    for (m, d) in sorted(set(zip(ms.tolist(), ds.tolist()))):
        rows = np.nonzero((ms == m) & (ds == d))[0]
        got = lad.axiswise_minimum_batched(np.ascontiguousarray(g["x"][rows][:, :m, :d]),
                                           np.ascontiguousarray(g["y"][rows][:, :m]), g["lam"][rows],
                                           np.ascontiguousarray(g["beta"][rows][:, :d]), skip=g["skip"][rows])
        assert np.array_equal(got, g["certified"][rows].astype(bool)), (m, d)


def test_sample_locus_batched_matches_reference():
    g = load_golden("curve")
    for k in range(len(g["s_lam"])):
        m, d, n = int(g["s_m"][k]), int(g["s_d"][k]), int(g["s_n"][k])
        X, Y = g["s_x"][k, :m, :d][None], g["s_y"][k, :m][None]
        br = lad.Bracket(*g["s_bracket"][k])
        s = lad.sample_locus_batched(X, Y, np.array([g["s_lam"][k]]), int(g["s_axis"][k]), br, n)
        assert np.array_equal(s["t"], g["s_t"][k, :n])
        assert np.array_equal(s["beta"][0], g["s_beta"][k, :n, :d]), k
        assert np.array_equal(s["value"][0], g["s_value"][k, :n]), k
        assert np.array_equal(s["inner_converged"][0], g["s_conv"][k, :n])
        assert np.array_equal(s["inner_evals"][0], g["s_evals"][k, :n])


def test_single_problem_mirrors_follow_reference_tests():
    """test_ccd.py:75-104 and test_locus.py:36-44, 108-119 restated on the GPU mirrors."""
    k = load_golden("kat")
    spec = lad.ProblemSpec(lad.Dataset(k["stall_x"], k["stall_y"]), float(k["stall_lam"]))
    stalled = lad.solve_ccd(spec)
    assert stalled.converged and lad.is_axiswise_minimum(spec, stalled.beta)
    nudged = lad.perturb_restart(spec, stalled.beta, axis=0, delta=0.5)
    assert nudged.converged and lad.is_axiswise_minimum(spec, nudged.beta)
    # a frozen axis is never moved and the point is certified with skip
    start = lad.Coefficients(np.array([0.0, 1.5]))
    res = lad.ccd_descend(spec, start, lad.CcdConfig(frozen_axis=1))
    assert res.beta.beta[1] == 1.5 and lad.is_axiswise_minimum(spec, res.beta, skip=1)
    # curve points are axis-wise minima off the frozen axis
    axis = lad.default_outer_axis(spec.data)
    for t in (0.3, 0.3 + 1e-3):
        pt = lad.locus_value(spec, axis, t)
        assert pt.inner_converged and lad.is_axiswise_minimum(spec, pt.beta, skip=axis)
    # d = 1: the median certifies, a 1e-5 nudge does not
    x = k["stall_x"][:, :1]
    s1 = lad.ProblemSpec(lad.Dataset(x, k["stall_y"]), 0.2)
    b = lad.solve_ccd(s1).beta.beta
    assert lad.is_axiswise_minimum(s1, b) and not lad.is_axiswise_minimum(s1, b + 1e-5)
    with pytest.raises(lad.InvalidInputError):
        lad.sample_locus(s1, 0, lad.Bracket(-1.0, 1.0), 2)
    pts = lad.sample_locus(s1, 0, lad.Bracket(-3.0, 3.0), 9)
    assert len(pts) == 9 and pts[0].t == -3.0 and pts[-1].t == 3.0


def test_certificate_invalid_and_skip_vector():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((4, 8, 3))
    Y = rng.standard_normal((4, 8))
    beta = np.zeros((4, 3))
    beta[2, 0] = np.nan
    with pytest.raises(lad.InvalidInputError):
        lad.axiswise_minimum_batched(X, Y, np.full(4, 0.1), beta)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    out = lad.axiswise_minimum_batched(Xd, Yd, torch.full((4,), 0.1, dtype=torch.float64, device="cuda"),
                                       torch.from_numpy(beta).cuda(), skip=torch.tensor([0, 1, 2, -1]).cuda())
    assert out.dtype == torch.bool and out.shape == (4,)
