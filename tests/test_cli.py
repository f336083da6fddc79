"""CLI / generator parity with the reference's ``ladlasso`` command line (cli.py, datagen.py, rng.py).

Fixtures: tests/golden/cli.json holds transcripts of the unmodified reference
CLI (oracle/gen_golden.py gen_cli); kat.npz / acceptance.npz hold reference
generator outputs.  CPU tests pin the generator, CSV I/O, the check-task
picker and argument parsing; GPU tests run `solve` / `check` / `bench` on the
device and compare every non-timing field with the reference transcript.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from paper_2510_15649_b200 import cli
from paper_2510_15649_b200.errors import InvalidInputError
from paper_2510_15649_b200.synth import (GenSpec, Pcg32, generate, metadata_path, read_dataset_csv, read_metadata,
                                         write_dataset_csv)


def _fixture():
    with open(os.path.join(GOLDEN, "cli.json")) as fh:
        return json.load(fh)


def _table(text):
    lines = text.strip("\n").split("\n")
    header = lines[0].split(",")
    return header, [dict(zip(header, ln.split(","))) for ln in lines[1:]]


# ---------------------------------------------------------------------------
# generator (rng.py / datagen.py)
# ---------------------------------------------------------------------------

def test_pcg32_stream_golden():
    k = load_golden("kat")
    g = Pcg32(42, stream=54)
    assert [g._step() for _ in range(200)] == k["pcg32_seed42"].tolist()
    for a in range(8):
        g = Pcg32(0x5EED + a)
        assert [g._step() for _ in range(64)] == k["pcg32_fan"][a].tolist()


def test_pcg32_helpers():
    g = Pcg32(9)
    assert all(0 <= g.below(7) < 7 for _ in range(500))
    assert all(0.0 <= g.uniform() < 1.0 for _ in range(500))
    assert all(2.0 <= g.uniform_in(2.0, 3.0) < 3.0 for _ in range(100))
    with pytest.raises(ValueError):
        g.below(0)
    # Box-Muller pairs: the spare is served by the next call
    a, b = Pcg32(1), Pcg32(1)
    assert a.normals(5) == [b.normal() for _ in range(5)]


def test_generate_matches_reference_stall_fixture():
    """fixtures.py:15: GenSpec(m=5, d=2, noise_sigma=3, outlier_fraction=0.2, seed=0)."""
    k = load_golden("kat")
    data, _ = generate(GenSpec(m=5, d=2, noise_sigma=3.0, outlier_fraction=0.2, seed=0))
    assert np.array_equal(data.x, k["stall_x"]) and np.array_equal(data.y, k["stall_y"])


def test_generate_matches_reference_acceptance_grid():
    """test_acceptance.py grid: seeds 9000+i over (d, m, lambda) -- every byte of x and y."""
    a = load_golden("acceptance")
    import itertools

    grid = list(itertools.product((1, 2, 3), range(4, 13), (0.01, 0.1, 1.0)))
    for i in range(200):
        d, m, _ = grid[i % len(grid)]
        data, _ = generate(GenSpec(m=m, d=d, noise_sigma=1.0, outlier_fraction=0.2, seed=9000 + i))
        assert np.array_equal(data.x, a["x"][i, :m, :d]), i
        assert np.array_equal(data.y, a["y"][i, :m]), i


@pytest.mark.parametrize("kw,msg", [(dict(m=0, d=1), "need m >= 1"), (dict(m=3, d=2, n_informative=3), "n_informative"),
                                    (dict(m=3, d=2, true_coefficients=(1.0,)), "length d"),
                                    (dict(m=3, d=1, noise_sigma=-1.0), "noise_sigma"),
                                    (dict(m=3, d=1, outlier_fraction=1.0), "outlier_fraction"),
                                    (dict(m=3, d=1, outlier_scale=0.5), "outlier_scale")])
def test_genspec_validation(kw, msg):
    with pytest.raises(InvalidInputError, match=msg):
        GenSpec(**kw)


def test_generate_true_coefficients_and_sparsity():
    data, beta = generate(GenSpec(m=6, d=3, true_coefficients=(1, 0, -2), noise_sigma=0.0))
    assert beta.beta.tolist() == [1.0, 0.0, -2.0]
    assert np.array_equal(data.y, data.x @ np.array([1.0, 0.0, -2.0]) + 0.0 * data.y)
    _, b2 = generate(GenSpec(m=6, d=4, n_informative=2, seed=3))
    assert b2.beta[2:].tolist() == [0.0, 0.0] and (b2.beta[:2] >= 1).all() and (b2.beta[:2] < 10).all()


# ---------------------------------------------------------------------------
# dataset CSV + sidecar
# ---------------------------------------------------------------------------

def test_gen_command_matches_reference_bytes(tmp_path, capsys):
    for case in _fixture()["gen"]:
        path = tmp_path / "g.csv"
        code = cli.main(["gen", str(path)] + case["argv"])
        assert code == case["code"] == 0
        assert capsys.readouterr().out.replace(str(path), "PATH") == case["stdout"].split(" to ")[0] + " to PATH\n"
        assert path.read_text() == case["csv"]
        assert open(metadata_path(path)).read() == case["meta"]
        meta = read_metadata(path)
        assert len(meta["true_beta"]) == meta["d"]


def test_csv_round_trip(tmp_path):
    data, _ = generate(GenSpec(m=9, d=4, outlier_fraction=0.3, seed=21))
    p = tmp_path / "d.csv"
    write_dataset_csv(data, p)
    back = read_dataset_csv(p)
    assert np.array_equal(back.x, data.x) and np.array_equal(back.y, data.y)


@pytest.mark.parametrize("text,msg", [("", "empty file"), ("x1,z\n1,2\n", "header row 1"), ("y\n1\n", "header row 1"),
                                      ("x1,y\n", "no data rows"), ("x1,y\n1,2,3\n", "row 2 has 3 fields"),
                                      ("x1,y\n1,2\nfoo,3\n", "row 3, column x1: cannot parse 'foo'")])
def test_csv_errors(tmp_path, text, msg):
    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(InvalidInputError, match=msg):
        read_dataset_csv(p)


def test_csv_blank_lines_skipped(tmp_path):
    p = tmp_path / "b.csv"
    p.write_text("x1,x2,y\n1,2,3\n\n4,5,6\n")
    ds = read_dataset_csv(p)
    assert ds.x.tolist() == [[1, 2], [4, 5]] and ds.y.tolist() == [3, 6]


# ---------------------------------------------------------------------------
# argument parsing / host logic
# ---------------------------------------------------------------------------

def test_parse_int_set():
    assert cli._parse_int_set("1,2,5") == [1, 2, 5]
    assert cli._parse_int_set("4-12") == list(range(4, 13))
    assert cli._parse_int_set("1,4-6,2") == [1, 2, 4, 5, 6]
    with pytest.raises(Exception):
        cli._parse_int_set(",")
    assert cli._parse_float_list("0.01,0.1,1") == [0.01, 0.1, 1.0]


def test_parser_defaults_match_reference():
    p = cli.build_parser()
    a = p.parse_args(["check"])
    assert (a.d, a.m, a.lam, a.n_instances, a.seed, a.noise_sigma, a.outlier_fraction) == (
        [1, 2, 3], list(range(4, 13)), [0.01, 0.1, 1.0], 50, 0, 1.0, 0.2)
    assert (a.outer_tol, a.inner_tol, a.probes) == (1e-9, 1e-10, 8)
    b = p.parse_args(["bench"])
    assert (b.d, b.m, b.repeats, b.lam, b.noise_sigma, b.outlier_fraction, b.out) == (
        [1, 2, 3, 4, 5], [10, 30], 5, 0.1, 0.0, 0.0, "bench.csv")
    s = p.parse_args(["solve", "x.csv", "--lambda", "0.5"])
    assert (s.solver, s.lambda_floor) == ("locus_ternary", 1e-9)


def test_check_task_picker_matches_reference():
    args = cli.build_parser().parse_args(["check"])
    tasks = cli.check_tasks(args)
    got = [[t["genspec"]["d"], t["genspec"]["m"], t["lam"], t["genspec"]["seed"]] for t in tasks]
    assert got == _fixture()["check_tasks_seed0"]


def test_unknown_bench_solver_is_an_input_error(tmp_path, capsys):
    assert cli.main(["bench", "--solvers", "simplex2", "--out", str(tmp_path / "b.csv")]) == 1
    assert "unknown solver" in capsys.readouterr().err


def test_solve_missing_file_exit_1(tmp_path, capsys):
    assert cli.main(["solve", str(tmp_path / "nope.csv"), "--lambda", "0.1"]) == 1
    assert capsys.readouterr().err.startswith("error:")


def test_medians_path():
    assert cli._medians_path("out/bench.csv") == "out/bench_medians.csv"
    assert cli._medians_path("bench") == "bench_medians"


# ---------------------------------------------------------------------------
# GPU: the subcommands against the reference transcripts
# ---------------------------------------------------------------------------

def _strip_wall(text):
    keep = []
    for line in text.strip("\n").split("\n"):
        if line.startswith("wall time:"):
            continue
        if line.startswith("RESULT "):
            line = " ".join(f for f in line.split(" ") if not f.startswith("wall_time_s="))
        keep.append(line)
    return keep


@pytest.mark.gpu
def test_solve_matches_reference_transcript(tmp_path, capsys):
    fx = _fixture()
    path = tmp_path / "s.csv"
    path.write_text(fx["solve_csv"])
    for case in fx["solve"]:
        code = cli.main(["solve", str(path)] + case["argv"])
        out = capsys.readouterr().out
        assert code == case["code"], case["argv"]
        assert _strip_wall(out) == _strip_wall(case["stdout"]), case["argv"]


@pytest.mark.gpu
def test_check_matches_reference_transcript(tmp_path, capsys):
    for case in _fixture()["check"]:
        out = tmp_path / "c.csv"
        code = cli.main(["check"] + case["argv"] + ["--out", str(out)])
        stdout = capsys.readouterr().out
        assert code == case["code"], case["argv"]
        assert stdout.strip().split("\n") == case["stdout"].strip().split("\n")
        rh, rrows = _table(case["csv"])
        mh, mrows = _table(out.read_text())
        assert mh == rh
        cols = [c for c in mh if not c.startswith("time_")]
        assert [[r[c] for c in cols] for r in mrows] == [[r[c] for c in cols] for r in rrows]


@pytest.mark.gpu
def test_solve_dump_lp_matches_reference_bytes(tmp_path, capsys):
    fx = _fixture()
    path = tmp_path / "s.csv"
    path.write_text(fx["solve_csv"])
    lp_path = tmp_path / "s.lp"
    assert cli.main(["solve", str(path), "--lambda", "0.3", "--solver", "lp", "--dump-lp", str(lp_path)]) == 0
    capsys.readouterr()
    assert lp_path.read_text() == fx["dump_lp"]


@pytest.mark.gpu
def test_check_default_sweep_passes(capsys):
    """The reference's default sweep (50 instances, seed 0) -- every locus gap below 1e-5 (exit 0)."""
    assert cli.main(["check"]) == 0
    assert "[FAIL]" not in capsys.readouterr().out


@pytest.mark.gpu
def test_bench_matches_reference_transcript(tmp_path, capsys):
    case = _fixture()["bench"]
    out = tmp_path / "b.csv"
    assert cli.main(["bench"] + case["argv"] + ["--out", str(out)]) == case["code"] == 0
    capsys.readouterr()
    rh, rrows = _table(case["csv"])
    mh, mrows = _table(out.read_text())
    assert mh == rh
    cols = [c for c in mh if c != "wall_time_s"]
    assert [[r[c] for c in cols] for r in mrows] == [[r[c] for c in cols] for r in rrows]
    rh, rmed = _table(case["medians"])
    mh, mmed = _table((tmp_path / "b_medians.csv").read_text())
    assert mh == rh
    cols = ["solver", "d", "m", "median_objective"]
    assert [[r[c] for c in cols] for r in mmed] == [[r[c] for c in cols] for r in rmed]
