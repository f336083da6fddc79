"""The C ABI library builds for sm_100a, loads without a GPU, and exports every declared symbol."""

import ctypes as C
import os
import re

import pytest

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "ladlasso_b200.h")).read()
    return sorted(set(re.findall(r"\b(lad_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_binding_table():
    from paper_2510_15649_b200 import _lib

    assert sorted(_lib.SYMBOLS) == _declared()


def test_library_exports_every_declared_symbol():
    from paper_2510_15649_b200 import _lib

    L = _lib.load(build_if_missing=True)
    for name in _declared():
        assert hasattr(L, name), name
    assert L.lad_version() >= 100
    p = _lib.LocusParams()
    L.lad_default_params(C.byref(p))
    # LocusConfig()/CcdConfig() defaults (locus.py:52-58, ccd.py:55-59, model.py:27)
    assert (p.outer_axis, p.outer_search, p.outer_tolerance, p.outer_probes, p.outer_max_iterations) == \
        (-1, 0, 1e-9, 8, 200)
    assert (p.inner_sweep_tol, p.inner_max_sweeps, p.lambda_floor) == (1e-10, 500, 1e-9)


def test_library_is_sm100a_code():
    from paper_2510_15649_b200 import _lib
    import subprocess

    path = _lib.lib_path()
    if not os.path.exists(path):
        pytest.skip("library not built")
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_validation_raises_reference_errors():
    import numpy as np
    import paper_2510_15649_b200 as lad

    with pytest.raises(lad.InvalidInputError):
        lad.LocusConfig(outer_search="golden")
    with pytest.raises(lad.InvalidInputError):
        lad.CcdConfig(max_sweeps=0)
    with pytest.raises(lad.InvalidInputError):
        lad.Bracket(1.0, 1.0)
    with pytest.raises(lad.DimensionMismatchError):
        lad.Dataset(np.ones((3, 2)), np.ones(4))
    with pytest.raises(lad.InvalidInputError):
        lad.Dataset(np.array([[np.nan]]), np.ones(1))
    with pytest.raises(lad.InvalidInputError):
        lad.ProblemSpec(lad.Dataset(np.ones((2, 1)), np.ones(2)), -1.0)
    from paper_2510_15649_b200.config import locus_params

    with pytest.raises(lad.InvalidInputError):
        locus_params(lad.LocusConfig(outer_probes=2))
    with pytest.raises(lad.InvalidInputError):
        locus_params(lad.LocusConfig(outer_axis=3), d=2)
    with pytest.raises(lad.InvalidInputError):
        locus_params(lad.LocusConfig(inner=lad.CcdConfig(line_search="ternary")))


def test_package_namespace_is_consistent():
    """The reference's names resolve to the reference's objects (no submodule shadowing)."""
    import types

    import paper_2510_15649_b200 as lad
    from paper_2510_15649_b200 import configgen, synth

    assert lad.generate is synth.generate and callable(lad.generate)
    assert isinstance(configgen, types.ModuleType) and hasattr(configgen, "CONFIG_SHAPES")
    for name in lad.__all__:
        assert not isinstance(getattr(lad, name), types.ModuleType), name
