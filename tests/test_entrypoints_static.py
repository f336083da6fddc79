"""bench.py and __graft_entry__.py run only on the GPU box: check them statically here.

Every name a function reads must be a parameter, a local, a module-level name, or a builtin
(a NameError in a rarely used bench mode would otherwise surface only at round end)."""

import builtins
import os
import symtable

import pytest

from conftest import ROOT


def _undefined(path):
    src = open(path).read()
    top = symtable.symtable(src, os.path.basename(path), "exec")
    module = {s.get_name() for s in top.get_symbols() if s.is_assigned() or s.is_imported()}
    known = module | set(dir(builtins)) | {"__file__"}
    bad = []

    def walk(t, outer):
        own = {s.get_name() for s in t.get_symbols() if s.is_assigned() or s.is_imported() or s.is_parameter()}
        scope = outer | own
        for s in t.get_symbols():
            n = s.get_name()
            if s.is_referenced() and n not in scope and n not in known:
                bad.append((t.get_name(), n))
        for c in t.get_children():
            walk(c, scope)

    walk(top, set())
    return bad


@pytest.mark.parametrize("name", ["bench.py", "__graft_entry__.py"])
def test_no_undefined_names(name):
    assert _undefined(os.path.join(ROOT, name)) == []


def test_bench_parses_every_mode():
    import subprocess
    import sys

    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True)
    assert out.returncode == 0 and "--solver" in out.stdout and "--dtype" in out.stdout and "--impl" in out.stdout
