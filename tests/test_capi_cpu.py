"""CPU: the C-ABI library loads and exports every symbol include/*.h declares,
with no compute calls (no GPU here); Python-side validation mirrors the
reference messages."""
import ctypes
import os
import re

import pytest

import paper_2005_10123_b200 as pk
from paper_2005_10123_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("sthk.h", "sthk_sim.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"\b(sthk_[a-z_0-9]+)\s*\(", src))
    return names


def test_library_exports_all_declared_symbols():
    lib = ctypes.CDLL(_lib.lib_path())
    names = declared_symbols()
    assert len(names) >= 18
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert declared_symbols() <= bound


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.lib_path()} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_version_string():
    lib = pk.load_library()
    assert b"sm_100a" in lib.sthk_version()


def test_params_validation_messages():
    with pytest.raises(ValueError, match="Params: mu0, tauX, tauT, omega, h must be positive"):
        pk.Params(omega=-1.0).validate()
    pk.Params(theta=0.0).validate()


def test_eventset_validation_messages():
    with pytest.raises(ValueError, match="need at least one event"):
        pk.EventSet([], [], [])
    with pytest.raises(ValueError, match="times not sorted at index 1"):
        pk.EventSet([0, 1], [0, 1], [1.0, 0.5])
    with pytest.raises(ValueError, match="negative time at index 0"):
        pk.EventSet([0, 1], [0, 1], [-0.5, 1.0])
    with pytest.raises(ValueError, match="windowEnd precedes last event"):
        pk.EventSet([0, 1], [0, 1], [0.5, 1.0], 0.9)
    ev = pk.EventSet.sortedByTime([0, 1, 2], [0, 1, 2], [3.0, 1.0, 2.0])
    assert list(ev.ts()) == [1.0, 2.0, 3.0] and list(ev.xs()) == [1, 2, 0]


def test_eventset_first_failure_in_reference_order():
    # types.hpp:90-104 stops at the first index with any failure
    with pytest.raises(ValueError, match="times not sorted at index 1"):
        pk.EventSet([0, 1, 2], [0, 1, 2], [1.0, 0.5, float("nan")])
    with pytest.raises(ValueError, match="non-finite entry at index 1"):
        pk.EventSet([0, float("inf"), 2], [0, 1, 2], [1.0, 0.5, 0.2])
    with pytest.raises(ValueError, match="negative time at index 1"):
        pk.EventSet([0, 1], [0, 1], [1.0, -1.0])


def test_stats_struct_layout_matches_header(tmp_path):
    """The Python mirror of sthk_stats (ctypes) has the C header's size and
    field offsets: compiled here with gcc against include/sthk.h."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    fields = [f for f, _ in _lib.StatsStruct._fields_]
    src = ["#include <stddef.h>", "#include <stdio.h>", '#include "sthk.h"', "int main(void) {",
           '  printf("%zu\\n", sizeof(sthk_stats));']
    src += ['  printf("%%zu\\n", offsetof(sthk_stats, %s));' % f for f in fields]
    src += ["  return 0;", "}"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    out = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    assert out[0] == ctypes.sizeof(_lib.StatsStruct)
    for f, off in zip(fields, out[1:]):
        assert getattr(_lib.StatsStruct, f).offset == off, f
