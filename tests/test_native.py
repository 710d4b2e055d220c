"""The C-ABI library: builds for sm_100a, loads without a GPU, and exports
every entry point include/kfbi_b200.h declares (CPU only, no compute)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2404_14864_b200 import _native as N

HEADER = os.path.join(ROOT, "include", "kfbi_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(kfbi_\w+)\s*\(", text, re.M)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "kfbi_richardson" in names and "kfbi_box_solve" in names
    assert len(names) >= 18


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(N.EXPORTED_SYMBOLS)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_version_and_error_paths_without_compute():
    lib = N.lib()
    assert b"sm_100a" in lib.kfbi_version()
    # invalid descriptors are rejected before any device call
    desc = N.GridDesc(24, 0.1, 0)
    h = ctypes.c_void_p()
    assert lib.kfbi_plan_create(ctypes.byref(desc), ctypes.byref(h)) == N.E_GRID
    assert "power of two" in N.last_error()
    desc = N.GridDesc(64, -1.0, 0)
    assert lib.kfbi_plan_create(ctypes.byref(desc), ctypes.byref(h)) == N.E_GRID
    with pytest.raises(Exception) as ei:
        N.check(N.E_CUDA)
    assert type(ei.value).__name__ == "DispatchError"


def test_oracle_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_2404_14864_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert not re.search(r"^\s*(from\s+\S*oracle|import\s+\S*oracle)", src, re.M), fn
