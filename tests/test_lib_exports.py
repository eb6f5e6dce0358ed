"""libbmv.so loads on a CPU-only host and exports exactly what include/bmv.h declares.

No compute call is made here (no GPU in the build container).
"""

import re
import subprocess
from pathlib import Path

import pytest

from paper_1907_01005_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "bmv.h"


def declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(bmv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_bound_symbols():
    names = declared()
    assert names, "no declarations parsed"
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == names


def test_library_loads_and_exports_every_symbol():
    if not _lib.LIB_PATH.exists():
        pytest.fail("libbmv.so not built (run __graft_entry__.build())")
    lib = _lib.load()
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.bmv_version() >= 1
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    exported = sorted(set(re.findall(r"\sT\s(bmv_[a-z0-9_]+)", out)))
    assert exported == declared()


def test_sm100a_code_present():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_plan_library_exports_every_declared_symbol():
    from paper_1907_01005_b200 import _plan

    header = ROOT / "include" / "bmv_plan.h"
    text = re.sub(r"/\*.*?\*/", "", header.read_text(), flags=re.S)
    names = sorted(set(re.findall(r"\b(bmvp_[a-z0-9_]+)\s*\(", text)))
    assert names
    lib = _plan.load()
    for name in names:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_plan.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert sorted(set(re.findall(r"\sT\s(bmvp_[a-z0-9_]+)", out))) == names
