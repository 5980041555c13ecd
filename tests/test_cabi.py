"""CPU-side checks of the C-ABI boundary (no GPU needed)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "mlk_b200.h"
LIB = ROOT / "paper_2212_10733_b200" / "libmlk_b200.so"


def declared():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(mlk_\w+)\(", txt, re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "mlk_project" in names and "mlk_stage1" in names and "mlk_newton_solve_batch" in names


def test_library_exports_every_declared_symbol():
    if not LIB.exists():
        pytest.skip("library not built (run __graft_entry__.build())")
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (mlk_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, f"declared but not exported: {missing}"
    ctypes.CDLL(str(LIB))  # loads without a GPU


def test_python_binding_covers_header():
    from paper_2212_10733_b200 import _lib
    assert set(declared()) <= set(_lib.exported_symbols())
