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


def test_host_exception_entries_and_fill_layout(monkeypatch):
    """compress()'s host fill of the exception sections (no GPU): the holes
    and the bytes written by mlk_host_exception_entries are the container's
    exception entries (<I member index> + the raw histogram) for every shard."""
    if not LIB.exists():
        pytest.skip("library not built (run __graft_entry__.build())")
    import numpy as np
    from types import SimpleNamespace

    from paper_2212_10733_b200 import _lib, fdata, pipeline
    from paper_2212_10733_b200.decomp import partition

    so = ctypes.CDLL(str(LIB))
    so.mlk_host_exception_entries.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64,
                                                                      ctypes.c_int32]
    monkeypatch.setattr(_lib, "lib", lambda: so)
    P, N, D = 3, 10, 39 * 39
    grid = fdata.make_grid(39, 39, 5.0, 5.0, 1.0)
    rng = np.random.default_rng(3)
    ds = fdata.FDataset(grid=grid, data=rng.random((P, N, 39, 39)), timestep=0)
    shards = partition(P, N, 2, "col")
    row = 4 + 8 * D
    members = [np.array([0, 4, 13], dtype=np.int64), np.array([2, 14], dtype=np.int64)]
    offs = [100, 100 + 3 * row + 50]
    out = SimpleNamespace(exceptions=list(zip(offs, members)))
    holes, fill = pipeline._exception_fills(out, shards, ds.data, ds)
    assert holes == [(offs[0], 3 * row), (offs[1], 2 * row)]
    buf = np.zeros(offs[1] + 2 * row + 10, dtype=np.uint8)
    for o, n in holes:
        for j in fill(buf, o, n):
            j.result()
    for (off, mem), sh in zip(zip(offs, members), shards):
        (p0, _), (x0, x1) = sh.planes_range, sh.nodes_range
        for k, g in enumerate(mem):
            e = buf[off + k * row:off + (k + 1) * row]
            assert int.from_bytes(e[:4].tobytes(), "little") == g
            want = ds.data[p0 + g // (x1 - x0), x0 + g % (x1 - x0)]
            assert e[4:].tobytes() == want.tobytes()
    assert not buf[:offs[0]].any() and not buf[offs[1] + 2 * row:].any()
