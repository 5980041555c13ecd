"""Host-side logic of the device pipeline (no GPU needed)."""

from __future__ import annotations

import numpy as np

from paper_2212_10733_b200 import engine as E


def _scalar_heap(st, depth):
    n = 1 << depth
    cand = np.full(n, np.nan)
    nodes = [None] * n
    nodes[1] = st
    for i in range(1, n):
        q = nodes[i]
        if q is None or q.stage == "done":
            continue
        cand[i] = float(q.query())
        if 2 * i < n:
            nodes[2 * i] = q.advance(True)
            nodes[2 * i + 1] = q.advance(False)
    return cand


def test_search_heap_matches_the_scalar_bisection():
    """The vectorised lookahead tree equals residual.find_error_bound's
    sequence of candidate bounds (residual.py:129-173) on every path."""
    rng = np.random.default_rng(0)
    seen = set()
    roots = []
    for _ in range(60):
        st = E._Search("hi", float(rng.uniform(1e-3, 1e15)))
        for _ in range(int(rng.integers(0, 24))):
            if st.stage == "done":
                break
            st = st.advance(bool(rng.integers(0, 2)))
        roots.append(st)
    low = E._Search("hi", 3.0)
    while low.stage != "low":
        low = low.advance(False)  # every bound rejected: the final lossless probe
    roots.append(low)
    for st in roots:
        if st.stage == "done":
            continue
        seen.add(st.stage)
        for depth in (1, 2, 5, 8):
            a, b = E._search_heap([st], depth)[0], _scalar_heap(st, depth)
            assert np.array_equal(np.isnan(a), np.isnan(b))
            assert np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])
    assert {"hi", "bis", "low"} <= seen


def test_search_walk_reaches_the_reference_bound():
    """Walking the heap with a monotone pass predicate gives the bound the
    sequential bisection returns."""
    for eb_hi, thr in [(1.0, 0.3), (5e9, 1e3), (1.0, 2.0), (1.0, 1e-9)]:
        st = E._Search("hi", eb_hi)
        seq = st
        while seq.stage != "done":
            seq = seq.advance(float(seq.query()) <= thr)
        while st.stage != "done":
            cand = E._search_heap([st], E.LOOKAHEAD)[0]
            node = 1
            for _ in range(E.LOOKAHEAD):
                if st.stage == "done":
                    break
                assert st.query() == cand[node]
                ok = cand[node] <= thr
                st = st.advance(ok)
                node = 2 * node + (0 if ok else 1)
        assert st.result == seq.result


def test_search_heap_groups_many_searches():
    rng = np.random.default_rng(1)
    sts = []
    for _ in range(12):
        st = E._Search("hi", float(rng.uniform(1e-3, 1e15)))
        for _ in range(int(rng.integers(0, 3))):
            st = st.advance(False)
        sts.append(st)
    got = E._search_heap(sts, 7)
    for row, st in zip(got, sts):
        want = _scalar_heap(st, 7)
        assert np.array_equal(np.isnan(row), np.isnan(want))
        assert np.array_equal(row[~np.isnan(row)], want[~np.isnan(want)])


def test_archive_bound_covers_every_fixture_archive():
    """compress() sizes the archive bytes object by _archive_bound and shrinks
    it in place: the bound must hold for every reference archive."""
    import json
    from types import SimpleNamespace

    from paper_2212_10733_b200 import PipelineConfig, fdata, pipeline
    from paper_2212_10733_b200.container import ArchivePreamble
    from tests.golden_util import GOLDEN

    grid = fdata.make_grid(39, 39, 5.0, 5.0, 1.0)
    for path in sorted(GOLDEN.glob("*.json")):
        meta = json.loads(path.read_text())
        if "runs" not in meta:
            continue
        ds = SimpleNamespace(grid=grid, n_planes=meta["P"], n_nodes=meta["N"])
        for run in meta["runs"]:
            c = dict(run["cfg"])
            c.pop("newton", None)
            cfg = PipelineConfig(**c)
            head = ArchivePreamble(n_shards=cfg.shards, decomp_mode=cfg.mode,
                                   n_planes=ds.n_planes, n_nodes=ds.n_nodes, grid=grid,
                                   timestep=0, tau=cfg.tau, seed=cfg.seed,
                                   config_digest=cfg.digest()).pack()
            bound = pipeline._archive_bound(ds, cfg, cfg.shards, len(head))
            assert run["archive_len"] <= bound, (path.name, run["archive_len"], bound)


def test_mapped_file_cache_follows_inode_and_size(tmp_path):
    """hostio.mapped_file: one cached shared mapping per (inode, size); a
    rewrite through it lands in the file, a size change maps afresh, and
    release_maps drops every mapping."""
    import os

    from paper_2212_10733_b200 import hostio
    path = tmp_path / "out.bin"
    fd = os.open(path, os.O_RDWR | os.O_CREAT, 0o644)
    try:
        os.ftruncate(fd, 4096)
        v = hostio.mapped_file(fd, 4096)
        v[:4] = np.frombuffer(b"abcd", np.uint8)
        assert hostio.mapped_file(fd, 4096).ctypes.data == v.ctypes.data  # cached
        del v
        os.ftruncate(fd, 8192)
        w = hostio.mapped_file(fd, 8192)
        assert len(w) == 8192 and bytes(w[:4]) == b"abcd"
        del w
        st = os.fstat(fd)
        assert [k for k in hostio._MAPS if k[:2] == (st.st_dev, st.st_ino)] == [
            (st.st_dev, st.st_ino, 8192)]
    finally:
        os.close(fd)
        hostio.release_maps()
    assert hostio._MAPS == {}
    assert path.read_bytes()[:4] == b"abcd"
