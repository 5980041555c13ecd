"""Pin the CPU oracle (oracle/) to the real reference's outputs.

The fixtures were produced by tests/golden/make_golden.py from
/root/reference (compiled backend, OPENBLAS_NUM_THREADS=1).  If this host
regenerates a different synthetic corpus (different libm/SIMD), the
pipeline-level checks skip; unit checks run on stored inputs.
"""

from __future__ import annotations

import struct

import numpy as np
import pytest

from oracle import native, port
from tests import golden_util as G

CASES = ["tiny", "small", "rowmode", "cfg1"]


def test_units_kmeans():
    meta, a = G.load("units")
    for t, seed in enumerate(meta["kmeans_seeds"]):
        got = port.kmeans(a[f"km{t}_v"], 16, seed)
        np.testing.assert_array_equal(got, a[f"km{t}_c"])


def test_units_newton_bit_exact():
    meta, a = G.load("units")
    g = G.oracle_grid()
    vol, vpar, vperp = g.cells()
    for t, (st, it) in enumerate(meta["newton_status_iters"]):
        f = a[f"nw{t}_f"].reshape(1, -1)
        q = a[f"nw{t}_q"].reshape(1, 4)
        lam, s, i = native.project_batch(f, vol, vpar, vperp, g.mass, q, 1e-12, 1.0, 50, 1e-13)
        assert (int(s[0]), int(i[0])) == (st, it)
        np.testing.assert_array_equal(lam[0], a[f"nw{t}_lam"])


def test_units_payload_bytes():
    meta, a = G.load("units")
    for t, eb in enumerate(meta["payload_ebs"]):
        r = a[f"pl{t}_r"]
        p = port.payload_lossless(r) if t % 8 == 7 else port.payload_quantized(r, eb)
        assert p == a[f"pl{t}_p"].tobytes()
        back = port.payload_decode(p)
        if t % 8 == 7:
            np.testing.assert_array_equal(back, r)
        else:
            assert np.max(np.abs(back - r)) <= eb * (1 + 1e-12)


def test_units_metrics_and_pack():
    _, a = G.load("units")
    np.testing.assert_array_equal(port.nrmse_rows(a["nr_o"], a["nr_r"]), a["nr_e"])
    np.testing.assert_array_equal(port.moments(a["nr_o"], G.oracle_grid()), a["qoi"])
    assert native.pack_indices(a["pack_idx"], 4) == a["pack_bytes"].tobytes()
    np.testing.assert_array_equal(native.unpack_indices(a["pack_bytes"].tobytes(), 1001, 4),
                                  a["pack_idx"])


def test_pack_known_answer():
    # test_quantizer.py:82-88: [3,3,3,3,10,10,10,10] at 4 bits -> 33 33 AA AA
    assert native.pack_indices(np.array([3, 3, 3, 3, 10, 10, 10, 10]), 4) == bytes(
        [0x33, 0x33, 0xAA, 0xAA])


@pytest.mark.parametrize("name", CASES)
def test_stage_intermediates(name):
    meta, a = G.load(name)
    ds, same = G.corpus(name)
    if not same:
        pytest.skip("this host generates a different synthetic corpus")
    run = meta["runs"][0]
    cfg = G.oracle_cfg(run)
    mods = G.models(name)
    for si, (pl, no) in enumerate(port.shard_members(ds.n_planes, ds.n_nodes, cfg.shards,
                                                     cfg.mode)):
        imgs = ds.data[pl, no]
        w, mean, std = mods[si]
        lat = port.ae_encode(w, mean, std, imgs.reshape(len(imgs), -1))
        np.testing.assert_array_equal(lat, a[f"st_s{si}_latents"])
        cents = port.pq_codebook(lat, 16, port.mix_seed(cfg.seed, si))
        np.testing.assert_array_equal(cents, a[f"st_s{si}_cents"])
        idx = port.pq_indices(cents, lat)
        assert native.pack_indices(idx.reshape(-1), 4) == a[f"st_s{si}_codes"].tobytes()
        rec = port.ae_decode(w, mean, std, port.pq_lookup(cents, idx)).reshape(imgs.shape)
        assert G.sha(rec) == run["shards"][si]["st_recon_sha"]
        err = port.nrmse_rows(imgs, rec)
        np.testing.assert_array_equal(err, a[f"st_s{si}_ae_err"])
        np.testing.assert_array_equal(port.moments(imgs, G.oracle_grid()), a[f"st_s{si}_qoi"])


@pytest.mark.parametrize("name", CASES)
def test_pipeline_archives(name):
    meta, a = G.load(name)
    ds, same = G.corpus(name)
    if not same:
        pytest.skip("this host generates a different synthetic corpus")
    for vi, run in enumerate(meta["runs"]):
        cfg = G.oracle_cfg(run)
        arc, rep, outs = port.compress(ds.data, G.oracle_grid(), cfg, G.models(name))
        assert [len(o.blob) for o in outs] == run["blob_len"], (name, vi)
        assert [G.sha(o.blob) for o in outs] == run["blob_sha"], (name, vi)
        assert G.sha(arc) == run["archive_sha"]
        assert rep["compression_ratio"] == run["ratio"]
        assert rep["exception_count"] == run["exceptions"]
        assert rep["pd_nrmse"] == run["pd_nrmse"]
        if vi == 0:
            dec, _, _ = port.decompress(arc)
            assert G.sha(dec) == run["decomp_sha"]
            for si, o in enumerate(outs):
                assert o.eb == run["shards"][si]["eb"]
                assert o.exceptions == run["shards"][si]["exceptions"]
