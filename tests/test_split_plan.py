"""Host logic of the split decomposition (distributed.SplitPlan +
engine.blob_layout) on CPU: every rank writes only its member range of every
shard, and the pieces of all ranks must tile the single-process blobs byte
for byte.  The device writes are simulated from the oracle's own blobs, so
this pins the layout arithmetic (offsets, prefixes, byte-aligned code
pieces, residual / exception entry placement) independently of the GPU."""

from __future__ import annotations

import os
import socket
import struct
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from paper_2212_10733_b200 import distributed, engine
from tests import golden_util as G

D = 39 * 39


def _parse(blob):
    info, secs = port.split_blob(blob)
    _, codes, pq, res, lam, exc = secs
    _, cnt = struct.unpack_from("<dI", res, 0)
    pos, entries = 12, []
    for _ in range(cnt):
        idx, ln = struct.unpack_from("<II", res, pos)
        entries.append((idx, res[pos:pos + 8 + ln]))
        pos += 8 + ln
    (ne,) = struct.unpack_from("<I", exc, 0)
    excs = []
    for k in range(ne):
        o = 4 + k * (4 + 8 * D)
        excs.append((struct.unpack_from("<I", exc, o)[0], exc[o:o + 4 + 8 * D]))
    return info, secs, entries, excs


@pytest.fixture(scope="module")
def small_blobs():
    meta, _ = G.load("small")
    ds, same = G.corpus("small")
    assert same
    run = meta["runs"][0]
    arc, _, outs = port.compress(ds.data, G.oracle_grid(), G.oracle_cfg(run), G.models("small"))
    return meta, run, [o.blob for o in outs]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_split_pieces_tile_the_single_process_blobs(small_blobs, world):
    meta, run, blobs = small_blobs
    P, N, S = meta["P"], meta["N"], run["cfg"]["shards"]
    cfg = SimpleNamespace(
        latent_dim=run["cfg"]["latent_dim"], pq_bits=run["cfg"]["pq_bits"],
        lambda_precision=run["cfg"]["lambda_precision"])
    L, bits = cfg.latent_dim, cfg.pq_bits
    lb = 4 if cfg.lambda_precision == "f32" else 8
    parsed = [_parse(b) for b in blobs]
    plans = [distributed.SplitPlan(P, N, S, "col", r, world, L, bits) for r in range(world)]
    # ranges: contiguous, covering, byte-aligned code pieces
    for s in range(S):
        cuts = plans[0].bounds[s]
        assert cuts[0] == 0 and cuts[-1] == len(plans[0].shards[s].members)
        assert np.all(np.diff(cuts) >= 0)
        assert all((int(c) * L * bits) % 8 == 0 for c in cuts[:-1])

    def local(r, s):
        a, e = plans[r].range(s)
        ents = [(i, b) for i, b in parsed[s][2] if a <= i < e]
        excs = [(i, b) for i, b in parsed[s][3] if a <= i < e]
        return a, e, ents, excs

    n_all = np.array([[plans[r].range(s)[1] - plans[r].range(s)[0] for s in range(S)]
                      for r in range(world)], dtype=np.int64)
    cnt_all = np.array([[len(local(r, s)[2]) for s in range(S)] for r in range(world)])
    res_all = np.array([[sum(len(b) for _, b in local(r, s)[2]) for s in range(S)]
                        for r in range(world)], dtype=np.int64)
    exc_all = np.array([[len(local(r, s)[3]) for s in range(S)] for r in range(world)])
    region = bytearray(sum(len(b) for b in blobs))
    covered = np.zeros(len(region), dtype=np.int32)
    for r in range(world):
        specs = [SimpleNamespace(n_img=int(n_all[r, s]), rows=39, cols=39) for s in range(S)]
        zlen = np.array([len(b) - 21 for s in range(S) for _, b in local(r, s)[2]],
                        dtype=np.int64)
        ranks = None if world == 1 else dict(rank=r, n=n_all, cnt=cnt_all, res=res_all,
                                               exc=exc_all)
        lay = engine.blob_layout(specs, cfg, D, cnt_all[r], zlen, exc_all[r], ranks)
        # the engine's form: per-shard entry bytes, entry offsets from ent_off
        # + the prefix sums of the entries (done on the device there)
        lay2 = engine.blob_layout(specs, cfg, D, cnt_all[r], None, exc_all[r], ranks,
                                  res_h=res_all[r])
        for k in lay:
            if k not in ("entry_off", "header", "segments"):
                np.testing.assert_array_equal(lay2[k], lay[k], err_msg=k)
        assert lay2["header"] == lay["header"] and lay2["segments"] == lay["segments"]
        zinc = np.concatenate([[0], np.cumsum(zlen + 21)])
        ent_shard = np.repeat(np.arange(S), cnt_all[r])
        base = lay2["ent_off"] - np.concatenate([[0], np.cumsum(res_all[r])[:-1]])
        np.testing.assert_array_equal(zinc[:-1] + base[ent_shard], lay["entry_off"])
        buf = bytearray(lay["total"])
        e0 = 0
        for s in range(S):
            info, secs, _, _ = parsed[s]
            a, e, ents, excs = local(r, s)
            blob = blobs[s]
            if r == 0:
                assert lay["hdr_off"][s] >= 0
                h = lay["hdr_off"][s]
                buf[h:h + 44 + len(secs[0])] = blob[:44 + len(secs[0])]
                buf[lay["pq_off"][s]:lay["pq_off"][s] + len(secs[2])] = secs[2]
                buf[lay["res_pre_off"][s]:lay["res_pre_off"][s] + 12] = secs[3][:12]
                buf[lay["exc_pre_off"][s]:lay["exc_pre_off"][s] + 4] = secs[5][:4]
                assert lay["exc_total"][s] == len(parsed[s][3])
            else:
                assert lay["hdr_off"][s] < 0 and lay["pq_off"][s] < 0
            c_lo = a * L * bits // 8
            c_hi = len(secs[1]) if e == len(plans[0].shards[s].members) else e * L * bits // 8
            buf[lay["codes_off"][s]:lay["codes_off"][s] + c_hi - c_lo] = secs[1][c_lo:c_hi]
            buf[lay["lam_off"][s]:lay["lam_off"][s] + (e - a) * 8 * lb] = \
                secs[4][a * 8 * lb:e * 8 * lb]
            for k, (_, b) in enumerate(ents):
                o = lay["entry_off"][e0 + k]
                buf[o:o + len(b)] = b
            e0 += len(ents)
            for k, (_, b) in enumerate(excs):
                o = lay["exc_base"][s] + 4 + k * (4 + 8 * D)
                buf[o:o + len(b)] = b
        assert list(lay["blob_len"]) == [len(b) for b in blobs]
        if world == 1:
            assert lay["segments"] == [(0, 0, len(region))]
        for lo, goff, n in lay["segments"]:
            region[goff:goff + n] = buf[lo:lo + n]
            covered[goff:goff + n] += 1
    assert np.all(covered == 1), "rank pieces must tile every blob exactly once"
    assert bytes(region) == b"".join(blobs)


def test_split_plan_planes_and_layout_addressing():
    # config 3 shape at 8 GPUs: one plane of every node block per rank
    for r in range(8):
        sp = distributed.SplitPlan(8, 16395, 8, "col", r, 8)
        assert (sp.plane_lo, sp.plane_hi) == (r, r + 1)
        for s, sh in enumerate(sp.shards):
            b = sh.nodes_range[1] - sh.nodes_range[0]
            assert sp.range(s) == (r * b, (r + 1) * b)
        works = engine.split_layout(sp, [SimpleNamespace()] * 8, 39, 39)
        for s, w in enumerate(works):
            # member j0 + j lives at plane (j0 + j) // block of the rank's slab
            g = w.j0
            addr = w.base + (g // w.block) * w.plane_stride + (g % w.block) * D
            assert addr == sp.shards[s].nodes_range[0] * D  # plane r -> slab plane 0
    # one plane, 3 ranks: element split, every rank needs plane 0
    sp = distributed.SplitPlan(1, 1000, 8, "col", 1, 3)
    assert (sp.plane_lo, sp.plane_hi) == (0, 1)
    assert sum(distributed.SplitPlan(1, 1000, 8, "col", r, 3).counts().sum()
               for r in range(3)) == 1000


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sp = distributed.SplitPlan(2, 240, 4, "col", rank, world)
    comm = distributed.Comm(sp)
    # each rank's latents tagged with (shard, member) -> gathered whole shards
    rows = []
    for s in range(4):
        a, e = sp.range(s)
        rows += [[s, j, 0, 0] for j in range(a, e)]
    lat = torch.tensor(rows, dtype=torch.float64)
    gidx, m = comm.gather_index(torch.device("cpu"))
    pad = torch.zeros((m, 4), dtype=torch.float64)
    pad[:lat.shape[0]] = lat
    full = comm.all_gather(pad).reshape(-1, 4).index_select(0, gidx)
    t = torch.tensor([rank + 1.0, -rank], dtype=torch.float64)
    comm.all_reduce_(t, "max")
    c = torch.tensor([rank + 1], dtype=torch.int32)
    comm.all_reduce_(c, "sum")
    q.put((rank, full[:, :2].tolist(), t.tolist(), c.tolist()))
    dist.destroy_process_group()


def test_comm_gathers_whole_shards_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sp = distributed.SplitPlan(2, 240, 4, "col", 0, 2)
    want = [[float(s), float(j)] for s in range(4) for j in range(len(sp.shards[s].members))]
    for _, full, t, c in res:
        assert full == want
        assert t == [2.0, 0.0]
        assert c == [3]
