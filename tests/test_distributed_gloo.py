"""N>1 host logic on CPU: 2 gloo ranks split the shards of a real archive and
must reproduce the single-process archive offsets and bytes, and the
reduced report statistics."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from paper_2212_10733_b200 import container, distributed
from tests import golden_util as G


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_, blobs, head_len, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rp = distributed.plan(1, 64, len(blobs), "col")
    local = [len(blobs[i]) for i in rp.mine]
    sizes, offs = distributed.exchange_sizes(rp, local, head_len)
    stats = distributed.reduce_stats({
        "n": ("sum", [len(rp.mine)]),
        "big": ("max", [max(local) if local else 0]),
        "small": ("min", [min(local) if local else 1e30]),
    })
    got = distributed.gather_bytes(b"".join(blobs[i] for i in rp.mine))
    q.put((rank, rp.mine, rp.node_range, sizes.tolist(), offs.tolist(),
           {k: v.tolist() for k, v in stats.items()}, None if got is None else b"".join(got)))
    dist.destroy_process_group()


def test_two_rank_archive_assembly_matches_single_process():
    meta, _ = G.load("tiny")
    ds, same = G.corpus("tiny")
    run = meta["runs"][0]
    cfg = G.oracle_cfg(run)
    # 4 shards so each rank owns two
    cfg4 = port.Cfg(**{**cfg.__dict__, "shards": 4})
    models = G.models("tiny") * 4
    arc, _, outs = port.compress(ds.data, G.oracle_grid(), cfg4, models)
    blobs = [o.blob for o in outs]
    pre, _ = container.ArchivePreamble.unpack(arc)
    head_len = pre.size()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_, blobs, head_len, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, mine0, nr0, sizes0, offs0, st0, body0), (_, mine1, nr1, sizes1, offs1, st1, body1) = res
    assert mine0 == [0, 1] and mine1 == [2, 3]
    assert nr0 == (0, 32) and nr1 == (32, 64)
    assert sizes0 == sizes1 == [len(b) for b in blobs]
    assert offs0 == offs1 == container.archive_offsets(head_len, [len(b) for b in blobs])
    assert st0["n"] == [4.0] and st0["big"] == [max(map(len, blobs))]
    assert st0["small"] == [min(map(len, blobs))]
    # rank 0 gathers the blobs: preamble + index + blobs is the single-process archive
    idx = np.asarray(offs0, dtype="<u8").tobytes()
    assert arc[:head_len] + idx + body0 == arc
    assert body1 is None
