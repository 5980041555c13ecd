"""On-device synthetic corpus (csrc/synth.cu, workload.synth.gen_synthetic_device):
the PCG64 jump-ahead restatement on CPU, bit-identical planes on the GPU."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2212_10733_b200 import fdata
from workload import synth


def _grid():
    return fdata.make_grid(39, 39, 5.0, 5.0, 1.0)


def test_pcg64_jump_matches_numpy_advance():
    params = fdata.SyntheticParams(seed=42, rho=0.003)
    words = fdata.synth_pcg_words(params)
    s0 = (int(words[0]) << 64) | int(words[1])
    inc = (int(words[2]) << 64) | int(words[3])
    for k in (1, 2, 31, 32, 1000, 24_936_795 * 63 + 17):
        a, c = fdata.pcg64_affine(k, inc)
        g = fdata._synth_rng(params).bit_generator
        g.advance(k)
        assert (a * s0 + c) & ((1 << 128) - 1) == g.state["state"]["state"]
    a32, c32 = fdata.pcg64_affine(32, inc)
    assert (int(words[4]) << 64 | int(words[5])) == a32
    assert (int(words[6]) << 64 | int(words[7])) == c32


def test_uniform_draw_restatement():
    """draw q = XSL-RR of state s_{q+1}; uniform(-1, 1) = -1 + 2 (x >> 11) 2^-53."""
    params = fdata.SyntheticParams(seed=7, rho=0.01)
    words = fdata.synth_pcg_words(params)
    s0 = (int(words[0]) << 64) | int(words[1])
    inc = (int(words[2]) << 64) | int(words[3])
    want = fdata._synth_rng(params).uniform(-1.0, 1.0, size=100)
    m64 = (1 << 64) - 1
    for q in (0, 1, 5, 99):
        a, c = fdata.pcg64_affine(q + 1, inc)
        s = (a * s0 + c) & ((1 << 128) - 1)
        x = ((s >> 64) ^ s) & m64
        r = s >> 122
        x = ((x >> r) | (x << ((64 - r) & 63))) & m64
        assert -1.0 + 2.0 * ((x >> 11) * (1.0 / 9007199254740992.0)) == want[q]


@pytest.mark.gpu
@pytest.mark.parametrize("P,N,lo,hi,rho", [(1, 64, 0, 1, 0.003), (3, 240, 0, 3, 0.003),
                                            (5, 333, 2, 5, 0.05), (2, 100, 0, 2, 0.0)])
def test_device_planes_bit_identical(P, N, lo, hi, rho):
    import torch
    dev = torch.device("cuda", 0)
    params = fdata.SyntheticParams(seed=42, rho=rho)
    host = synth.gen_synthetic(P, N, _grid(), params).data[lo:hi]
    got = synth.gen_synthetic_device(P, N, _grid(), params, dev, (lo, hi))
    nd = N * 39 * 39
    arr = got.cpu().numpy()
    assert np.array_equal(arr[:(hi - lo) * nd].view(np.uint64),
                          np.ascontiguousarray(host).reshape(-1).view(np.uint64))
    assert np.all(arr[(hi - lo) * nd:] == 0.0)


@pytest.mark.gpu
def test_config5_shape_device_corpus_matches_oracle():
    """BASELINE configs[4]'s shape (64 planes, S = 8 column shards) at a
    reduced node count: the device-generated corpus equals the host's, and the
    public-API archive equals the oracle's shard blobs (codes, PQ tables,
    residual payloads incl. zlib bytes, exceptions bit-exact; lambda sections
    within the f32 tie tolerance), with every per-image NRMSE <= tau."""
    from concurrent.futures import ThreadPoolExecutor

    import torch

    import paper_2212_10733_b200 as mb
    from oracle import port
    from paper_2212_10733_b200 import container
    from tests import golden_util as G
    from tests.test_gpu_parity import _check_lambdas

    P, N = 64, 512
    dev = torch.device("cuda", 0)
    params = fdata.SyntheticParams(seed=42, rho=0.003)
    ds = synth.gen_synthetic(P, N, _grid(), params)
    got = synth.gen_synthetic_device(P, N, _grid(), params, dev).cpu().numpy()
    assert np.array_equal(got[:ds.data.size].view(np.uint64), ds.data.reshape(-1).view(np.uint64))
    cfg = mb.PipelineConfig(workers=8, shards=8, seed=0, tau=1e-3, lambda_precision="f32",
                            static_model=True)
    models = [mb.AEModel(weights=w, norm_mean=m, norm_std=s) for (w, m, s) in G.models("cfg3")]
    arc, rep, _ = mb.compress(ds, cfg, mb.TimestepState(models=models, timestep_index=1))
    _, blobs = container.read_archive(arc)
    ocfg = port.Cfg(shards=8, mode="col", tau=1e-3, seed=0)
    members = port.shard_members(P, N, 8, "col")

    def job(i):
        pl, no = members[i]
        return port.compress_shard(ds.data[pl, no], G.oracle_grid(), ocfg, G.models("cfg3")[i],
                                   i).blob

    with ThreadPoolExecutor(max_workers=8) as ex:
        want = list(ex.map(job, range(8)))
    for si, (b, w) in enumerate(zip(blobs, want)):
        sg, sw = container.read_shard(b).sections, container.read_shard(w).sections
        for name in ("codes", "pq_table", "residuals", "exceptions"):
            assert sg[name] == sw[name], (si, name)
        if sg["lambdas"] != sw["lambdas"]:
            _check_lambdas(sg["lambdas"], sw["lambdas"], "f32")
        assert len(b) == len(w)
    assert rep.max_per_image_nrmse() <= cfg.tau
