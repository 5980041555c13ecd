"""Multi-GPU compress / decompress on one box (one process per GPU, NCCL):
the archive compress_distributed writes equals the single-process archive
byte for byte, decompress_distributed returns the single-process decode, and
distributed training (shard s trained on rank s % G, weights broadcast)
gives the single-process models.  Skipped unless >= 2 GPUs are visible."""

from __future__ import annotations

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
    pytest.skip("needs >= 2 CUDA devices", allow_module_level=True)

import paper_2212_10733_b200 as mb  # noqa: E402
from tests import golden_util as G  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(name, out, n, train=False):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           str(ROOT / "tests" / "dist_worker.py"), name, str(out)] + (["--train"] if train else [])
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def _single(name, train=False):
    meta, _ = G.load(name)
    ds, same = G.corpus(name)
    if not same:
        pytest.skip("host generates a different corpus")
    c = dict(meta["runs"][0]["cfg"])
    c["newton"] = mb.NewtonOptions(**c["newton"])
    cfg = mb.PipelineConfig(**c)
    state = None if train else mb.TimestepState(
        models=[mb.AEModel(weights=w, norm_mean=m, norm_std=s) for w, m, s in G.models(name)],
        timestep_index=1)
    arc, rep, st = mb.compress(ds, cfg, state)
    return ds, arc, rep, st


@pytest.mark.parametrize("n", [2, 4])
def test_distributed_archive_is_the_single_process_archive(n, tmp_path):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    ds, arc, rep, _ = _single("cfg3")
    out = tmp_path / "cfg3.mlk"
    _run("cfg3", out, n)
    got = out.read_bytes()
    assert got == arc
    r = np.load(str(out) + ".rep.npy")
    assert r[0] == rep.compression_ratio and int(r[1]) == rep.exception_count
    assert r[2] == rep.residual_fraction
    assert abs(r[3] - rep.pd_nrmse) <= 1e-9 * rep.pd_nrmse
    dec = np.load(str(out) + ".dec.npy")
    single = mb.decompress(arc).data
    bad = np.argwhere(~(dec == single).all(axis=(2, 3)))
    rel = 0.0
    if len(bad):
        p, q = bad[0]
        rel = float(np.max(np.abs(dec[p, q] - single[p, q]) / np.maximum(np.abs(single[p, q]),
                                                                           1e-300)))
    assert len(bad) == 0, (len(bad), bad[:8].tolist(), rel)
    planes = np.fromfile(str(out) + ".planes.f64", dtype="<f8").reshape(single.shape)
    assert np.array_equal(planes, dec)  # decompress_distributed(out_path=...)


def test_distributed_training_gives_the_single_process_models(tmp_path):
    ds, arc, rep, st = _single("small", train=True)
    out = tmp_path / "small.mlk"
    _run("small", out, 2, train=True)
    m = np.load(str(out) + ".models.npz")
    for i, mod in enumerate(st.models):
        assert np.array_equal(m["W"][i], mod.weights)
        assert m["mean"][i] == mod.norm_mean and m["std"][i] == mod.norm_std
    assert out.read_bytes() == arc
