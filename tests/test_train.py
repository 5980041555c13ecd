"""AE training: selection + device Adam vs the oracle.

Pinning: oracle.port.select_training / ae_train reproduce the models the
REAL reference trained when the golden fixtures were made
(tests/golden/make_golden.py: ``compress(ds, cfg, None)`` with epochs_full =
100, scheme colrandind / row) bit for bit -- CPU tests below.

Device parity (GPU tests): the normaliser (fit_normalizer's np.mean /
np.std) is numpy's pairwise summation reproduced exactly (the host tree of
autoencoder.pairwise_tree, pinned on CPU below), so mean and std are
bit-identical.  The Adam elementwise updates are in numpy's rounding order,
but the contractions (z, err W^T, grad, mse) reduce in a different order than
OpenBLAS, so the device weights match within a tolerance, not bit for bit:
the float32 weights agree to max |dW| <= 1e-5 * max |W| (measured on B200:
see DESIGN.md §4a).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import port
from paper_2212_10733_b200 import decomp
from tests import golden_util as G

W_TOL = 1e-5


def _golden_shards(name):
    meta, a = G.load(name)
    c = meta["runs"][0]["cfg"]
    return meta, a, c, port.shard_members(meta["P"], meta["N"], c["shards"], c["mode"])


@pytest.mark.parametrize("name", ["tiny", "small", "rowmode"])
def test_oracle_training_matches_reference_models(name):
    meta, a, c, shards = _golden_shards(name)
    ds, same = G.corpus(name)
    if not same:
        pytest.skip("this host's numpy generates a different corpus")
    for i, (pl, no) in enumerate(shards):
        seed = port.mix_seed(c["seed"], i)
        sel = port.select_training(pl, no, c["scheme"], meta["P"], seed, i)
        w, mu, sd = port.ae_train(ds.data[pl[sel], no[sel]], c["learning_rate"],
                                  c["batch_size"], c["epochs_full"], seed=seed,
                                  latent_dim=c["latent_dim"])
        assert np.array_equal(w, a["model_W"][i])
        assert mu == a["model_mean"][i] and sd == a["model_std"][i]


@pytest.mark.parametrize("scheme", [s.value for s in decomp.SelectionScheme])
@pytest.mark.parametrize("P,N,S,mode", [(1, 50, 2, "col"), (3, 40, 4, "col"), (3, 40, 3, "row")])
def test_select_training_matches_oracle(scheme, P, N, S, mode):
    shards = decomp.partition(P, N, S, mode)
    ref = port.shard_members(P, N, S, mode)
    for sh, (pl, no) in zip(shards, ref):
        seed = decomp.mix_seed(7, sh.worker_id)
        try:
            want = port.select_training(pl, no, scheme, P, seed, sh.worker_id)
        except ValueError:
            with pytest.raises(decomp.ConfigError):
                decomp.select_training(sh, scheme, P, seed)
            continue
        got = decomp.select_training(sh, scheme, P, seed)
        assert np.array_equal(np.asarray(got), np.asarray(want))


def _pw_leaf(a):
    n = len(a)
    if n < 8:
        s = 0.0
        for x in a:
            s += x
        return s
    r, lim = list(a[:8]), n - n % 8
    for i in range(8, lim, 8):
        for k in range(8):
            r[k] += a[i + k]
    s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    for i in range(lim, n):
        s += a[i]
    return s


def _pw_tree_sum(x, tree):
    """What k_pw_leaves + k_pw_combine compute, on the host."""
    lo, ln, ch, lv = tree
    al = x.tolist()
    nodes = [_pw_leaf(al[a:a + b]) for a, b in zip(lo, ln)] + [0.0] * int(lv[-1])
    nl = len(lo)
    for L in range(len(lv) - 1):
        for k in range(lv[L], lv[L + 1]):
            nodes[nl + k] = nodes[ch[2 * k]] + nodes[ch[2 * k + 1]]
    return nodes[nl + lv[-1] - 1] if lv[-1] else nodes[0]


@pytest.mark.parametrize("n", [1, 7, 8, 128, 129, 1000, 1521 * 3, 1521 * 700 + 5])
def test_pairwise_tree_is_numpys_summation(n):
    """autoencoder.pairwise_tree (the layout the device normaliser walks)
    reproduces np.mean / np.std of the training selection bit for bit."""
    from paper_2212_10733_b200.autoencoder import pairwise_tree
    x = np.random.default_rng(n).exponential(size=n) ** 3 * 1e12
    tree = pairwise_tree(n)
    m = _pw_tree_sum(x, tree) / n
    assert m == np.mean(x)
    assert np.sqrt(_pw_tree_sum((x - m) ** 2, tree) / n) == np.std(x)


# ---------------------------------------------------------------------------
# device training (GPU)

def _close(model, w, mu, sd):
    W = np.asarray(model.weights)
    assert np.max(np.abs(W - w)) <= W_TOL * np.max(np.abs(w)), np.max(np.abs(W - w))
    assert model.norm_mean == mu and model.norm_std == sd, (model.norm_mean - mu,
                                                            model.norm_std - sd)


@pytest.mark.gpu
@pytest.mark.parametrize("n,batch,epochs,L", [(64, 128, 20, 4), (500, 128, 3, 4),
                                               (300, 250, 4, 4), (97, 16, 3, 8), (1, 128, 5, 2)])
def test_device_train_matches_oracle(n, batch, epochs, L):
    import paper_2212_10733_b200 as mb
    ds, _ = G.corpus("small")
    imgs = ds.data.reshape(-1, 39, 39)[:n]
    tc = mb.TrainConfig(batch_size=batch, epochs=epochs, seed=11)
    model = mb.train(imgs, tc, latent_dim=L)
    w, mu, sd = port.ae_train(imgs, batch=batch, epochs=epochs, seed=11, latent_dim=L)
    _close(model, w, mu, sd)
    # warm start continues from the trained weights (autoencoder.py:153-157)
    tc2 = mb.TrainConfig(batch_size=batch, epochs=2, seed=12)
    m2 = mb.train(imgs, tc2, init=model)
    w2, mu2, sd2 = port.ae_train(imgs, batch=batch, epochs=2, seed=12, init_w=model.weights)
    _close(m2, w2, mu2, sd2)


@pytest.mark.gpu
def test_device_train_errors():
    import paper_2212_10733_b200 as mb
    ds, _ = G.corpus("tiny")
    imgs = ds.data.reshape(-1, 39, 39)[:10].copy()
    with pytest.raises(mb.ConfigError):
        mb.train(imgs[:0], mb.TrainConfig())
    bad = mb.AEModel(weights=np.zeros((4, 100), np.float32), norm_mean=0.0, norm_std=1.0)
    with pytest.raises(mb.DimensionError):
        mb.train(imgs, mb.TrainConfig(epochs=1), init=bad)
    imgs[3, 5, 5] = np.inf
    with pytest.raises(mb.TrainingDivergedError) as ei:
        mb.train(imgs, mb.TrainConfig(epochs=2))
    assert ei.value.epoch == 0
    with pytest.raises(FloatingPointError):
        port.ae_train(imgs, epochs=2)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tiny", "small", "cfg3"])
def test_compress_trains_like_reference(name):
    """compress(ds, cfg, None) trains every shard on the device (one launch)
    and the models match the reference-trained golden models (normaliser
    bit-identical, weights within W_TOL); at configs[2] the archive then has
    the reference's codes, PQ tables, residuals and exceptions."""
    import paper_2212_10733_b200 as mb
    meta, a, c, _ = _golden_shards(name)
    ds, same = G.corpus(name)
    if not same:
        pytest.skip("corpus differs on this host")
    cfg = mb.PipelineConfig(**{k: v for k, v in c.items() if k != "newton"})
    cfg_static = mb.PipelineConfig(**{**{k: v for k, v in c.items() if k != "newton"},
                                      "static_model": False})
    for conf in ((cfg,) if name == "cfg3" else (cfg, cfg_static)):
        arc, rep, st = mb.compress(ds, conf, None)
        if name == "cfg3":
            from paper_2212_10733_b200 import container
            _, blobs = container.read_archive(arc)
            for si, b in enumerate(blobs):
                sec = container.read_shard(b).sections
                ref = meta["runs"][0]["shards"][si]
                for k, key in (("codes", "codes_sha"), ("pq_table", "ptab_sha"),
                               ("residuals", "res_sha"), ("exceptions", "exc_sha")):
                    assert G.sha(sec[k]) == ref[key], (si, k)
        assert st.timestep_index == 1 and len(st.models) == len(a["model_W"])
        for i, m in enumerate(st.models):
            _close(m, a["model_W"][i], a["model_mean"][i], a["model_std"][i])
        dec = mb.decompress(arc)
        assert rep.max_per_image_nrmse() <= conf.tau
        per = port.nrmse_rows(ds.data.reshape(-1, 1521), dec.data.reshape(-1, 1521))
        assert np.all(per <= conf.tau)
        assert rep.stage_timings["train"]["sum"] > 0


@pytest.mark.gpu
def test_run_timesteps_modes():
    import paper_2212_10733_b200 as mb
    ds, _ = G.corpus("tiny")
    cfg = mb.PipelineConfig(shards=1, epochs_full=3, epochs_incremental=1, retrain_period=2)
    out = mb.run_timesteps([ds, ds, ds], cfg)
    assert [m for _, _, m in out] == ["full", "incremental", "full"]
    for arc, rep, _ in out:
        assert rep.max_per_image_nrmse() <= cfg.tau
        assert mb.decompress(arc).data.shape == ds.data.shape
    out = mb.run_timesteps([ds, ds], mb.PipelineConfig(shards=1, epochs_full=2,
                                                       static_model=True))
    assert [m for _, _, m in out] == ["full", "static"]
    assert out[0][0][:100] == out[1][0][:100]


def test_train_config_validation_and_no_cpu_fallback():
    """TrainConfig rejects what the reference rejects (autoencoder.py:70-75);
    without a CUDA device train() raises BackendError -- there is no host
    fallback for the trainer."""
    import torch

    import paper_2212_10733_b200 as mb
    with pytest.raises(mb.ConfigError):
        mb.TrainConfig(learning_rate=0.0)
    with pytest.raises(mb.ConfigError):
        mb.TrainConfig(batch_size=0)
    with pytest.raises(mb.ConfigError):
        mb.TrainConfig(epochs=0)
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    imgs = np.ones((4, 39, 39))
    with pytest.raises(mb.BackendError):
        mb.train(imgs, mb.TrainConfig(epochs=1))
