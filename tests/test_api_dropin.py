"""The reference's public per-call API (mlk/__init__.py:9-38) on the B200.

The reference's own known-answer and property tests for these functions
(pkg/tests/test_quantizer.py, test_residual.py, test_lagrange.py,
test_qoi.py, test_autoencoder.py), re-pointed at the device-backed
implementations, plus bit-exact agreement with the oracle restatement /
reference-generated vectors where the reference is deterministic.
CPU test at the bottom: the names exist.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2212_10733_b200 as mb
from paper_2212_10733_b200 import lagrange, qoi, quantizer, residual

torch = pytest.importorskip("torch")
gpu = pytest.mark.gpu
needs_cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")

REF_NAMES = ["AEModel", "TrainConfig", "ae_accuracy", "train", "SelectionScheme", "Shard",
             "partition", "select_training", "FDataset", "SyntheticParams", "VelocityGrid",
             "load_dataset", "make_grid", "save_dataset", "BACKEND", "ConstraintSystem",
             "NewtonOptions", "apply_lambda", "build_constraints", "newton_project",
             "PipelineConfig", "TimestepState", "compress", "decompress", "evaluate",
             "run_timesteps", "ErrorReport", "compression_ratio", "compute_qoi", "nrmse",
             "PQCodebook", "kmeans_1d", "pq_decode", "pq_encode", "pq_train", "BuiltinCodec",
             "EBCodec", "find_error_bound"]


def test_reference_public_names_exist():
    """Every name of the reference's __all__ except gen_synthetic (input
    production, workload/) is exported."""
    missing = [n for n in REF_NAMES if not hasattr(mb, n)]
    assert missing == []
    assert set(REF_NAMES) <= set(mb.__all__)


# --------------------------------------------------------------- quantizer

@gpu
@needs_cuda
def test_kmeans_known_answers():
    assert np.allclose(mb.kmeans_1d([0.0, 0.0, 10.0, 10.0], k=2, seed=0), [0.0, 10.0])
    assert np.allclose(mb.kmeans_1d([1.0, 2.0, 3.0], k=3, seed=0), [1.0, 2.0, 3.0])
    c = mb.kmeans_1d([5.0, 5.0, 7.0], k=4, seed=0)
    assert set(np.unique(c)) == {5.0, 7.0} and len(c) == 4
    with pytest.raises(mb.ConfigError):
        mb.kmeans_1d([], k=2, seed=0)


@gpu
@needs_cuda
def test_kmeans_matches_reference_vectors():
    """The reference's own kmeans_1d outputs (tests/golden/units.npz, made by
    importing the reference): float64 centroids bit for bit."""
    from tests import golden_util as G
    meta, a = G.load("units")
    for t, seed in enumerate(meta["kmeans_seeds"]):
        got = mb.kmeans_1d(a[f"km{t}_v"], 16, seed)
        assert np.array_equal(got, a[f"km{t}_c"]), t


@gpu
@needs_cuda
def test_kmeans_ties_and_duplicates_match_oracle():
    """Lattice values (many duplicates, members exactly midway between two
    centroids, centroids that coincide): the device's sorted-centroid
    nearest must pick np.argmin's first minimum like the oracle."""
    from oracle import port
    rng = np.random.default_rng(21)
    cases = [rng.integers(0, 24, 600) * 0.5,
             np.concatenate([rng.integers(0, 40, 300).astype(float), np.full(50, 2.5),
                             np.full(20, 7.5)]),
             np.concatenate([np.zeros(100), np.full(100, 1e-300), np.ones(30),
                             rng.integers(-40, 40, 200) * 0.25]),
             rng.integers(0, 6, 400) * 1e16 + rng.integers(0, 4, 400)]
    for i, v in enumerate(cases):
        for seed in range(4):
            got = mb.kmeans_1d(v, 16, seed)
            want = port.kmeans(v, 16, seed)
            assert np.array_equal(got, want), (i, seed)


@gpu
@needs_cuda
@pytest.mark.parametrize("n", [4096, 9001, 16395, 30000, 60000, 131160])
def test_kmeans_large_matches_oracle(n):
    """Shards of >= 4096 members run on a thread-block cluster (csrc/kmeans.cu
    k_kmeans_cl: 4 CTAs with everything in shared memory, or 8 CTAs with d2
    in global scratch beyond ~40k members): the codebook equals the oracle's
    bit for bit, also with duplicates, a cluster that dies and few distinct
    values."""
    from oracle import port
    rng = np.random.default_rng(n)
    cases = [rng.normal(0, 1, n) * 3.0,
             np.round(rng.normal(0, 1, n) * 8) / 4,                      # many duplicates
             np.concatenate([rng.normal(0, 1, n - 40), np.full(40, 1e6)]),  # far outliers
             rng.integers(0, 9, n).astype(np.float64)]                   # <= 16 distinct
    for i, v in enumerate(cases):
        for seed in (0, 5):
            assert np.array_equal(mb.kmeans_1d(v, 16, seed), port.kmeans(v, 16, seed)), (i, seed)


@gpu
@needs_cuda
def test_kmeans_cluster_path_with_256_centroids():
    """pq_bits = 8 (K = 256) on the cluster path (>= 4096 members)."""
    from oracle import port
    rng = np.random.default_rng(256)
    v = np.concatenate([rng.normal(0, 1, 12000), rng.normal(6, 0.3, 6000),
                        np.round(rng.normal(-4, 2, 2500) * 4) / 4])
    for seed in (0, 3):
        assert np.array_equal(mb.kmeans_1d(v, 256, seed), port.kmeans(v, 256, seed)), seed


@gpu
@needs_cuda
def test_kmeans_deterministic_and_quality():
    rng = np.random.default_rng(12)
    v = np.concatenate([rng.normal(0, 1, 80), rng.normal(8, 0.5, 60), rng.normal(-5, 2, 60)])

    def sse(c):
        return float(np.sum((v[:, None] - c[None, :]).min(axis=1) ** 2))
    got = sse(mb.kmeans_1d(v, k=4, seed=0))
    best = min(sse(mb.kmeans_1d(v, k=4, seed=s)) for s in range(20))
    assert got <= best * 1.05
    x = np.random.default_rng(3).normal(size=300)
    assert np.array_equal(mb.kmeans_1d(x, 16, seed=9), mb.kmeans_1d(x, 16, seed=9))


@gpu
@needs_cuda
def test_pq_known_answers():
    cents = np.arange(16.0)[None, :].repeat(4, axis=0)
    cb = mb.PQCodebook(centroids=cents)
    packed = mb.pq_encode(cb, np.array([[3.0] * 4, [10.0] * 4]))
    assert packed == bytes([0x33, 0x33, 0xAA, 0xAA])   # test_quantizer.py:82-88
    cb1 = mb.PQCodebook(centroids=np.array([[0.0, 1.0]]))
    assert mb.pq_decode(cb1, mb.pq_encode(cb1, np.array([[0.5]])), 1)[0, 0] == 0.0  # tie -> low
    lat = np.tile([1.5, -2.0, 0.25, 7.0], (20, 1))
    cb = mb.pq_train(lat, k=16, seed=0)
    for d in range(4):
        assert np.float32(lat[0, d]) in cb.centroids[d]
    with pytest.raises(mb.ConfigError):
        mb.pq_train(np.zeros((5, 4)), k=10, seed=0)
    with pytest.raises(mb.SizeMismatchError):
        mb.pq_decode(cb, b"\0", 20)


@gpu
@needs_cuda
def test_pq_train_is_per_dimension_kmeans_and_roundtrip_is_nearest():
    rng = np.random.default_rng(4)
    lat = np.stack([rng.normal(i * 3, 1, 200) for i in range(4)], axis=1)
    cb = mb.pq_train(lat, k=16, seed=7)
    for d in range(4):
        assert np.array_equal(cb.centroids[d],
                              mb.kmeans_1d(lat[:, d], 16, seed=7 + d).astype(np.float32))
    lat = rng.normal(size=(300, 4)) * [1, 10, 0.1, 100]
    cb = mb.pq_train(lat, k=64, seed=3)
    dec = mb.pq_decode(cb, mb.pq_encode(cb, lat), 300)
    cents = cb.centroids.astype(np.float64)
    for d in range(4):
        near = cents[d][np.argmin(np.abs(lat[:, d, None] - cents[d][None, :]), axis=1)]
        assert np.array_equal(dec[:, d], near)


# --------------------------------------------------------------- residual codec

@gpu
@needs_cuda
def test_codec_known_answers_and_errors():
    codec = mb.BuiltinCodec()
    out = codec.decompress(codec.compress(np.array([[0.7]]), eb=0.5))
    assert out[0, 0] == pytest.approx(1.0)                  # test_residual.py:26-30
    z = np.zeros((33, 37))
    p = codec.compress(z, eb=1.0)
    assert len(p) < 60 and np.array_equal(codec.decompress(p), z)
    r = np.random.default_rng(5).normal(0, 1e8, (9, 11))
    assert np.array_equal(codec.decompress(codec.compress_lossless(r)), r)
    with pytest.raises(mb.ConfigError):
        codec.compress(np.ones((2, 2)), eb=0.0)
    with pytest.raises(mb.ConfigError):
        codec.compress(np.array([[np.inf]]), eb=1.0)
    with pytest.raises(mb.FormatError):
        codec.decompress(b"moo")
    good = codec.compress(np.ones((2, 2)), eb=0.5)
    with pytest.raises(mb.FormatError):
        codec.decompress(good[:-2] + b"xx")


@gpu
@needs_cuda
def test_codec_bytes_equal_reference_payloads():
    """Payload bytes (quantised and lossless) equal the reference's
    (tests/golden/units.npz: BuiltinCodec outputs recorded from the reference)."""
    from tests import golden_util as G
    meta, a = G.load("units")
    codec = mb.BuiltinCodec()
    for t, eb in enumerate(meta["payload_ebs"]):
        r = a[f"pl{t}_r"]
        p = codec.compress_lossless(r) if t % 8 == 7 else codec.compress(r, eb)
        assert p == a[f"pl{t}_p"].tobytes(), t
        back = codec.decompress(p)
        assert np.max(np.abs(back - r)) <= (0.0 if t % 8 == 7 else eb)


@gpu
@needs_cuda
def test_codec_linf_fuzz_and_roundtrip_equals_byte_path():
    codec = mb.BuiltinCodec()
    rng = np.random.default_rng(2)
    for _ in range(120):
        rows, cols = rng.integers(1, 8, 2)
        scale = 10.0 ** rng.integers(-6, 12)
        r = rng.normal(0, scale, (rows, cols))
        eb = scale * 10.0 ** rng.uniform(-4, 1)
        out = codec.decompress(codec.compress(r, eb))
        assert out.shape == r.shape and np.max(np.abs(r - out)) <= eb
    r = rng.normal(0, 5, (20, 30))
    for eb in (1e-3, 0.17, 42.0):
        assert np.array_equal(codec.quantize_roundtrip(r, eb),
                              codec.decompress(codec.compress(r, eb)))
    assert codec.compress(r, 0.1) == codec.compress(r, 0.1)


def _near_threshold(rng, n=24, tau=1e-3):
    imgs = rng.lognormal(10, 0.2, (n, 8, 9))
    flat = imgs.reshape(n, -1)
    ranges = flat.max(axis=1) - flat.min(axis=1)
    noise = rng.normal(0, 1, imgs.shape)
    noise /= np.sqrt(np.mean(noise ** 2, axis=(1, 2)))[:, None, None]
    return imgs, imgs + noise * (1.3 * tau) * ranges[:, None, None]


@gpu
@needs_cuda
def test_find_error_bound_matches_oracle_search_and_gate():
    """The bisection visits the reference's bounds (numpy log/exp on the
    host) and decides each probe with the exact per-image NRMSE, so eb
    equals the oracle's restatement bit for bit; the corrected images pass."""
    from oracle import port
    codec = mb.BuiltinCodec()
    rng = np.random.default_rng(6)
    imgs, recons = _near_threshold(rng)
    tau = 1e-3
    sel = residual.select_residuals(imgs, recons, tau)
    assert sel.size == len(imgs)
    eb, lossless = mb.find_error_bound(imgs[sel], recons[sel], tau, codec)
    want_eb, want_ll, _ = port.search_bound(imgs[sel].reshape(len(sel), -1),
                                         recons[sel].reshape(len(sel), -1), tau)
    assert (eb, lossless) == (want_eb, want_ll)
    flat = imgs.reshape(len(imgs), -1)
    assert eb >= tau * float((flat.max(axis=1) - flat.min(axis=1)).max()) / 4
    plan = residual.ResidualPlan(tau=tau, eb=eb, lossless=False, selected=sel,
                                 payloads=[codec.compress(imgs[i] - recons[i], eb) for i in sel])
    fixed = residual.apply_residuals(recons, plan, codec)
    assert np.all(port.nrmse_rows(imgs.reshape(len(imgs), -1), fixed.reshape(len(imgs), -1))
                  <= tau)
    with pytest.raises(mb.ConfigError):
        mb.find_error_bound(np.zeros((0, 2, 2)), np.zeros((0, 2, 2)), 1e-3, codec)
    # flat references can never pass inexactly -> lossless (test_residual.py:143-158)
    flat_imgs = np.full((2, 3, 3), 7.0)
    eb, lossless = mb.find_error_bound(flat_imgs, flat_imgs + rng.normal(0, 1, (2, 3, 3)),
                                       1e-3, codec)
    assert lossless


@gpu
@needs_cuda
def test_find_error_bound_with_a_user_codec():
    """A user EBCodec plugs in through quantize_roundtrip (the plugin point,
    residual.py:39-54): a codec that rounds like the built-in one finds the
    same bound."""
    class Mine(mb.EBCodec):
        def quantize_roundtrip(self, residual, eb):
            return np.rint(residual / (2.0 * eb)) * (2.0 * eb)
    imgs, recons = _near_threshold(np.random.default_rng(8), n=10)
    a = mb.find_error_bound(imgs, recons, 1e-3, Mine())
    b = mb.find_error_bound(imgs, recons, 1e-3, mb.BuiltinCodec())
    assert a == b


# --------------------------------------------------------------- lagrange

def _instance(rng, rows=3, cols=3, perturb=0.05):
    grid = mb.make_grid(rows, cols, 2.0, 2.0, 1.0)
    f_true = rng.lognormal(0, 1, (rows, cols))
    q = mb.compute_qoi(f_true, grid)
    return grid, f_true, f_true * rng.uniform(1 - perturb, 1 + perturb, f_true.shape), q, \
        mb.build_constraints(grid, q)


@gpu
@needs_cuda
def test_constraints_and_qoi_known_answers():
    grid = mb.VelocityGrid(v_perp=np.array([0.0, 3.0]), v_par=np.array([0.0, 2.0]),
                           vol=np.ones((2, 2)), mass=1.0)
    img = np.zeros((2, 2))
    img[1, 1] = 2.0
    assert mb.compute_qoi(img, grid) == pytest.approx((2.0, 2.0, 4.5, 0.0))
    cs = mb.build_constraints(grid, (2.0, 2.0, 4.5, 0.0))
    assert (cs.a[:, 3] * cs.row_scales)[:3] == pytest.approx([1.0, 2.0, 4.5])
    assert cs.b * cs.row_scales == pytest.approx([2.0, 4.0, 9.0, 0.0])
    with pytest.raises(mb.ConfigError):
        mb.build_constraints(grid, (0.0, 0.0, 0.0, 0.0))
    n, u, tp, tl = mb.compute_qoi(np.zeros((2, 2)), grid)
    assert n == 0.0 and np.isnan(u) and np.isnan(tp) and np.isnan(tl)
    with pytest.raises(mb.DimensionError):
        mb.compute_qoi(np.zeros((3, 2)), grid)
    rng = np.random.default_rng(0)
    for _ in range(5):
        g, f_true, _, q, cs = _instance(rng)
        assert np.allclose(cs.a @ f_true.reshape(-1), cs.b, rtol=1e-12)


@gpu
@needs_cuda
def test_newton_project_known_answers():
    rng = np.random.default_rng(2)
    _, f_true, _, _, cs = _instance(rng)
    lam, f_corr, status, iters = mb.newton_project(f_true, cs)
    assert status == lagrange.NewtonStatus.CONVERGED and iters <= 1
    assert np.allclose(lam, 0.0, atol=1e-10)
    # one cell, f_hat = 1, target 2: lam0 = -ln 2 (test_lagrange.py:72-84)
    a = np.array([np.ones(4), np.zeros(4), np.zeros(4), np.zeros(4)])
    cs1 = mb.ConstraintSystem(a=a, b=np.array([8.0, 0, 0, 0]), row_scales=np.ones(4))
    lam, f_corr, status, _ = mb.newton_project(np.ones((2, 2)), cs1)
    assert status == lagrange.NewtonStatus.CONVERGED
    assert lam[0] == pytest.approx(-np.log(2.0), rel=1e-10)
    assert np.allclose(f_corr, 2.0, rtol=1e-10)


@gpu
@needs_cuda
def test_newton_feasibility_positivity_and_replay():
    rng = np.random.default_rng(5)
    opts = mb.NewtonOptions()
    for _ in range(20):
        _, _, f_hat, _, cs = _instance(rng, perturb=0.08)
        lam, f_corr, status, _ = mb.newton_project(f_hat, cs, opts)
        assert status == lagrange.NewtonStatus.CONVERGED
        resid = np.abs(cs.a @ f_corr.reshape(-1) - cs.b)
        assert np.max(resid) <= 10 * opts.tol * np.max(np.abs(cs.b))
        assert np.all(f_corr > 0)
        # the decoder-side replay is the same bytes (test_lagrange.py:158-164)
        assert mb.apply_lambda(f_hat, lam, cs).tobytes() == f_corr.tobytes()
    _, _, f_hat, _, cs = _instance(rng)
    floored = np.maximum(f_hat, 1e-12 * f_hat.max())
    assert np.array_equal(mb.apply_lambda(f_hat, np.zeros(4), cs), floored)
    with pytest.raises(mb.ConfigError):
        mb.apply_lambda(f_hat, np.array([np.nan, 0, 0, 0]), cs)


@gpu
@needs_cuda
def test_apply_lambda_matches_numpy_within_exp_ulps():
    """apply_lambda's only difference from the reference is exp: CUDA's vs
    numpy's SIMD exp (both <= 1 ulp from exact): <= 4 ulp, mostly identical."""
    rng = np.random.default_rng(8)
    grid = mb.make_grid(5, 7, 2.0, 2.0, 1.3)
    for _ in range(12):
        img = rng.lognormal(0, 1, (5, 7))
        cs = mb.build_constraints(grid, mb.compute_qoi(img, grid))
        lam = rng.normal(0, 0.1, 4)
        got = mb.apply_lambda(img, lam, cs)
        fp = np.maximum(img.reshape(-1), 1e-12 * img.max())
        t = lam[0] * cs.a[0] + lam[1] * cs.a[1] + lam[2] * cs.a[2] + lam[3] * cs.a[3]
        want = (fp * np.exp(-np.clip(t, -700.0, 700.0))).reshape(5, 7)
        assert np.max(np.abs(got - want) / np.abs(want)) <= 4 * 2.0 ** -52


# --------------------------------------------------------------- qoi / autoencoder

@gpu
@needs_cuda
def test_compute_qoi_matches_reference_moments():
    """Moments of the reference's unit images (tests/golden/units.npz) within
    summation-order noise (test_qoi.py: 1e-13)."""
    from tests import golden_util as G
    _, a = G.load("units")
    grid = G.grid()
    q = qoi.compute_qoi_batch(a["nr_o"], grid)
    got = np.stack([q.n, q.u_par, q.t_perp, q.t_par], axis=1)
    # u_par cancels to ~1e-2 of the thermal speed: summation-order noise is
    # absolute there (~1e-16), relative everywhere else
    np.testing.assert_allclose(got[:, [0, 2, 3]], a["qoi"][:, [0, 2, 3]], rtol=1e-12)
    np.testing.assert_allclose(got[:, 1], a["qoi"][:, 1], rtol=1e-12, atol=1e-14)
    for i in range(3):
        want = tuple(a["qoi"][i])
        assert mb.compute_qoi(a["nr_o"][i], grid) == pytest.approx(want, rel=1e-12, abs=1e-14)


@gpu
@needs_cuda
def test_ae_accuracy_extremes_and_oracle():
    from oracle import port
    from tests import golden_util as G
    ds, _ = G.corpus("tiny")
    (w, m, s), = G.models("tiny")
    model = mb.AEModel(weights=w, norm_mean=m, norm_std=s)
    imgs = ds.data.reshape(-1, 39, 39)
    assert mb.ae_accuracy(imgs, model, 1e9) == 1.0
    assert mb.ae_accuracy(imgs, model, 1e-300) == 0.0
    lat = port.ae_encode(w, m, s, imgs.reshape(len(imgs), -1))
    rec = port.ae_decode(w, m, s, lat)
    err = port.nrmse_rows(imgs.reshape(len(imgs), -1), rec.reshape(len(imgs), -1))
    for tau in (1e-3, 1e-2, float(np.median(err))):
        assert mb.ae_accuracy(imgs, model, tau) == float(np.mean(err <= tau))
    with pytest.raises(mb.ConfigError):
        mb.ae_accuracy(imgs, model, 0.0)
