"""Generate the golden fixtures from the REAL reference (build container only).

Run (needs /root/reference, which does not exist on the GPU box):

    cp -r /root/reference/pkg /tmp/refbuild && (cd /tmp/refbuild && \
        python setup.py build_ext --inplace)          # compiled backend
    OPENBLAS_NUM_THREADS=1 PYTHONPATH=/tmp/refbuild/src \
        python tests/golden/make_golden.py [case ...]

Every fixture records the reference backend, numpy/zlib versions and the
sha256 of its generated input so the tests can tell whether a host
regenerates the same corpus.  AE training is not on the hot path: the models
trained here (reference ``ae.train`` via ``compress(..., state=None)``) are
stored and replayed through ``static_model=True``, exactly as SURVEY §8d
prescribes for the oracle and the B200 path.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
import zlib
from pathlib import Path

import numpy as np

assert os.environ.get("OPENBLAS_NUM_THREADS") == "1", "run with OPENBLAS_NUM_THREADS=1"
import mlk  # noqa: E402  (the reference, from PYTHONPATH)
from mlk import autoencoder as ae  # noqa: E402
from mlk import container, kernels, lagrange, qoi, quantizer, residual  # noqa: E402
from mlk.decomp import mix_seed, partition  # noqa: E402
from mlk.pipeline import PipelineConfig, TimestepState, _shard_images  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def env() -> dict:
    return {"backend": kernels.BACKEND, "numpy": np.__version__,
            "zlib": zlib.ZLIB_RUNTIME_VERSION, "openblas_threads": 1}


def corpus(P, N, seed=42, rho=0.003):
    g = mlk.make_grid(39, 39, 5.0, 5.0, 1.0)
    return mlk.gen_synthetic(P, N, g, mlk.SyntheticParams(seed=seed, rho=rho))


def train_models(ds, cfg):
    _, _, state = mlk.compress(ds, cfg, None)
    return state.models


def models_arrays(models):
    return dict(W=np.stack([m.weights for m in models]).astype(np.float32),
                mean=np.array([m.norm_mean for m in models]),
                std=np.array([m.norm_std for m in models]))


def stage_dump(ds, cfg, models):
    """Re-run the reference's own stage functions shard by shard (the same
    calls _compress_shard makes, pipeline.py:196-292) to expose intermediates."""
    shards = partition(ds.n_planes, ds.n_nodes, cfg.shards, cfg.mode)
    per = []
    for sh, model in zip(shards, models):
        imgs = _shard_images(ds, sh)
        seed = mix_seed(cfg.seed, sh.worker_id)
        lat = ae.encode_batch(model, imgs)
        cb = quantizer.pq_train(lat, 2 ** cfg.pq_bits, seed)
        codes = quantizer.pq_encode(cb, lat)
        rec = ae.decode_batch(model, quantizer.pq_decode(cb, codes, len(imgs)), imgs.shape[1:])
        err = qoi.image_nrmse_batch(imgs, rec)
        bad = ~np.isfinite(err)
        sel = np.flatnonzero(~bad & (err > cfg.tau))
        eb, lossless = (residual.find_error_bound(imgs[sel], rec[sel], cfg.tau,
                                                  residual.BuiltinCodec())
                        if sel.size else (0.0, False))
        q = qoi.compute_qoi_batch(imgs, ds.grid)
        qm = np.stack([q.n, q.u_par, q.t_perp, q.t_par], axis=1)
        per.append(dict(latents=lat, cents=cb.centroids, codes=np.frombuffer(codes, np.uint8),
                        recon_sha=sha(rec), ae_err=err, selected=sel, eb=float(eb),
                        lossless=bool(lossless), qoi=qm))
    return per


def load_models(name):
    """The models an earlier case trained (its npz), replayed as static weights."""
    a = np.load(OUT / f"{name}.npz")
    return [ae.AEModel(weights=a["model_W"][i], norm_mean=float(a["model_mean"][i]),
                       norm_std=float(a["model_std"][i])) for i in range(a["model_W"].shape[0])]


def run_case(name, P, N, cfg_kw, taus=None, store_arrays=True, seed=42, rho=0.003,
             train_cfg=None, models_from=None, decompress=True, workers=8):
    t0 = time.time()
    ds = corpus(P, N, seed, rho)
    base = dict(workers=workers, seed=0, static_model=True)
    base.update(cfg_kw)
    cfg = PipelineConfig(**base)
    models = (load_models(models_from) if models_from else
              train_models(ds, PipelineConfig(**{**base, **(train_cfg or {})})))
    arrays = {f"model_{k}": v for k, v in models_arrays(models).items()}
    meta = {"case": name, "P": P, "N": N, "seed": seed, "rho": rho, "env": env(),
            "data_sha": sha(ds.data), "models_from": models_from, "runs": []}
    variants = taus or [dict()]
    for vi, var in enumerate(variants):
        c = PipelineConfig(**{**base, **var})
        arc, rep, _ = mlk.compress(ds, c, TimestepState(models=models, timestep_index=1))
        pre, blobs = container.read_archive(arc)
        dec = mlk.decompress(arc).data if decompress else None
        run = {"cfg": c.to_dict(), "digest": c.digest().hex(), "archive_len": len(arc),
               "archive_sha": sha(arc), "blob_len": [len(b) for b in blobs],
               "blob_sha": [sha(b) for b in blobs], "decomp_sha": sha(dec) if dec is not None else None,
               "ratio": rep.compression_ratio, "exceptions": rep.exception_count,
               "residual_fraction": rep.residual_fraction,
               "convergence_fraction": rep.convergence_fraction,
               "pd_nrmse": rep.pd_nrmse, "qoi_nrmse": rep.qoi_nrmse,
               "max_qoi_nrmse": rep.max_qoi_nrmse, "ae_accuracy": rep.ae_accuracy,
               "max_per_image": rep.max_per_image_nrmse(), "shards": []}
        for si, b in enumerate(blobs):
            sb = container.read_shard(b)
            s = sb.sections
            eb, count = __import__("struct").unpack_from("<dI", s["residuals"], 0)
            exc_n = __import__("struct").unpack_from("<I", s["exceptions"], 0)[0]
            off, exc = 4, []
            for _ in range(exc_n):
                exc.append(__import__("struct").unpack_from("<I", s["exceptions"], off)[0])
                off += 4 + 8 * 1521
            run["shards"].append({"eb": eb, "n_sel": count, "exceptions": exc,
                                  "sec_len": list(sb.header.section_lengths),
                                  "codes_sha": sha(s["codes"]), "ptab_sha": sha(s["pq_table"]),
                                  "res_sha": sha(s["residuals"]), "lam_sha": sha(s["lambdas"]),
                                  "exc_sha": sha(s["exceptions"])})
            if store_arrays:
                arrays[f"r{vi}_s{si}_codes"] = np.frombuffer(s["codes"], np.uint8)
                arrays[f"r{vi}_s{si}_ptab"] = np.frombuffer(s["pq_table"], np.uint8)
                arrays[f"r{vi}_s{si}_lam"] = np.frombuffer(s["lambdas"], np.uint8)
                if len(s["residuals"]) < 100_000:
                    arrays[f"r{vi}_s{si}_res"] = np.frombuffer(s["residuals"], np.uint8)
        meta["runs"].append(run)
        del arc, dec
        if store_arrays and vi == 0:
            for si, d in enumerate(stage_dump(ds, c, models)):
                for k, v in d.items():
                    if isinstance(v, np.ndarray):
                        arrays[f"st_s{si}_{k}"] = v
                    else:
                        run["shards"][si][f"st_{k}"] = v
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1, default=float))
    print(f"{name}: {time.time() - t0:.1f}s", flush=True)


def unit_cases():
    rng = np.random.default_rng(2212)
    arrays, meta = {}, {"env": env()}
    # k-means (quantizer.py:53-91)
    km = []
    for t in range(24):
        n = int(rng.integers(5, 3000))
        kind = t % 4
        if kind == 0:
            v = rng.standard_normal(n)
        elif kind == 1:
            v = np.round(rng.standard_normal(n) * 3) / 3        # few distinct values
        elif kind == 2:
            v = np.concatenate([rng.standard_normal(n // 2) * 1e-3, rng.standard_normal(n - n // 2) + 40])
        else:
            v = rng.exponential(size=n) ** 3
        seed = int(rng.integers(0, 2 ** 62))
        arrays[f"km{t}_v"] = v
        arrays[f"km{t}_c"] = quantizer.kmeans_1d(v, 16, seed)
        km.append(seed)
    meta["kmeans_seeds"] = km
    # Newton (compiled kernel, _ckernels.pyx:62-137)
    grid = mlk.make_grid(39, 39, 5.0, 5.0, 1.0)
    nw = []
    for t in range(16):
        n_true = float(np.exp(rng.uniform(0, 30)))
        u = float(rng.uniform(-0.8, 0.8))
        tp, tl = float(np.exp(rng.uniform(-1, 1))), float(np.exp(rng.uniform(-1, 1)))
        f = np.exp(-grid.v_perp[:, None] ** 2 / (2 * tp) - (grid.v_par[None, :] - u) ** 2 / (2 * tl))
        f = f * (1 + 0.05 * rng.uniform(-1, 1, f.shape)) * n_true
        cs = lagrange.build_constraints(grid, (n_true, u, tp, tl))
        fp = np.maximum(f.reshape(-1), 1e-12 * f.max())
        lam, st, it = kernels.newton_solve(fp, cs.a, cs.b, 1.0, 50, 1e-13)
        arrays[f"nw{t}_f"] = f
        arrays[f"nw{t}_q"] = np.array([n_true, u, tp, tl])
        arrays[f"nw{t}_lam"] = lam
        nw.append([int(st), int(it)])
    meta["newton_status_iters"] = nw
    # residual codec payloads (residual.py:60-98) -- DEFLATE golden bytes
    codec = residual.BuiltinCodec()
    pl = []
    for t in range(24):
        r = rng.standard_normal((39, 39)) * 10 ** rng.uniform(-3, 3)
        if t % 5 == 4:
            r[rng.uniform(size=r.shape) < 0.7] = 0.0
        eb = float(10 ** rng.uniform(-4, 1)) * float(np.abs(r).max() + 1e-30)
        p = codec.compress_lossless(r) if t % 8 == 7 else codec.compress(r, eb)
        arrays[f"pl{t}_r"] = r
        arrays[f"pl{t}_p"] = np.frombuffer(p, np.uint8)
        pl.append(eb)
    meta["payload_ebs"] = pl
    # per-image NRMSE (qoi.py:107-119) and moments (qoi.py:60-76)
    o = rng.exponential(size=(12, 39, 39)) * 1e12
    r = o * (1 + 1e-3 * rng.standard_normal(o.shape))
    o[3] = 7.0
    r[3] = 7.0
    o[4] = 7.0
    arrays["nr_o"], arrays["nr_r"] = o, r
    arrays["nr_e"] = qoi.image_nrmse_batch(o, r)
    q = qoi.compute_qoi_batch(o, grid)
    arrays["qoi"] = np.stack([q.n, q.u_par, q.t_perp, q.t_par], axis=1)
    # pack golden from test_quantizer.py:82-88 style
    idx = rng.integers(0, 16, 1001).astype(np.uint16)
    arrays["pack_idx"] = idx
    arrays["pack_bytes"] = np.frombuffer(kernels.pack_indices(idx, 4), np.uint8)
    np.savez_compressed(OUT / "units.npz", **arrays)
    (OUT / "units.json").write_text(json.dumps(meta, indent=1))
    print("units done", flush=True)


CASES = {
    "units": lambda: unit_cases(),
    # tiny: OpenBLAS small-matrix path (N*L*D <= 1e6)
    "tiny": lambda: run_case("tiny", 1, 64, dict(shards=1),
                             taus=[dict(), dict(tau=1e-2), dict(lambda_precision="f64")]),
    # two planes, 4 col shards + a row-mode run
    "small": lambda: run_case("small", 2, 240, dict(shards=4),
                              taus=[dict(), dict(tau=1e-4), dict(tau=1e-5)]),
    "rowmode": lambda: run_case("rowmode", 2, 200, dict(shards=4, mode="row", scheme="row"),
                                taus=[dict()]),
    # config 1 (BASELINE.json configs[0]): 1 x 1000, S=1; tau sweep + f64
    "cfg1": lambda: run_case("cfg1", 1, 1000, dict(shards=1),
                             taus=[dict(), dict(tau=1e-2), dict(tau=1e-4), dict(tau=1e-5),
                                   dict(lambda_precision="f64")]),
    # config 2 (configs[1]): 1 x 16395, S=8 -- hashes + small arrays only
    "cfg2": lambda: run_case("cfg2", 1, 16395, dict(shards=8), store_arrays=False,
                             taus=[dict(), dict(tau=1e-2), dict(tau=1e-4)]),
    # config 3 (configs[2]): 8 x 16395, S=8 -- the bench workload's weights
    "cfg3": lambda: run_case("cfg3", 8, 16395, dict(shards=8), store_arrays=False),
    # configs[3]'s remaining points on the config-2 corpus with cfg2's models:
    # tau=1e-5 (every selected image falls back to lossless) and f64 lambdas
    "cfg2x": lambda: run_case("cfg2x", 1, 16395, dict(shards=8), store_arrays=False,
                              models_from="cfg2",
                              taus=[dict(tau=1e-5), dict(lambda_precision="f64")]),
    # configs[4]: 64 x 16395 (12.8 GB), S=8 col shards of ~131k members with
    # config 3's node blocks and weights; shard hashes only (2 workers: memory)
    "cfg5": lambda: run_case("cfg5", 64, 16395, dict(shards=8), store_arrays=False,
                             models_from="cfg3", decompress=False, workers=2),
}

if __name__ == "__main__":
    for name in (sys.argv[1:] or list(CASES)):
        CASES[name]()
