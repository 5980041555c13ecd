"""Device AE training at configs[2] (8 planes x 16,395 nodes, S = 8 shards,
colrandind selection, 100 epochs): time of the one mlk_ae_train launch,
deviation from the reference-trained golden models (tests/golden/cfg3.npz),
and the oracle restatement (= the reference's numpy algorithm) timed on one
shard on the host.  Prints one JSON line.

    python tools/train_bench.py [--reps 3] [--cpu-shards 1]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_10733_b200 as mb  # noqa: E402
from paper_2212_10733_b200 import pipeline  # noqa: E402
from oracle import port  # noqa: E402
from tests import golden_util as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu-shards", type=int, default=1)
    args = ap.parse_args()
    meta, a = G.load("cfg3")
    ds, same = G.corpus("cfg3")
    c = meta["runs"][0]["cfg"]
    cfg = mb.PipelineConfig(**{k: v for k, v in c.items() if k != "newton"})
    dev = torch.device("cuda", 0)
    shards = mb.partition(ds.n_planes, ds.n_nodes, cfg.shards, cfg.mode)
    f0 = pipeline.upload_f0(ds.data, dev)
    torch.cuda.synchronize()
    times, models = [], None
    for _ in range(args.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        models = pipeline._train_models(f0, shards, ds, cfg, None, True)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    dev_ms = float(np.median(times[1:]))
    n_train = [len(mb.select_training(sh, cfg.scheme, ds.n_planes,
                                      mb.mix_seed(cfg.seed, sh.worker_id))) for sh in shards]
    steps = [cfg.epochs_full * -(-n // cfg.batch_size) for n in n_train]
    dw = max(float(np.max(np.abs(m.weights - a["model_W"][i])) / np.max(np.abs(a["model_W"][i])))
             for i, m in enumerate(models))
    dmean = max(abs(m.norm_mean - a["model_mean"][i]) / abs(a["model_mean"][i])
                for i, m in enumerate(models))
    exact = sum(int(np.array_equal(m.weights, a["model_W"][i])) for i, m in enumerate(models))
    ulps = max(int(np.max(np.abs(m.weights.view(np.int32).astype(np.int64)
                                 - a["model_W"][i].view(np.int32).astype(np.int64))))
               for i, m in enumerate(models))
    # the reference algorithm on the host (oracle restatement), one shard at a time
    ref = port.shard_members(ds.n_planes, ds.n_nodes, cfg.shards, cfg.mode)
    t0 = time.perf_counter()
    for i in range(args.cpu_shards):
        pl, no = ref[i]
        seed = port.mix_seed(cfg.seed, i)
        sel = port.select_training(pl, no, cfg.scheme, ds.n_planes, seed, i)
        w, mu, sd = port.ae_train(ds.data[pl[sel], no[sel]], cfg.learning_rate,
                                  cfg.batch_size, cfg.epochs_full, seed=seed,
                                  latent_dim=cfg.latent_dim)
        assert np.array_equal(w, a["model_W"][i])
    cpu_s = (time.perf_counter() - t0) / max(1, args.cpu_shards)
    from paper_2212_10733_b200 import _lib
    lc = np.zeros(4, dtype=np.int32)
    _lib.call("mlk_ae_train_config", lc.ctypes.data)
    print(json.dumps({
        "launch": {"cluster": int(lc[0]), "rows_per_chunk": int(lc[1]),
                   "cols_per_cta": int(lc[2]), "smem_bytes": int(lc[3])},
        "workload": "configs[2] AE training: 8 shards, colrandind, 100 epochs, batch 128",
        "corpus_matches_golden": bool(same),
        "device_ms_all_shards": dev_ms, "device_ms_reps": times[1:],
        "train_images_per_shard": n_train, "adam_steps_per_shard": steps,
        "us_per_step": 1e3 * dev_ms / max(steps),
        "max_rel_dW_vs_reference": dw, "max_f32_ulps_vs_reference": ulps,
        "bit_exact_shards": exact, "max_rel_dmean": dmean,
        "cpu_oracle_s_per_shard": cpu_s, "cpu_threads": 1,
        "cpu_oracle_s_all_shards_serial": cpu_s * len(shards),
    }))


if __name__ == "__main__":
    main()
