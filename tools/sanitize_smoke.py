"""A tiny compress + decompress + train under compute-sanitizer (one tool per
process): python tools/sanitize_smoke.py  (run as
compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_smoke.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

import paper_2212_10733_b200 as mb  # noqa: E402
from tests import golden_util as G  # noqa: E402


def main():
    meta, _ = G.load("tiny")
    ds, _ = G.corpus("tiny")
    models = [mb.AEModel(weights=w, norm_mean=m, norm_std=s) for w, m, s in G.models("tiny")]
    for run in meta["runs"]:
        c = dict(run["cfg"])
        c["newton"] = mb.NewtonOptions(**c["newton"])
        cfg = mb.PipelineConfig(**c)
        arc, rep, _ = mb.compress(ds, cfg, mb.TimestepState(models=models, timestep_index=1))
        assert len(arc) == run["archive_len"]
        back = mb.decompress(arc).data
        assert back.shape == ds.data.shape
    imgs = ds.data.reshape(-1, 39, 39)
    mb.train(imgs[:40], mb.TrainConfig(epochs=2, seed=3))
    codec = mb.BuiltinCodec()
    r = np.random.default_rng(0).normal(size=(39, 39))
    assert np.max(np.abs(codec.decompress(codec.compress(r, 0.01)) - r)) <= 0.01
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
