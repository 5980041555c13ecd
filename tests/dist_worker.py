"""torchrun worker for tests/test_multi_gpu.py (one rank per GPU, NCCL):
compress_distributed the named golden corpus (and, with --train, with
state=None so every rank's models come from the rank that trained them),
decompress_distributed it, and write the archive / decoded planes where the
test reads them."""

import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2212_10733_b200 as mb  # noqa: E402
from paper_2212_10733_b200 import pipeline  # noqa: E402
from tests import golden_util as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("out")
    ap.add_argument("--train", action="store_true")
    a = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    meta, _ = G.load(a.name)
    ds, _ = G.corpus(a.name)
    c = dict(meta["runs"][0]["cfg"])
    c["newton"] = mb.NewtonOptions(**c["newton"])
    cfg = mb.PipelineConfig(**c)
    state = None if a.train else mb.TimestepState(
        models=[mb.AEModel(weights=w, norm_mean=m, norm_std=s) for w, m, s in G.models(a.name)],
        timestep_index=1)
    _, rep, st = pipeline.compress_distributed(ds, cfg, state, out_path=a.out)
    dist.barrier()
    arc = Path(a.out).read_bytes()
    dec = pipeline.decompress_distributed(arc)
    # the file variant: every rank DMAs its planes into one shared output file
    # (run twice: the second call reuses the cached, page-locked mapping)
    for _ in range(2):
        pipeline.decompress_distributed(arc, out_path=a.out + ".planes.f64")
    if dist.get_rank() == 0:
        np.save(a.out + ".dec.npy", dec.data)
        np.save(a.out + ".rep.npy", np.array([rep.compression_ratio, rep.exception_count,
                                              rep.residual_fraction, rep.pd_nrmse,
                                              rep.max_qoi_nrmse]))
        if a.train:
            np.savez(a.out + ".models.npz", W=np.stack([m.weights for m in st.models]),
                     mean=np.array([m.norm_mean for m in st.models]),
                     std=np.array([m.norm_std for m in st.models]))
    dist.barrier()
    from paper_2212_10733_b200 import hostio
    hostio.release_maps()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
