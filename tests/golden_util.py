"""Helpers to load the reference-generated fixtures under tests/golden/."""

from __future__ import annotations

import functools
import hashlib
import json
from pathlib import Path

import numpy as np

from oracle import port
from paper_2212_10733_b200 import fdata
from workload import synth

GOLDEN = Path(__file__).resolve().parent / "golden"


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


@functools.lru_cache(maxsize=None)
def load(name):
    meta = json.loads((GOLDEN / f"{name}.json").read_text())
    npz = GOLDEN / f"{name}.npz"
    arrays = dict(np.load(npz)) if npz.exists() else {}
    return meta, arrays


def grid():
    return fdata.make_grid(39, 39, 5.0, 5.0, 1.0)


@functools.lru_cache(maxsize=4)
def corpus(name):
    meta, _ = load(name)
    ds = synth.gen_synthetic(meta["P"], meta["N"], grid(),
                             fdata.SyntheticParams(seed=meta["seed"], rho=meta["rho"]))
    return ds, sha(ds.data) == meta["data_sha"]


def models(name):
    _, a = load(name)
    return [(a["model_W"][i], float(a["model_mean"][i]), float(a["model_std"][i]))
            for i in range(a["model_W"].shape[0])]


def oracle_grid():
    g = grid()
    return port.Grid(g.v_perp, g.v_par, g.vol, g.mass)


def oracle_cfg(run):
    c = run["cfg"]
    nw = c["newton"]
    return port.Cfg(shards=c["shards"], mode=c["mode"], tau=c["tau"],
                    latent_dim=c["latent_dim"], pq_bits=c["pq_bits"],
                    lambda_precision=c["lambda_precision"], seed=c["seed"],
                    newton=port.Newton(step=nw["step"], max_iter=nw["max_iter"],
                                       tol=nw["tol"], floor=nw["floor"], retry=nw["retry"],
                                       retry_step=nw["retry_step"],
                                       retry_max_iter=nw["retry_max_iter"]),
                    digest=bytes.fromhex(run["digest"]))
