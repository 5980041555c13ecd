"""Tied-weight linear autoencoder model container (reference autoencoder.py:26-74).

The hot path consumes trained weights (static-model mode,
pipeline.py:206-207); the contraction itself runs on device in
``csrc/stage1.cu`` (encode) and every kernel that needs a reconstruction
(decode).  Training is outside the B200 hot path.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

__all__ = ["AEModel", "TrainConfig", "train", "STD_FLOOR"]

STD_FLOOR = 1e-30


@dataclass(frozen=True)
class AEModel:
    weights: np.ndarray   # (latent_dim, D) float32
    norm_mean: float
    norm_std: float

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=np.float32)
        if w.ndim != 2:
            raise ConfigError("weights must be a (latent_dim, D) matrix")
        if not self.norm_std > 0:
            raise ConfigError("normalizer std must be positive")
        object.__setattr__(self, "weights", w)

    @property
    def latent_dim(self) -> int:
        return self.weights.shape[0]

    @property
    def input_dim(self) -> int:
        return self.weights.shape[1]

    def to_bytes(self) -> bytes:
        """Weights section payload: ``<dd`` normaliser + f32 weights (autoencoder.py:44-46)."""
        return struct.pack("<dd", self.norm_mean, self.norm_std) + \
            self.weights.astype("<f4").tobytes()

    @classmethod
    def from_bytes(cls, raw: bytes, latent_dim: int, input_dim: int):
        mean, std = struct.unpack_from("<dd", raw, 0)
        w = np.frombuffer(raw, dtype="<f4", offset=16, count=latent_dim * input_dim)
        return cls(weights=w.reshape(latent_dim, input_dim).copy(), norm_mean=mean,
                   norm_std=std)


@dataclass(frozen=True)
class TrainConfig:
    learning_rate: float = 0.001
    batch_size: int = 128
    epochs: int = 100
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    seed: int = 0


def train(images, config: TrainConfig, init=None, latent_dim: int = 4):
    raise ConfigError("AE training is outside the B200 hot path: supply static per-shard "
                      "models through TimestepState (static_model=True)")
