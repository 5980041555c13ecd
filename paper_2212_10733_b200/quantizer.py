"""Product-quantiser codebook container (reference quantizer.py:22-50).

Training (k-means++ + Lloyd), encoding and decoding run on device
(``csrc/kmeans.cu``, ``csrc/select.cu``); this is the section codec.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

__all__ = ["PQCodebook", "ALLOWED_K"]

ALLOWED_K = (16, 64, 256)


@dataclass(frozen=True)
class PQCodebook:
    centroids: np.ndarray  # (latent_dim, k) float32, each row sorted

    def __post_init__(self):
        c = np.asarray(self.centroids, dtype=np.float32)
        if c.ndim != 2:
            raise ConfigError("centroids must be (latent_dim, k)")
        object.__setattr__(self, "centroids", c)

    @property
    def latent_dim(self) -> int:
        return self.centroids.shape[0]

    @property
    def k(self) -> int:
        return self.centroids.shape[1]

    @property
    def bits(self) -> int:
        return int(self.k - 1).bit_length()

    def to_bytes(self) -> bytes:
        return self.centroids.astype("<f4").tobytes()

    @classmethod
    def from_bytes(cls, raw: bytes, latent_dim: int, k: int):
        return cls(centroids=np.frombuffer(raw, dtype="<f4").reshape(latent_dim, k).copy())
