"""Bi-Maxwellian synthetic f0 corpus (reference fdata.py:170-347), restated.

Every numpy call that touches a PCG64 stream or rounds a value is kept in
the reference's order, so the corpus is byte-identical to
``mlk.gen_synthetic`` (pinned by ``data_sha`` in every golden fixture).
"""

from __future__ import annotations

import numpy as np

from paper_2212_10733_b200.errors import ConfigError
from paper_2212_10733_b200.fdata import FDataset, SyntheticParams, VelocityGrid

TWO_PI = 2 * np.pi
GOLDEN = 0.6180339887498949
PLANE_SEED_OFFSET = 0x9E3779B97F4A7C15


class SyntheticCorpus:
    """The per-node plasma state of one corpus and the images it implies."""

    def __init__(self, n_nodes: int, grid: VelocityGrid, params: SyntheticParams):
        if n_nodes < 1:
            raise ConfigError("need at least one plane and one node")
        self.n_nodes, self.grid, self.p = n_nodes, grid, params

    # -- node layout (fdata.py:195-240) ---------------------------------
    def layout(self):
        """ln-density per surface and the node count of each surface."""
        k = min(self.p.n_surfaces, self.n_nodes)
        if k == 1:
            return np.zeros(1), np.array([self.n_nodes])
        lev = -self.p.density_ln_span * np.arange(k) / (k - 1)
        wt = np.exp(-1.5 * lev)
        cnt = np.maximum(np.floor(self.n_nodes * wt / wt.sum()), 1.0).astype(np.int64)
        cnt[-1] += self.n_nodes - cnt.sum()
        if cnt[-1] < 1:
            cnt = np.full(k, self.n_nodes // k, dtype=np.int64)
            cnt[:self.n_nodes % k] += 1
        return lev, cnt

    def surface(self):
        """Surface index of every node (golden-ratio stratified)."""
        _, cnt = self.layout()
        frac = (np.arange(self.n_nodes) * GOLDEN) % 1.0
        return np.searchsorted(np.cumsum(cnt)[:-1] / self.n_nodes, frac, side="right")

    # -- random node fields (fdata.py:170-192) --------------------------
    def _fourier(self, rng, smooth):
        x = np.arange(self.n_nodes) / self.n_nodes
        acc = np.zeros(self.n_nodes)
        for m in range(1, max(1, int(round(1.0 / smooth))) + 1):
            a, b = rng.standard_normal(2)
            acc += (a * np.cos(TWO_PI * m * x) + b * np.sin(TWO_PI * m * x)) / (1.0 + m)
        top = np.max(np.abs(acc))
        return acc / top if top > 0 else acc

    def _window(self, rng):
        out = np.zeros(self.n_nodes)
        if self.p.turbulent_fraction <= 0:
            return out
        width = max(4, int(self.p.turbulent_fraction * self.n_nodes / 2))
        x = np.arange(self.n_nodes)
        for _ in range(2):
            mid = rng.integers(width, max(self.n_nodes // 2, width + 1))
            out = np.maximum(out, np.exp(-((x - mid) / (0.7 * width)) ** 4))
        return out

    # -- moments and images (fdata.py:243-320) --------------------------
    def fields(self):
        """(n, u_par, t_perp, t_par) per node, n scaled to value_max."""
        p, g = self.p, self.grid
        rng = np.random.Generator(np.random.PCG64(p.seed))
        t0 = 0.5 * g.mass * (p.blob_fraction * g.v_perp[-1]) ** 2
        lev, _ = self.layout()
        surf = self.surface()
        n_edge = max(min(3, p.n_surfaces // 2), 1)
        win = self._window(rng) * (surf >= p.n_surfaces - n_edge)
        bursts = []
        for signed in (True, False, False):
            f = self._fourier(rng, p.smoothness / 2) ** 3
            prod = win * (f if signed else np.abs(f))
            top = np.max(np.abs(prod))
            bursts.append(prod / top if top > 0 else prod)
        vth = np.sqrt(2.0 * t0 / g.mass)
        u = vth * (p.bulk_amplitude * self._fourier(rng, p.smoothness)
                   + p.turbulence_flow * bursts[0])
        temps = [t0 * np.exp(np.clip(p.bulk_amplitude * self._fourier(rng, p.smoothness)
                                     + p.turbulence_temp * b, -1.5, 3.5)) for b in bursts[1:]]
        n = np.exp(lev[surf])
        shp, z = self.shapes(u, *temps)
        n = n * (p.value_max / np.max(n / z * np.max(shp, axis=(1, 2))))
        return n, u, temps[0], temps[1]

    def shapes(self, u, t_perp, t_par):
        """exp(-m v_perp^2 / 4 t_perp - m (v_par - u)^2 / 4 t_par) and sum(shape * vol)."""
        g = self.grid
        e_perp = g.mass * g.v_perp[:, None] ** 2
        d_par = g.v_par[None, None, :] - u[:, None, None]
        img = np.exp(-e_perp[None, :, :] / (4.0 * t_perp[:, None, None])
                     - g.mass * d_par ** 2 / (4.0 * t_par[:, None, None]))
        return img, np.einsum("nrc,rc->n", img, g.vol)

    def base(self):
        """(n_nodes, rows, cols): every plane's image before its rho term."""
        n, u, tp, tl = self.fields()
        shp, z = self.shapes(u, tp, tl)
        return shp * (n / z)[:, None, None]

    def planes(self, n_planes: int) -> np.ndarray:
        """(n_planes, n_nodes, rows, cols) with the per-plane rho / noise draws."""
        if n_planes < 1:
            raise ConfigError("need at least one plane and one node")
        p, base = self.p, self.base()
        out = np.empty((n_planes,) + base.shape)
        rng = np.random.Generator(np.random.PCG64(p.seed + PLANE_SEED_OFFSET))
        for k in range(n_planes):
            img = base.copy()
            if p.rho > 0:
                img *= 1.0 + p.rho * rng.uniform(-1.0, 1.0, size=img.shape)
            if p.noise > 0:
                img += (p.noise * np.max(img, axis=(1, 2), keepdims=True)
                        * rng.uniform(-1.0, 1.0, size=img.shape))
            img = np.maximum(img, 0.0)
            img[img < p.value_min] = 0.0
            out[k] = img
        return out


def synth_base(n_nodes: int, grid: VelocityGrid, params: SyntheticParams) -> np.ndarray:
    return SyntheticCorpus(n_nodes, grid, params).base()


def gen_synthetic(n_planes: int, n_nodes: int, grid: VelocityGrid,
                  params: SyntheticParams) -> FDataset:
    """Byte-identical to the reference's gen_synthetic (fdata.py:322-347)."""
    if n_planes < 1 or n_nodes < 1:
        raise ConfigError("need at least one plane and one node")
    return FDataset(grid=grid, data=SyntheticCorpus(n_nodes, grid, params).planes(n_planes),
                    timestep=0)


def gen_synthetic_device(n_planes: int, n_nodes: int, grid: VelocityGrid,
                         params: SyntheticParams, device, plane_range=None, pad_elems: int = 2):
    """Planes [lo, hi) of the same corpus generated in device memory by the
    product's plane kernel (paper_2212_10733_b200.fdata.synth_planes_device)
    from this module's per-node base images."""
    from paper_2212_10733_b200.fdata import synth_planes_device
    if n_planes < 1 or n_nodes < 1:
        raise ConfigError("need at least one plane and one node")
    lo, hi = plane_range or (0, n_planes)
    base = synth_base(n_nodes, grid, params) if hi > lo else None
    return synth_planes_device(base, n_planes, n_nodes, grid, params, device, (lo, hi),
                               pad_elems)
