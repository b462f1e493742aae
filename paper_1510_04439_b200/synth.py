"""Seeded synthetic functional datasets shaped like BASELINE.json's configs.

The processes follow the reference's simulation models (simulate.hpp:98-150):
mean + sum_l sqrt(lambda_l) xi_l phi_l + noise, with unit-norm product-sine
eigenfunctions on midpoint grids.  Draws use numpy's PCG64 (the data only
has to be the same for both arms of a comparison, not bit-equal to the
reference generator).  Returned as CSR arrays (offsets, coords, values) plus
a FunctionalDataset view on request.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SynthData:
    dim: int
    axes: list           # grid axes
    mask: object         # None or uint8[G]
    offsets: np.ndarray  # int64[n+1]
    coords: np.ndarray   # float64[N*dim]
    values: np.ndarray   # float64[N]
    h: list              # bandwidth per axis

    @property
    def n_samples(self) -> int:
        return self.offsets.size - 1

    def dataset(self):
        from .api import FunctionalDataset
        return FunctionalDataset.from_csr(self.dim, self.offsets, self.coords, self.values)

    def grid(self):
        from .api import EvaluationGrid
        return EvaluationGrid(self.axes, self.mask)


def midpoint_axis(n: int, lo: float = 0.0, hi: float = 1.0) -> list:
    d = (hi - lo) / float(n)
    return [lo + d * (float(i) + 0.5) for i in range(n)]


def _product_sines(pts: np.ndarray, L: int) -> np.ndarray:
    """phi_l(t) = sqrt(2^d) prod_k sin(2 l pi t_k), l = 1..L  (unit norm on [0,1]^d)."""
    d = pts.shape[1]
    out = np.empty((L, pts.shape[0]))
    for l in range(1, L + 1):
        out[l - 1] = np.sqrt(2.0 ** d) * np.prod(np.sin(2.0 * l * np.pi * pts), axis=1)
    return out


def _bump_mean(pts: np.ndarray) -> np.ndarray:
    return np.exp(np.sum((pts - 0.5) ** 2, axis=1))


def grid_nodes(dim: int, cells: int, n: int, h: float, seed: int = 20260815,
               lam=(16.0, 4.0, 1.0, 0.25), sigma2: float = 1.0 / 16.0) -> SynthData:
    """Every sample observed at every node of a midpoint [0,1]^dim grid
    (SimDesign::GridNodes; configs 2, 3 and 5)."""
    ax = midpoint_axis(cells)
    axes = [ax] * dim
    mesh = np.meshgrid(*[np.asarray(ax)] * dim, indexing="ij")
    pts = np.stack([m.ravel() for m in mesh], axis=1)  # [G, dim], last axis fastest
    G = pts.shape[0]
    rng = np.random.default_rng(seed)
    phi = _product_sines(pts, len(lam))
    mu = _bump_mean(pts)
    scores = rng.standard_normal((n, len(lam))) * np.sqrt(np.asarray(lam))
    values = (mu[None, :] + scores @ phi + np.sqrt(sigma2) * rng.standard_normal((n, G))).ravel()
    coords = np.tile(pts.ravel(), n)
    offsets = np.arange(n + 1, dtype=np.int64) * G
    return SynthData(dim, axes, None, offsets, np.ascontiguousarray(coords), np.ascontiguousarray(values),
                     [h] * dim)


def sparse_masked(cells: int, n: int, h: float, seed: int = 20260815, n_min: int = 5, n_max: int = 20,
                  lam=(16.0, 4.0, 1.0, 0.25), sigma2: float = 1.0 / 16.0) -> SynthData:
    """Config 4: sparse longitudinal 2-d design on an elliptical (PM2.5-style)
    mask over a uniform [0,1]^2 grid; N_i ~ U{n_min..n_max} observations per
    subject, uniform inside the mask by rejection."""
    ax = [float(i) / float(cells - 1) for i in range(cells)]
    X, Y = np.meshgrid(np.asarray(ax), np.asarray(ax), indexing="ij")
    mask = ((((X - 0.5) / 0.45) ** 2 + ((Y - 0.5) / 0.3) ** 2) <= 1.0).astype(np.uint8).ravel()
    rng = np.random.default_rng(seed)
    counts = rng.integers(n_min, n_max + 1, size=n)
    coords, values = [], []
    for i in range(n):
        pts = np.empty((0, 2))
        while pts.shape[0] < counts[i]:
            cand = rng.random((2 * counts[i], 2))
            keep = (((cand[:, 0] - 0.5) / 0.45) ** 2 + ((cand[:, 1] - 0.5) / 0.3) ** 2) <= 1.0
            pts = np.vstack([pts, cand[keep]])
        pts = pts[:counts[i]]
        sc = rng.standard_normal(len(lam)) * np.sqrt(np.asarray(lam))
        y = _bump_mean(pts) + sc @ _product_sines(pts, len(lam)) + np.sqrt(sigma2) * rng.standard_normal(counts[i])
        coords.append(pts.ravel())
        values.append(y)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return SynthData(2, [ax, ax], mask, offsets, np.ascontiguousarray(np.concatenate(coords)),
                     np.ascontiguousarray(np.concatenate(values)), [h, h])


def random_points(dim: int, cells: int, n: int, n_obs: int, h: float, seed: int = 7,
                  uniform_grid: bool = True) -> SynthData:
    """Off-node observations uniform in the hull (exercises fractional
    multilinear masses and all 3^d band codes)."""
    ax = ([float(i) / float(cells - 1) for i in range(cells)] if uniform_grid else midpoint_axis(cells))
    lo, hi = ax[0], ax[-1]
    rng = np.random.default_rng(seed)
    pts = lo + (hi - lo) * rng.random((n * n_obs, dim))
    y = _bump_mean(pts) + rng.standard_normal(n * n_obs)
    offsets = np.arange(n + 1, dtype=np.int64) * n_obs
    return SynthData(dim, [ax] * dim, None, offsets, np.ascontiguousarray(pts.ravel()), np.ascontiguousarray(y),
                     [h] * dim)


def sim1(n: int = 200, points: int = 100, cells: int = 100, h: float = 0.25, seed: int = 20260815) -> SynthData:
    """Config 1: the reference's Sim I process (simulate.hpp:101-118) on
    [0, 10] with an equispaced design."""
    ax = midpoint_axis(cells, 0.0, 10.0)
    t = np.linspace(0.0, 10.0, points)
    phi = np.stack([-np.cos(np.pi * t / 10.0) / np.sqrt(5.0), np.sin(np.pi * t / 10.0) / np.sqrt(5.0)])
    rng = np.random.default_rng(seed)
    sc = rng.standard_normal((n, 2)) * np.sqrt(np.array([4.0, 1.0]))
    y = (t + np.sin(t))[None, :] + sc @ phi + 0.5 * rng.standard_normal((n, points))
    offsets = np.arange(n + 1, dtype=np.int64) * points
    return SynthData(1, [ax], None, offsets, np.ascontiguousarray(np.tile(t, n)), np.ascontiguousarray(y.ravel()),
                     [h])


def long_format_bytes(sd: SynthData, n_samples: int | None = None) -> bytes:
    """The dataset as the reference's write_long_format (io.hpp:158-178) lays
    it out: tab-separated, header sample_id/t1../y, ids s<i>, %.17g numbers.
    n_samples limits the table to the first subjects (bounded samples)."""
    n = sd.offsets.size - 1 if n_samples is None else min(n_samples, sd.offsets.size - 1)
    d = sd.dim
    N = int(sd.offsets[n])
    coords = sd.coords[:N * d]
    uniq, inv = np.unique(coords, return_inverse=True)
    ctxt = np.char.mod("%.17g", uniq)[inv].reshape(N, d)
    rows = ["\t".join(r) for r in ctxt.tolist()] if d > 1 else ctxt[:, 0].tolist()
    vtxt = np.char.mod("%.17g", sd.values[:N]).tolist()
    parts = ["sample_id\t" + "\t".join("t%d" % (k + 1) for k in range(d)) + "\ty\n"]
    for i in range(n):
        a, b = int(sd.offsets[i]), int(sd.offsets[i + 1])
        sid = "s%d\t" % i
        parts.append("".join([sid + rows[j] + "\t" + vtxt[j] + "\n" for j in range(a, b)]))
    return "".join(parts).encode()
