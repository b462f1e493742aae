"""Seeded synthetic functional datasets shaped like BASELINE.json's configs.

The processes follow the reference's simulation models (simulate.hpp:98-150):
mean + sum_l sqrt(lambda_l) xi_l phi_l + noise, with unit-norm product-sine
eigenfunctions on midpoint grids.  Draws use numpy's PCG64 (the data only
has to be the same for both arms of a comparison, not bit-equal to the
reference generator).  Returned as CSR arrays (offsets, coords, values) plus
a FunctionalDataset view on request.

The BASELINE configs themselves (`config()`, `simulate()`) are drawn with the
reference's own generator, restated in the library (`dfpca_simulate`,
simulate.hpp:163-245): bit-identical to the reference's generate(), so the
configs' inputs are the reference's.
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


# ---------------------------------------------------- reference generator --

SIM_SIM1, SIM_SIM2, SIM_IMAGES2, SIM_SPARSE2 = 1, 2, 3, 4


def ellipse_mask(axes) -> np.ndarray:
    """Config 4's PM2.5-style domain on the grid nodes."""
    X, Y = np.meshgrid(np.asarray(axes[0]), np.asarray(axes[1]), indexing="ij")
    return ((((X - 0.5) / 0.45) ** 2 + ((Y - 0.5) / 0.3) ** 2) <= 1.0).astype(np.uint8).ravel()


def simulate(kind: int, axes, mask, n: int, h: float, points_per_sample: int = 0,
             seed: int = 20260815) -> SynthData:
    """The reference's generate() for one of the models of dfpca_simulate
    (include/dfpca_cuda.h), through the library (host code, no device)."""
    import ctypes as C
    from . import _lib
    from .api import EvaluationGrid
    lib = _lib.load()
    g = EvaluationGrid([list(a) for a in axes], mask)
    offsets = np.zeros(n + 1, dtype=np.int64)
    PD = C.POINTER(C.c_double)
    PI64 = C.POINTER(C.c_int64)
    st = lib.dfpca_simulate(kind, C.byref(g.desc()), n, points_per_sample, seed, offsets.ctypes.data_as(PI64),
                            None, None)
    if st != 0:
        raise ValueError(f"dfpca_simulate: invalid model {kind} / grid / n")
    dim = len(axes)
    N = int(offsets[-1])
    coords = np.empty(N * dim)
    values = np.empty(N)
    st = lib.dfpca_simulate(kind, C.byref(g.desc()), n, points_per_sample, seed, offsets.ctypes.data_as(PI64),
                            coords.ctypes.data_as(PD), values.ctypes.data_as(PD))
    assert st == 0
    return SynthData(dim, [list(a) for a in axes], mask, offsets, coords, values, [h] * dim)


# BASELINE.json configs: model, grid, n, bandwidth.
CONFIGS = {
    1: "d=1 Sim I: n=200 curves x 100 equispaced points, midpoint [0,10] 100 nodes, h=0.25",
    2: "d=2 images: n=500 on midpoint 32x32, h=0.1",
    3: "d=2 images: n=2000 on midpoint 64x64, h=0.1 (and 0.3)",
    4: "d=2 sparse longitudinal: n=2000, N_i in 5..20, ellipse mask on uniform 64x64, h=0.15",
    5: "d=3 Sim II: n=1000 on midpoint 32^3, h=0.1",
}


def config(cfg: int, n: int | None = None, h: float | None = None, cells: int | None = None,
           seed: int = 20260815) -> SynthData:
    """Inputs of BASELINE config `cfg` drawn by the reference's generator;
    n / h / cells override the config's sample count, bandwidth, grid size."""
    if cfg == 1:
        c = cells or 100
        return simulate(SIM_SIM1, [midpoint_axis(c, 0.0, 10.0)], None, n or 200, h or 0.25, 100, seed)
    if cfg in (2, 3):
        c = cells or (32 if cfg == 2 else 64)
        ax = midpoint_axis(c)
        return simulate(SIM_IMAGES2, [ax, ax], None, n or (500 if cfg == 2 else 2000), h or 0.1, 0, seed)
    if cfg == 4:
        c = cells or 64
        ax = [float(i) / float(c - 1) for i in range(c)]
        ax[-1] = 1.0
        return simulate(SIM_SPARSE2, [ax, ax], ellipse_mask([ax, ax]), n or 2000, h or 0.15, 0, seed)
    if cfg == 5:
        c = cells or 32
        ax = midpoint_axis(c)
        return simulate(SIM_SIM2, [ax, ax, ax], None, n or 1000, h or 0.1, 0, seed)
    raise ValueError(f"no config {cfg}")
