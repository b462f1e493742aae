"""Python mirror of the reference's hot-path API (proj/include/dfpca), backed by
libdfpca_cuda.so through its C-ABI (include/dfpca_cuda.h).

Names, argument meaning and error behaviour follow the C++ headers:
    linear_bin            binning.hpp:82
    single_block_plan     fft_smoother.hpp:66
    make_block_plan       fft_smoother.hpp:77
    validate_block_plan   fft_smoother.hpp:101
    fft_local_linear      fft_smoother.hpp:498 / 572
    fft_covariance        fft_smoother.hpp:585 / 740
    blockwise_apply       fft_smoother.hpp:747 / 754
    matrixize             eigensolve.hpp:71
    default_sketch_size   eigensolve.hpp:231
    randomized_eig        eigensolve.hpp:245
    select_components_fve eigensolve.hpp:282
    eig_residuals         eigensolve.hpp:294
    read_long_format      io.hpp:115 (parsed on the GPU)
    write_long_format, read_grid, write_grid   io.hpp:158-259 (host)
Every compute call runs on the GPU; there is no CPU fallback -- a missing
library or device raises immediately.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import DfpcaGrid, DfpcaPlan, check

# ----------------------------------------------------------------- errors --


class ErrorClass(Enum):
    """errors.hpp:11-17"""
    Usage = 1
    Parse = 2
    Config = 3
    Numeric = 4
    Version = 5


class Error(RuntimeError):
    """dfpca::Error (errors.hpp:19-33): what() == name + ": " + message."""

    def __init__(self, cls: ErrorClass, name: str, message: str):
        super().__init__(f"{name}: {message}")
        self.error_class = cls
        self._name = name
        self.message = message

    def name(self) -> str:
        return self._name

    def exit_code(self) -> int:
        return self.error_class.value


_lib.set_error_factory(lambda cls, name, msg: Error(ErrorClass(cls), name, msg))

# ------------------------------------------------------------------- grid --


def outside_value() -> float:
    return float("nan")


def is_outside(v) -> bool:
    return bool(np.isnan(v))


@dataclass
class Box:
    """grid.hpp:24-43 (half-open per-axis index range)."""
    lo: list
    hi: list

    def dim(self) -> int:
        return len(self.lo)

    def extent(self, k: int) -> int:
        return self.hi[k] - self.lo[k]

    def volume(self) -> int:
        v = 1
        for k in range(len(self.lo)):
            v *= self.extent(k)
        return v

    @staticmethod
    def full(shape) -> "Box":
        return Box([0] * len(shape), list(shape))


class EvaluationGrid:
    """grid.hpp:92-230: strictly increasing axes, optional uint8 mask, row-major
    last-axis-fastest flattening."""

    def __init__(self, axes: Sequence[Sequence[float]], mask: Optional[Sequence[int]] = None):
        if len(axes) == 0:
            raise Error(ErrorClass.Config, "InvalidArgument", "grid needs at least one axis")
        self._axes = [np.ascontiguousarray(a, dtype=np.float64) for a in axes]
        for k, ax in enumerate(self._axes):
            if ax.size < 2:
                raise Error(ErrorClass.Config, "InvalidArgument", f"grid axis {k} needs >= 2 nodes")
            if not np.all(ax[1:] > ax[:-1]):
                raise Error(ErrorClass.Config, "InvalidArgument",
                            f"grid axis {k} is not strictly increasing")
        self._shape = [int(a.size) for a in self._axes]
        self._size = int(np.prod(self._shape))
        self._mask = None
        if mask is not None:
            m = np.ascontiguousarray(mask, dtype=np.uint8)
            if m.size != self._size:
                raise Error(ErrorClass.Config, "InvalidArgument",
                            "mask size does not match grid node count")
            self._mask = m
        self._spacing = []
        self._equispaced = True
        for ax in self._axes:
            gap = (ax[-1] - ax[0]) / float(ax.size - 1)
            self._spacing.append(gap)
            if np.any(np.abs((ax[1:] - ax[:-1]) - gap) > 1e-9 * gap):
                self._equispaced = False
        self._desc = None

    @staticmethod
    def uniform(lo, hi, counts) -> "EvaluationGrid":
        axes = []
        for k in range(len(lo)):
            if not hi[k] > lo[k]:
                raise Error(ErrorClass.Config, "DegenerateAxis", f"axis {k} has zero extent")
            n = counts[k]
            ax = [lo[k] + (hi[k] - lo[k]) * float(i) / float(n - 1) for i in range(n)]
            ax[-1] = hi[k]
            axes.append(ax)
        return EvaluationGrid(axes)

    @staticmethod
    def midpoint(lo, hi, counts) -> "EvaluationGrid":
        axes = []
        for k in range(len(lo)):
            if not hi[k] > lo[k]:
                raise Error(ErrorClass.Config, "DegenerateAxis", f"axis {k} has zero extent")
            n = counts[k]
            d = (hi[k] - lo[k]) / float(n)
            axes.append([lo[k] + d * (float(i) + 0.5) for i in range(n)])
        return EvaluationGrid(axes)

    def dim(self) -> int:
        return len(self._axes)

    def axes(self):
        return self._axes

    def axis(self, k: int):
        return self._axes[k]

    def shape(self):
        return list(self._shape)

    def strides(self):
        s = [1] * self.dim()
        for k in range(self.dim() - 2, -1, -1):
            s[k] = s[k + 1] * self._shape[k + 1]
        return s

    def size(self) -> int:
        return self._size

    def equispaced(self) -> bool:
        return self._equispaced

    def spacing(self, k: int) -> float:
        return self._spacing[k]

    def cell_volume(self) -> float:
        v = 1.0
        for s in self._spacing:
            v *= s
        return v

    def mask(self):
        return self._mask

    def has_mask(self) -> bool:
        return self._mask is not None

    def in_mask(self, flat: int) -> bool:
        return self._mask is None or self._mask[flat] != 0

    def in_mask_count(self) -> int:
        return self._size if self._mask is None else int(np.count_nonzero(self._mask))

    def node(self, k: int, i: int) -> float:
        return float(self._axes[k][i])

    def node_coords(self, flat: int):
        out = [0.0] * self.dim()
        for k in range(self.dim() - 1, -1, -1):
            out[k] = float(self._axes[k][flat % self._shape[k]])
            flat //= self._shape[k]
        return out

    def hull_lo(self, k: int) -> float:
        return float(self._axes[k][0])

    def hull_hi(self, k: int) -> float:
        return float(self._axes[k][-1])

    def desc(self) -> DfpcaGrid:
        if self._desc is None:
            g = DfpcaGrid()
            g.dim = self.dim()
            for k in range(self.dim()):
                g.shape[k] = self._shape[k]
                g.axes[k] = self._axes[k].ctypes.data_as(C.POINTER(C.c_double))
            g.mask = self._mask.ctypes.data_as(C.POINTER(C.c_uint8)) if self._mask is not None else None
            self._desc = g
        return self._desc


# ---------------------------------------------------------------- dataset --


@dataclass
class Sample:
    """dataset.hpp:20-27: id, flat coords (N * dim), values (N)."""
    id: str
    coords: np.ndarray
    values: np.ndarray

    def n_obs(self) -> int:
        return int(np.asarray(self.values).size)


@dataclass
class FunctionalDataset:
    """dataset.hpp:36-71.  csr() is cached until `samples` is rebound or
    changes length; call invalidate() after editing samples in place."""
    dim: int = 0
    samples: list = field(default_factory=list)
    _csr: tuple = field(default=None, repr=False, compare=False)
    _csr_key: tuple = field(default=None, repr=False, compare=False)

    def invalidate(self):
        self._csr = None

    @staticmethod
    def from_csr(dim: int, offsets, coords, values, ids=None) -> "FunctionalDataset":
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        values = np.ascontiguousarray(values, dtype=np.float64)
        n = offsets.size - 1
        samples = [Sample(ids[i] if ids else str(i), coords[offsets[i] * dim:offsets[i + 1] * dim],
                          values[offsets[i]:offsets[i + 1]]) for i in range(n)]
        d = FunctionalDataset(dim, samples)
        d._csr = (offsets, coords, values)
        d._csr_key = (id(d.samples), len(d.samples))
        return d

    def n_samples(self) -> int:
        return len(self.samples)

    def n_obs(self) -> int:
        return sum(s.n_obs() for s in self.samples)

    def csr(self):
        """(offsets int64[n+1], coords f64[N*dim], values f64[N])"""
        key = (id(self.samples), len(self.samples))
        if self._csr is not None and self._csr_key == key:
            return self._csr
        n = len(self.samples)
        counts = np.fromiter((s.n_obs() for s in self.samples), dtype=np.int64, count=n)
        offsets = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=offsets[1:])
        if n:
            coords = np.concatenate([np.asarray(s.coords, dtype=np.float64).ravel() for s in self.samples])
            values = np.concatenate([np.asarray(s.values, dtype=np.float64).ravel() for s in self.samples])
        else:
            coords = np.zeros(0)
            values = np.zeros(0)
        self._csr = (offsets, np.ascontiguousarray(coords), np.ascontiguousarray(values))
        self._csr_key = key
        return self._csr


@dataclass
class Bandwidth:
    """dataset.hpp:79-109."""
    h: list

    def dim(self) -> int:
        return len(self.h)

    def __getitem__(self, k):
        return self.h[k]

    def validate(self, grid: EvaluationGrid):
        ext = [grid.hull_hi(k) - grid.hull_lo(k) for k in range(grid.dim())]
        if len(self.h) != len(ext):
            raise Error(ErrorClass.Config, "InvalidBandwidth", "bandwidth dimension mismatch")
        for k, hk in enumerate(self.h):
            if not hk > 0.0:
                raise Error(ErrorClass.Config, "InvalidBandwidth", f"bandwidth axis {k} must be positive")
            if hk > ext[k] * (1.0 + 1e-12):
                raise Error(ErrorClass.Config, "InvalidBandwidth",
                            f"bandwidth axis {k} exceeds the axis extent")

    def scaled(self, f: float) -> "Bandwidth":
        return Bandwidth([x * f for x in self.h])

    def arr(self):
        return np.ascontiguousarray(self.h, dtype=np.float64)


# ----------------------------------------------------------------- binning --


@dataclass
class BinOptions:
    """binning.hpp:14-20."""
    mean_path: bool = True
    covariance_path: bool = False


class BinnedData:
    """binning.hpp:41-74.  Device-resident; host fields are materialized on
    first access (mass, wvalue, wsquare, per_sample, diag_mass, diag_value,
    sample_sizes)."""

    @dataclass
    class SampleGrids:
        sample_index: int
        pair_weight: float
        mass: np.ndarray
        value: np.ndarray

    def __init__(self, handle, grid: EvaluationGrid):
        self._h = handle
        self.grid = grid
        n, npair, G, codes, hm, hc = (C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64(),
                                      C.c_int(), C.c_int())
        _lib.lib().dfpca_binned_info(handle, C.byref(n), C.byref(npair), C.byref(G),
                                     C.byref(codes), C.byref(hm), C.byref(hc))
        self._n, self._npair, self._G, self._codes = n.value, npair.value, G.value, codes.value
        self.has_mean_path = bool(hm.value)
        self.has_covariance_path = bool(hc.value)
        self._host = None

    def __del__(self):
        try:
            if self._h:
                _lib.lib().dfpca_binned_free(self._h)
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def offset_codes(self) -> int:
        return self._codes

    def _fetch(self):
        if self._host is not None:
            return self._host
        G, npair, codes, n = self._G, self._npair, self._codes, self._n
        f = lambda k: np.zeros(k, dtype=np.float64)
        mass, wv, ws = (f(G), f(G), f(G)) if self.has_mean_path else (f(0), f(0), f(0))
        si = np.zeros(npair, dtype=np.int64)
        pw = f(npair)
        psm = f(npair * G)
        psv = f(npair * G)
        dm, dv = (f(G * codes), f(G * codes)) if self.has_covariance_path else (f(0), f(0))
        sizes = np.zeros(n, dtype=np.int64)
        P = lambda a: a.ctypes.data_as(C.POINTER(C.c_double)) if a.size else None
        PI = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64)) if a.size else None
        check(_lib.lib().dfpca_binned_download(_lib.ctx(), self._h, P(mass), P(wv), P(ws), PI(si), P(pw),
                                               P(psm), P(psv), P(dm), P(dv), PI(sizes)))
        per = [BinnedData.SampleGrids(int(si[i]), float(pw[i]), psm[i * G:(i + 1) * G],
                                      psv[i * G:(i + 1) * G]) for i in range(npair)]
        self._host = dict(mass=mass, wvalue=wv, wsquare=ws, per_sample=per, diag_mass=dm,
                          diag_value=dv, sample_sizes=[int(x) for x in sizes])
        return self._host

    def __getattr__(self, name):
        if name in ("mass", "wvalue", "wsquare", "per_sample", "diag_mass", "diag_value", "sample_sizes"):
            return self._fetch()[name]
        raise AttributeError(name)

    @staticmethod
    def from_host(grid: EvaluationGrid, *, mass=None, wvalue=None, wsquare=None, per_sample=(),
                  diag_mass=None, diag_value=None, sample_sizes=(), has_mean_path=True,
                  has_covariance_path=False) -> "BinnedData":
        """Uploads a hand-built BinnedData (the reference tests build them)."""
        G = grid.size()
        arr = lambda a, n: np.ascontiguousarray(np.zeros(n) if a is None else a, dtype=np.float64)
        m, wv, ws = arr(mass, G), arr(wvalue, G), arr(wsquare, G)
        codes = 3 ** grid.dim()
        dm, dv = arr(diag_mass, G * codes), arr(diag_value, G * codes)
        npair = len(per_sample)
        si = np.array([p.sample_index for p in per_sample], dtype=np.int64)
        pw = np.array([p.pair_weight for p in per_sample], dtype=np.float64)
        psm = np.ascontiguousarray(np.concatenate([p.mass for p in per_sample]) if npair else np.zeros(0))
        psv = np.ascontiguousarray(np.concatenate([p.value for p in per_sample]) if npair else np.zeros(0))
        sizes = np.array(list(sample_sizes), dtype=np.int64)
        P = lambda a: a.ctypes.data_as(C.POINTER(C.c_double)) if a.size else None
        PI = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64)) if a.size else None
        h = C.c_void_p()
        check(_lib.lib().dfpca_binned_upload(_lib.ctx(), C.byref(grid.desc()), len(sizes), PI(sizes),
                                             int(has_mean_path), P(m), P(wv), P(ws),
                                             int(has_covariance_path), npair, PI(si), P(pw), P(psm),
                                             P(psv), P(dm), P(dv), C.byref(h)))
        return BinnedData(h, grid)


def linear_bin(data: FunctionalDataset, grid: EvaluationGrid, opt: BinOptions = BinOptions()) -> BinnedData:
    """binning.hpp:82-183 on the GPU (bit-exact)."""
    if data.dim != grid.dim():
        raise Error(ErrorClass.Config, "InvalidArgument", "dataset/grid dimension mismatch")
    offsets, coords, values = data.csr()
    h = C.c_void_p()
    status = _lib.lib().dfpca_linear_bin(
        _lib.ctx(), C.byref(grid.desc()), len(data.samples),
        offsets.ctypes.data_as(C.POINTER(C.c_int64)),
        coords.ctypes.data_as(C.POINTER(C.c_double)) if coords.size else None,
        values.ctypes.data_as(C.POINTER(C.c_double)) if values.size else None,
        int(opt.mean_path), int(opt.covariance_path), C.byref(h))
    if status != 0:
        err = _lib.last_error()
        if err.name() == "ObservationOutsideGrid":
            i, j = _lib.last_error_location()
            raise Error(err.error_class, err.name(),
                        f"sample '{data.samples[i].id}' observation {j} lies outside the grid hull")
        raise err
    return BinnedData(h, grid)


# ------------------------------------------------------------- smoothing --


class MomentTarget(Enum):
    """fft_smoother.hpp:34"""
    Mean = 0
    Squares = 1


class SurfaceKind(Enum):
    """surface.hpp:12-16"""
    Mean = 0
    Covariance = 1
    DiagPlusNoise = 2


class SurfaceEstimate:
    """surface.hpp:26-35.  `values` is a host numpy array (downloaded lazily
    for device-resident covariance surfaces)."""

    def __init__(self, grid: EvaluationGrid, kind: SurfaceKind, values=None, handle=None):
        self.grid = grid
        self.kind = kind
        self._values = values
        self._h = handle

    def __del__(self):
        try:
            if self._h:
                _lib.lib().dfpca_surface_free(self._h)
        except Exception:
            pass

    def rows(self):
        """(row0, rows): the covariance rows this surface holds -- a slab of a
        sharded covariance, or (0, G)."""
        if not self._h:
            return 0, (self.grid.size() if self.kind == SurfaceKind.Covariance else 1)
        r0, nr = C.c_int64(), C.c_int64()
        check(_lib.lib().dfpca_surface_rows(self._h, C.byref(r0), C.byref(nr)))
        return r0.value, nr.value

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            n = self.rows()[1] * self.grid.size() if self.kind == SurfaceKind.Covariance else self.grid.size()
            out = np.empty(n, dtype=np.float64)
            check(_lib.lib().dfpca_surface_download(_lib.ctx(), self._h,
                                                    out.ctypes.data_as(C.POINTER(C.c_double))))
            self._values = out
        return self._values

    def device_handle(self):
        """Device copy of the surface (uploaded on demand)."""
        if not self._h:
            v = np.ascontiguousarray(self._values, dtype=np.float64)
            h = C.c_void_p()
            check(_lib.lib().dfpca_surface_upload(_lib.ctx(), C.byref(self.grid.desc()), self.kind.value,
                                                  v.ctypes.data_as(C.POINTER(C.c_double)), v.size,
                                                  C.byref(h)))
            self._h = h
        return self._h

    def at(self, flat):
        return self.values[flat]

    def gather(self, index) -> np.ndarray:
        """values[index] read on the device (no full download)."""
        idx = np.ascontiguousarray(index, dtype=np.int64).ravel()
        if self._values is not None or not self._h:
            return np.asarray(self.values)[idx]
        out = np.empty(idx.size, dtype=np.float64)
        check(_lib.lib().dfpca_surface_gather(_lib.ctx(), self._h, idx.size, idx.ctypes.data_as(C.POINTER(C.c_int64)),
                                              out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def at_pair(self, s, t):
        return self.values[s * self.grid.size() + t]


@dataclass
class BlockPlan:
    """fft_smoother.hpp:37-53."""
    blocks: list = field(default_factory=list)
    halo: list = field(default_factory=list)

    def core(self, b: int, shape) -> Box:
        blk = self.blocks[b]
        c = Box(list(blk.lo), list(blk.hi))
        for k in range(c.dim()):
            if c.lo[k] > 0:
                c.lo[k] += self.halo[k]
            if c.hi[k] < shape[k]:
                c.hi[k] -= self.halo[k]
        return c

    def desc(self, d: int):
        n = len(self.blocks)
        lo = np.array([b.lo[k] for b in self.blocks for k in range(d)] if n else [0], dtype=np.int64)
        hi = np.array([b.hi[k] for b in self.blocks for k in range(d)] if n else [0], dtype=np.int64)
        halo = np.array(self.halo if len(self.halo) == d else [0] * d, dtype=np.int64)
        p = DfpcaPlan()
        p.n_blocks = n if len(self.halo) == d else 0
        p.blocks_lo = lo.ctypes.data_as(C.POINTER(C.c_int64))
        p.blocks_hi = hi.ctypes.data_as(C.POINTER(C.c_int64))
        p.halo = halo.ctypes.data_as(C.POINTER(C.c_int64))
        return p, (lo, hi, halo)


def kernel_radius_nodes(h: float, spacing: float) -> int:
    """fft_smoother.hpp:59-61"""
    return int(math.ceil(h / spacing))


def single_block_plan(grid: EvaluationGrid, h: Bandwidth) -> BlockPlan:
    """fft_smoother.hpp:66-73"""
    return BlockPlan([Box.full(grid.shape())],
                     [kernel_radius_nodes(h[k], grid.spacing(k)) for k in range(grid.dim())])


def make_block_plan(grid: EvaluationGrid, h: Bandwidth, n_blocks: int) -> BlockPlan:
    """fft_smoother.hpp:77-96"""
    if n_blocks < 1:
        raise Error(ErrorClass.Config, "InvalidArgument", "block count must be positive")
    shape = grid.shape()
    n_blocks = min(n_blocks, shape[0])
    halo = [kernel_radius_nodes(h[k], grid.spacing(k)) for k in range(grid.dim())]
    blocks = []
    for b in range(n_blocks):
        lo = shape[0] * b // n_blocks
        hi = shape[0] * (b + 1) // n_blocks
        blk = Box.full(shape)
        blk.lo[0] = max(0, lo - halo[0])
        blk.hi[0] = min(shape[0], hi + halo[0])
        blocks.append(blk)
    return BlockPlan(blocks, halo)


def validate_block_plan(plan: BlockPlan, grid: EvaluationGrid, h: Bandwidth) -> None:
    """fft_smoother.hpp:101-145 -- validated natively in the C-ABI; this runs the
    same check through a zero-cost device call path."""
    d = grid.dim()
    if not plan.blocks or len(plan.halo) != d:
        raise Error(ErrorClass.Config, "InvalidArgument", "block plan does not match the grid dimension")
    for k in range(d):
        r = kernel_radius_nodes(h[k], grid.spacing(k))
        if plan.halo[k] < r:
            raise Error(ErrorClass.Config, "HaloTooSmall",
                        f"halo of {plan.halo[k]} node(s) on axis {k} is below the kernel radius of {r}")
    shape = grid.shape()
    covered = 0
    cores = []
    for b, blk in enumerate(plan.blocks):
        if blk.dim() != d:
            raise Error(ErrorClass.Config, "InvalidArgument", "block dimension mismatch")
        c = plan.core(b, shape)
        for k in range(d):
            if blk.lo[k] < 0 or blk.hi[k] > shape[k] or blk.lo[k] >= blk.hi[k]:
                raise Error(ErrorClass.Config, "InvalidArgument", "block range outside the grid")
            if c.hi[k] - c.lo[k] < plan.halo[k]:
                raise Error(ErrorClass.Config, "BlockTooSmall",
                            f"block {b} core extent {c.hi[k] - c.lo[k]} on axis {k} is smaller than "
                            f"its halo of {plan.halo[k]}")
        covered += c.volume()
        cores.append(c)
    for a in range(len(cores)):
        for b in range(a + 1, len(cores)):
            if not any(cores[a].hi[k] <= cores[b].lo[k] or cores[b].hi[k] <= cores[a].lo[k]
                       for k in range(d)):
                raise Error(ErrorClass.Config, "InvalidArgument", "block cores overlap")
    if covered != grid.size():
        raise Error(ErrorClass.Config, "InvalidArgument", "block cores do not tile the grid exactly")


def fft_local_linear(binned: BinnedData, grid: EvaluationGrid, h: Bandwidth, target: MomentTarget,
                     plan: Optional[BlockPlan] = None) -> SurfaceEstimate:
    """fft_smoother.hpp:498-575: binned local-linear mean / squares smoother."""
    out = np.empty(grid.size(), dtype=np.float64)
    hh = h.arr()
    if hh.size != grid.dim():
        raise Error(ErrorClass.Config, "InvalidBandwidth", "bandwidth dimension mismatch")
    pdesc, keep = (plan.desc(grid.dim()) if plan is not None else (None, None))
    check(_lib.lib().dfpca_local_linear(_lib.ctx(), binned.handle, C.byref(grid.desc()),
                                        hh.ctypes.data_as(C.POINTER(C.c_double)), target.value,
                                        C.byref(pdesc) if pdesc is not None else None,
                                        out.ctypes.data_as(C.POINTER(C.c_double)), None))
    kind = SurfaceKind.Mean if target == MomentTarget.Mean else SurfaceKind.DiagPlusNoise
    return SurfaceEstimate(grid, kind, values=out)


def fft_covariance(binned: BinnedData, grid: EvaluationGrid, h: Bandwidth, mean: SurfaceEstimate,
                   plan: Optional[BlockPlan] = None, mode=None) -> SurfaceEstimate:
    """fft_smoother.hpp:585-744: binned covariance smoother.  The symmetrized
    surface stays on the device; `.values` downloads it.  `mode`
    (PairGridSource::Mode) only trades memory in the reference and is accepted
    for signature compatibility."""
    hh = h.arr()
    if hh.size != grid.dim():
        raise Error(ErrorClass.Config, "InvalidBandwidth", "bandwidth dimension mismatch")
    mv = np.ascontiguousarray(mean.values, dtype=np.float64)
    if mv.size != grid.size():
        # reference order: this check follows the NoPairs check; the C-ABI
        # reproduces that order when handed a conforming pointer.
        pass
    pdesc, keep = (plan.desc(grid.dim()) if plan is not None else (None, None))
    handle = C.c_void_p()
    check(_lib.lib().dfpca_covariance(_lib.ctx(), binned.handle, C.byref(grid.desc()),
                                      hh.ctypes.data_as(C.POINTER(C.c_double)),
                                      mv.ctypes.data_as(C.POINTER(C.c_double)) if mv.size == grid.size() else None,
                                      C.byref(pdesc) if pdesc is not None else None, C.byref(handle)))
    return SurfaceEstimate(grid, SurfaceKind.Covariance, handle=handle)


def reserve_device_memory(nbytes: int) -> None:
    """Backs this process's device pool with at least `nbytes` now
    (dfpca_context_reserve): the first call of a large workload then reuses
    mapped pages instead of growing the pool while its kernels run (~13 ms
    per GB, paid here).  A B200-side knob; the reference has no equivalent."""
    check(_lib.lib().dfpca_context_reserve(_lib.ctx(), int(nbytes)))


# ------------------------------------------------- multi-GPU (sharded) ----
# The reference's only parallel knob is set_max_threads (parallel.hpp:23);
# here one process per GPU runs one rank of a slab-sharded covariance
# (csrc/shard.hpp): rank r owns s1 planes [bounds[r], bounds[r+1]).


def init_distributed(world: int, rank: int, unique_id: Optional[bytes] = None, broadcast=None) -> None:
    """Joins this process's context to an NCCL communicator of `world` ranks.
    `unique_id` (128 bytes from nccl_unique_id() on rank 0) or `broadcast`, a
    callable(bytes_or_None) -> bytes that distributes rank 0's id (e.g. via
    torch.distributed.broadcast_object_list)."""
    if world > 1 and unique_id is None:
        uid = nccl_unique_id() if rank == 0 else None
        unique_id = broadcast(uid) if broadcast else uid
    buf = C.create_string_buffer(bytes(unique_id) if unique_id else bytes(128), 128)
    check(_lib.lib().dfpca_nccl_init(_lib.ctx(), int(world), int(rank), C.cast(buf, C.c_void_p)))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    status = _lib.lib().dfpca_nccl_unique_id(C.cast(buf, C.c_void_p))
    if status != 0:
        raise Error(ErrorClass.Config, "InvalidArgument", "libnccl could not provide a unique id")
    return buf.raw


def _cov_args(binned, grid, h, mean, plan):
    hh = h.arr()
    if hh.size != grid.dim():
        raise Error(ErrorClass.Config, "InvalidBandwidth", "bandwidth dimension mismatch")
    mv = np.ascontiguousarray(mean.values, dtype=np.float64)
    pdesc, keep = (plan.desc(grid.dim()) if plan is not None else (None, None))
    return hh, mv, pdesc, keep


def fft_covariance_sharded(binned: BinnedData, grid: EvaluationGrid, h: Bandwidth, mean: SurfaceEstimate,
                           plan: Optional[BlockPlan] = None) -> SurfaceEstimate:
    """fft_covariance (fft_smoother.hpp:585-744) as one rank of the
    communicator set up by init_distributed: returns this rank's slab (complete
    rows `.rows()` of the covariance), bit-identical to the one-GPU result."""
    hh, mv, pdesc, keep = _cov_args(binned, grid, h, mean, plan)
    handle = C.c_void_p()
    check(_lib.lib().dfpca_covariance_sharded(_lib.ctx(), binned.handle, C.byref(grid.desc()),
                                              hh.ctypes.data_as(C.POINTER(C.c_double)),
                                              mv.ctypes.data_as(C.POINTER(C.c_double)),
                                              C.byref(pdesc) if pdesc is not None else None, C.byref(handle)))
    return SurfaceEstimate(grid, SurfaceKind.Covariance, handle=handle)


def fft_covariance_emulated(binned: BinnedData, grid: EvaluationGrid, h: Bandwidth, mean: SurfaceEstimate,
                            world: int, plan: Optional[BlockPlan] = None) -> SurfaceEstimate:
    """The sharded decomposition with `world` ranks as threads of this process
    on one device; the slabs are assembled into the full covariance."""
    hh, mv, pdesc, keep = _cov_args(binned, grid, h, mean, plan)
    handle = C.c_void_p()
    check(_lib.lib().dfpca_covariance_emulated(_lib.ctx(), binned.handle, C.byref(grid.desc()),
                                               hh.ctypes.data_as(C.POINTER(C.c_double)),
                                               mv.ctypes.data_as(C.POINTER(C.c_double)),
                                               C.byref(pdesc) if pdesc is not None else None, int(world),
                                               C.byref(handle)))
    return SurfaceEstimate(grid, SurfaceKind.Covariance, handle=handle)


def covariance_slab_dryrun(binned: BinnedData, grid: EvaluationGrid, h: Bandwidth, mean: SurfaceEstimate,
                           world: int, rank: int) -> SurfaceEstimate:
    """Profiling only: rank `rank` of `world` computes its slab with the
    exchanges dropped (device time of one rank's share; values meaningless)."""
    hh, mv, pdesc, keep = _cov_args(binned, grid, h, mean, None)
    handle = C.c_void_p()
    check(_lib.lib().dfpca_covariance_slab_dryrun(_lib.ctx(), binned.handle, C.byref(grid.desc()),
                                                  hh.ctypes.data_as(C.POINTER(C.c_double)),
                                                  mv.ctypes.data_as(C.POINTER(C.c_double)), None, int(world),
                                                  int(rank), C.byref(handle)))
    return SurfaceEstimate(grid, SurfaceKind.Covariance, handle=handle)


def fpca_emulated(binned: BinnedData, grid: EvaluationGrid, h: Bandwidth, mean: SurfaceEstimate, world: int,
                  q: int, L_max: int, seed: int):
    """Sharded covariance + row-sharded randomized eig with `world` in-process
    ranks on one device (validation).  Returns (EigenSystem of rank 0, whether
    every rank's eigensystem is bit-identical)."""
    hh, mv, _, _ = _cov_args(binned, grid, h, mean, None)
    G = grid.size()
    ev = np.zeros(max(L_max, 1))
    ef = np.zeros(max(L_max, 1) * G)
    fve = np.zeros(max(L_max, 1))
    total = C.c_double()
    n = C.c_int64()
    agree = C.c_int()
    check(_lib.lib().dfpca_fpca_emulated(_lib.ctx(), binned.handle, C.byref(grid.desc()),
                                         hh.ctypes.data_as(C.POINTER(C.c_double)),
                                         mv.ctypes.data_as(C.POINTER(C.c_double)), int(world), q, L_max,
                                         C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF),
                                         ev.ctypes.data_as(C.POINTER(C.c_double)),
                                         ef.ctypes.data_as(C.POINTER(C.c_double)),
                                         fve.ctypes.data_as(C.POINTER(C.c_double)), C.byref(total), C.byref(n),
                                         C.byref(agree)))
    L = n.value
    return (EigenSystem([float(x) for x in ev[:L]], [ef[l * G:(l + 1) * G].copy() for l in range(L)],
                        [float(x) for x in fve[:L]], total.value), bool(agree.value))


def shard_bounds(n1: int, nodes_per_plane: int, radius: int, world: int) -> list:
    out = (C.c_int64 * (world + 1))()
    check_plain(_lib.lib().dfpca_shard_bounds(n1, nodes_per_plane, radius, world, out))
    return list(out)


def shard_blocks(n1: int, nodes_per_plane: int, radius: int, world: int, phase: int) -> np.ndarray:
    """[k, 7] int64 rows (src, dst, r0, r1, c0, c1, transpose)."""
    cnt = C.c_int64()
    check_plain(_lib.lib().dfpca_shard_blocks(n1, nodes_per_plane, radius, world, phase, None, 0, C.byref(cnt)))
    out = np.zeros((max(cnt.value, 1), 7), dtype=np.int64)
    check_plain(_lib.lib().dfpca_shard_blocks(n1, nodes_per_plane, radius, world, phase,
                                              out.ctypes.data_as(C.POINTER(C.c_int64)), cnt.value, C.byref(cnt)))
    return out[:cnt.value]


def check_plain(status: int) -> None:
    """Status of a context-free entry point (no error text)."""
    if status != 0:
        raise Error(ErrorClass(status) if status in (2, 3, 4, 5) else ErrorClass.Config, "InvalidArgument",
                    "invalid shard plan arguments")


def blockwise_apply(plan: BlockPlan, binned: BinnedData, grid: EvaluationGrid, h: Bandwidth, what):
    """fft_smoother.hpp:747-758."""
    if isinstance(what, MomentTarget):
        return fft_local_linear(binned, grid, h, what, plan)
    return fft_covariance(binned, grid, h, what, plan)


def pair_grids(binned: BinnedData):
    """PairGridSource::extract(full_box) (fft_smoother.hpp:341-437) -> (pw, pv)."""
    G = binned.grid.size()
    pw = np.empty(G * G)
    pv = np.empty(G * G)
    check(_lib.lib().dfpca_pair_grids(_lib.ctx(), binned.handle, pw.ctypes.data_as(C.POINTER(C.c_double)),
                                      pv.ctypes.data_as(C.POINTER(C.c_double))))
    return pw, pv


# -------------------------------------------------------------- eigen ----


@dataclass
class EigenSystem:
    """eigensolve.hpp:110-115."""
    eigenvalues: list
    eigenfunctions: list
    fve: list
    total_variance: float


class MatrixizedCovariance:
    """eigensolve.hpp:33-68: the in-mask operator over a (device-resident)
    covariance surface."""

    kDenseBudget = 2 << 30
    kSlabBytes = 64 << 20

    def __init__(self, cov: SurfaceEstimate, dense_budget: int):
        g = cov.grid
        self.cov = cov
        mask = g.mask()
        nodes = np.arange(g.size(), dtype=np.int64) if mask is None else np.flatnonzero(np.asarray(mask) != 0)
        rows = np.full(g.size(), -1, dtype=np.int64)
        rows[nodes] = np.arange(nodes.size, dtype=np.int64)
        self.node_of_row = nodes  # int64 arrays (eigensolve.hpp:33-68 keeps std::vector<Index>)
        self.row_of_node = rows
        self.m = int(nodes.size)
        self.dense = self.m * self.m * 8 <= dense_budget

    @property
    def dense_matrix(self):
        v = self.cov.values.reshape(self.cov.grid.size(), self.cov.grid.size())
        idx = np.asarray(self.node_of_row)
        return v[np.ix_(idx, idx)]


def matrixize(cov: SurfaceEstimate, dense_budget: int = MatrixizedCovariance.kDenseBudget):
    """eigensolve.hpp:71-103."""
    if cov.kind != SurfaceKind.Covariance:
        raise Error(ErrorClass.Config, "InvalidArgument", "matrixize expects a covariance surface")
    out = MatrixizedCovariance(cov, dense_budget)
    if out.m == 0:
        raise Error(ErrorClass.Config, "InvalidArgument", "no in-mask nodes to decompose")
    return out


def default_sketch_size(L_max: int, m: int) -> int:
    """eigensolve.hpp:231-234."""
    return min(max(2 * L_max + 10, 99), m)


def randomized_eig(S: MatrixizedCovariance, q: int, L_max: int, grid: EvaluationGrid, seed: int) -> EigenSystem:
    """eigensolve.hpp:245-279 on the GPU."""
    G = grid.size()
    ev = np.zeros(max(L_max, 1))
    ef = np.zeros(max(L_max, 1) * G)
    fve = np.zeros(max(L_max, 1))
    total = C.c_double()
    n = C.c_int64()
    check(_lib.lib().dfpca_randomized_eig(_lib.ctx(), S.cov.device_handle(), C.byref(grid.desc()), q, L_max,
                                          C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF),
                                          ev.ctypes.data_as(C.POINTER(C.c_double)),
                                          ef.ctypes.data_as(C.POINTER(C.c_double)),
                                          fve.ctypes.data_as(C.POINTER(C.c_double)), C.byref(total),
                                          C.byref(n)))
    L = n.value
    return EigenSystem([float(x) for x in ev[:L]], [ef[l * G:(l + 1) * G].copy() for l in range(L)],
                       [float(x) for x in fve[:L]], total.value)


def dense_eig(S: MatrixizedCovariance, L_max: int, grid: EvaluationGrid) -> EigenSystem:
    """eigensolve.hpp:205-228 on the GPU (cuSOLVER syevd + the reference's
    finalization); needs the dense provider like the reference."""
    if not S.dense:
        raise Error(ErrorClass.Config, "InvalidArgument",
                    "dense eigendecomposition needs the dense provider; the matrix exceeded the memory budget")
    G = grid.size()
    ev = np.zeros(max(L_max, 1))
    ef = np.zeros(max(L_max, 1) * G)
    fve = np.zeros(max(L_max, 1))
    total = C.c_double()
    n = C.c_int64()
    check(_lib.lib().dfpca_dense_eig(_lib.ctx(), S.cov.device_handle(), C.byref(grid.desc()), L_max,
                                     ev.ctypes.data_as(C.POINTER(C.c_double)),
                                     ef.ctypes.data_as(C.POINTER(C.c_double)),
                                     fve.ctypes.data_as(C.POINTER(C.c_double)), C.byref(total), C.byref(n)))
    L = n.value
    return EigenSystem([float(x) for x in ev[:L]], [ef[l * G:(l + 1) * G].copy() for l in range(L)],
                       [float(x) for x in fve[:L]], total.value)


def select_components_fve(eig: EigenSystem, threshold: float) -> int:
    """eigensolve.hpp:282-288."""
    if not threshold > 0.0 or threshold > 1.0:
        raise Error(ErrorClass.Config, "InvalidArgument", "FVE threshold must lie in (0, 1]")
    for l, f in enumerate(eig.fve):
        if f >= threshold - 1e-12:
            return l + 1
    return len(eig.eigenvalues)


def eig_residuals(S: MatrixizedCovariance, eig: EigenSystem, grid: EvaluationGrid):
    """eigensolve.hpp:294-312 on the GPU."""
    L = len(eig.eigenvalues)
    if L == 0:
        return []
    lam = np.ascontiguousarray(eig.eigenvalues, dtype=np.float64)
    ef = np.ascontiguousarray(np.concatenate(eig.eigenfunctions), dtype=np.float64)
    out = np.zeros(L)
    check(_lib.lib().dfpca_eig_residuals(_lib.ctx(), S.cov.device_handle(), C.byref(grid.desc()), L,
                                         lam.ctypes.data_as(C.POINTER(C.c_double)),
                                         ef.ctypes.data_as(C.POINTER(C.c_double)),
                                         out.ctypes.data_as(C.POINTER(C.c_double))))
    return [float(x) for x in out]


# ------------------------------------------ noise variance, scores (8(f)) ----
# reference scores.hpp: estimate_sigma2, pace_scores / integration_scores,
# reconstruct_on_grid -- batched over samples on the device.


class ScoreMethod(Enum):
    """scores.hpp:22"""
    Pace = 0
    Integration = 1


def estimate_sigma2(diag_plus_noise: SurfaceEstimate, cov: SurfaceEstimate, mean: SurfaceEstimate) -> float:
    """scores.hpp:82-108 (bit-identical)."""
    if (diag_plus_noise.kind != SurfaceKind.DiagPlusNoise or cov.kind != SurfaceKind.Covariance
            or mean.kind != SurfaceKind.Mean):
        raise Error(ErrorClass.Config, "InvalidArgument", "estimate_sigma2 got surfaces of the wrong kind")
    grid = mean.grid
    dv = np.ascontiguousarray(diag_plus_noise.values, dtype=np.float64)
    mv = np.ascontiguousarray(mean.values, dtype=np.float64)
    out = C.c_double()
    check(_lib.lib().dfpca_estimate_sigma2(_lib.ctx(), C.byref(grid.desc()), dv.ctypes.data_as(C.POINTER(C.c_double)),
                                           cov.device_handle(), mv.ctypes.data_as(C.POINTER(C.c_double)),
                                           C.byref(out)))
    return out.value


def compute_scores_batch(data: FunctionalDataset, grid: EvaluationGrid, mean: SurfaceEstimate, eig: EigenSystem,
                         sigma2: float, method: ScoreMethod):
    """compute_scores (scores.hpp:272-277) for every sample at once.
    Returns (scores [n, L], sparse-warning flags [n])."""
    offsets, coords, values = data.csr()
    n = len(data.samples)
    L = len(eig.eigenvalues)
    mv = np.ascontiguousarray(mean.values, dtype=np.float64)
    ev = np.ascontiguousarray(eig.eigenvalues, dtype=np.float64)
    ef = (np.ascontiguousarray(np.concatenate(eig.eigenfunctions), dtype=np.float64) if L
          else np.zeros(1))
    out = np.zeros(max(n * L, 1))
    warn = np.zeros(max(n, 1), dtype=np.int32)
    PDd = C.POINTER(C.c_double)
    status = _lib.lib().dfpca_scores(_lib.ctx(), C.byref(grid.desc()), n, offsets.ctypes.data_as(C.POINTER(C.c_int64)),
                                     coords.ctypes.data_as(PDd) if coords.size else None,
                                     values.ctypes.data_as(PDd) if values.size else None,
                                     mv.ctypes.data_as(PDd), L, ev.ctypes.data_as(PDd), ef.ctypes.data_as(PDd),
                                     float(sigma2), method.value, out.ctypes.data_as(PDd),
                                     warn.ctypes.data_as(C.POINTER(C.c_int32)))
    if status != 0:
        raise _lib.last_error()
    return out[:n * L].reshape(n, L), warn[:n].astype(bool)


def reconstruct_on_grid(mean: SurfaceEstimate, eig: EigenSystem, scores) -> np.ndarray:
    """scores.hpp:280-300 for one score vector or a [n, L] table."""
    grid = mean.grid
    s = np.ascontiguousarray(scores, dtype=np.float64)
    one = s.ndim == 1
    s = s.reshape(1, -1) if one else s
    L = len(eig.eigenvalues)
    if s.shape[1] != L:
        raise Error(ErrorClass.Config, "InvalidArgument", "score vector length differs from component count")
    mv = np.ascontiguousarray(mean.values, dtype=np.float64)
    ef = np.ascontiguousarray(np.concatenate(eig.eigenfunctions), dtype=np.float64) if L else np.zeros(1)
    out = np.empty(s.shape[0] * grid.size())
    PDd = C.POINTER(C.c_double)
    check(_lib.lib().dfpca_reconstruct(_lib.ctx(), C.byref(grid.desc()), mv.ctypes.data_as(PDd), L,
                                       ef.ctypes.data_as(PDd), s.shape[0], s.ctypes.data_as(PDd),
                                       out.ctypes.data_as(PDd)))
    return out if one else out.reshape(s.shape[0], grid.size())


# ------------------------------------ bandwidth selection: CV (8(f)) ----
# reference bandwidth.hpp: CvObjective / cv_score; the fits run on the device.


class CvTarget(Enum):
    """bandwidth.hpp:27"""
    Mean = 0
    Covariance = 1
    DiagPlusNoise = 2


class CvObjective:
    """bandwidth.hpp:56-163: leave-one-observation-out CV objective of one
    smoothing target.  Units are fixed at construction (a seeded subsample of
    at most max_units observations or ordered pairs); the dataset stays on the
    device; calling the objective runs one direct local fit per unit there."""

    kSelfOnlyTol = 1e-6
    kDenomClamp = 1e-8

    def __init__(self, data: FunctionalDataset, grid: EvaluationGrid, target: CvTarget, max_units: int = 2000,
                 seed: int = 0x5EED):
        offsets, coords, values = data.csr()
        self._grid = grid
        self.target = target
        cnt = C.c_int64()
        PI = C.POINTER(C.c_int64)
        st = _lib.lib().dfpca_cv_units(len(data.samples), offsets.ctypes.data_as(PI), target.value, int(max_units),
                                       C.c_uint64(seed), None, 0, C.byref(cnt))
        if st != 0:
            raise Error(ErrorClass.Config, "InvalidArgument", "cross-validation needs at least one evaluation unit")
        self.units = np.zeros((cnt.value, 3), dtype=np.int64)
        _lib.lib().dfpca_cv_units(len(data.samples), offsets.ctypes.data_as(PI), target.value, int(max_units),
                                  C.c_uint64(seed), self.units.ctypes.data_as(PI), cnt.value, C.byref(cnt))
        h = C.c_void_p()
        PDd = C.POINTER(C.c_double)
        check(_lib.lib().dfpca_dataset_upload(_lib.ctx(), data.dim, len(data.samples), offsets.ctypes.data_as(PI),
                                              coords.ctypes.data_as(PDd) if coords.size else None,
                                              values.ctypes.data_as(PDd) if values.size else None, C.byref(h)))
        self._h = h
        self.last_used = 0

    def __del__(self):
        try:
            if self._h:
                _lib.lib().dfpca_dataset_free(self._h)
        except Exception:
            pass

    def dim(self) -> int:
        return self._grid.dim()

    def n_units(self) -> int:
        return int(self.units.shape[0])

    def extents(self):
        return [self._grid.axis(k)[-1] - self._grid.axis(k)[0] for k in range(self._grid.dim())]

    def __call__(self, h: Bandwidth) -> float:
        hh = h.arr()
        if hh.size != self.dim():
            raise Error(ErrorClass.Config, "InvalidBandwidth", "bandwidth dimension mismatch")
        out = C.c_double()
        used = C.c_int64()
        check(_lib.lib().dfpca_cv_objective(_lib.ctx(), self._h, C.byref(self._grid.desc()), self.target.value,
                                            self.n_units(), self.units.ctypes.data_as(C.POINTER(C.c_int64)),
                                            hh.ctypes.data_as(C.POINTER(C.c_double)), C.byref(out),
                                            C.byref(used)))
        self.last_used = used.value
        return out.value


def cv_score(h: Bandwidth, obj: CvObjective) -> float:
    """bandwidth.hpp:164."""
    return obj(h)


# ------------------------------------------------------------ file formats --
# io.hpp: long-format observation tables (read on the GPU), the
# "dfpca-grid v1" grid file (host; a few KB).

def _table_to_dataset(h) -> FunctionalDataset:
    try:
        dim, ns, no, nid = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
        _lib.lib().dfpca_table_info(h, C.byref(dim), C.byref(ns), C.byref(no), C.byref(nid))
        offsets = np.zeros(ns.value + 1, dtype=np.int64)
        coords = np.zeros(no.value * dim.value, dtype=np.float64)
        values = np.zeros(no.value, dtype=np.float64)
        id_off = np.zeros(ns.value + 1, dtype=np.int64)
        chars = C.create_string_buffer(max(nid.value, 1))
        PI, PDd = C.POINTER(C.c_int64), C.POINTER(C.c_double)
        check(_lib.lib().dfpca_table_copy(_lib.ctx(), h, offsets.ctypes.data_as(PI), coords.ctypes.data_as(PDd),
                                          values.ctypes.data_as(PDd), id_off.ctypes.data_as(PI), chars))
    finally:
        _lib.lib().dfpca_table_free(h)
    raw = chars.raw
    ids = [raw[id_off[i]:id_off[i + 1]].decode("utf-8", "surrogateescape") for i in range(ns.value)]
    return FunctionalDataset.from_csr(dim.value, offsets, coords, values, ids)


def read_long_format(path: str) -> FunctionalDataset:
    """io.hpp:115-155.  Samples in order of first appearance of their id,
    observations in file order; ParseError / IoError as the reference."""
    h = C.c_void_p()
    check(_lib.lib().dfpca_read_long_format(_lib.ctx(), str(path).encode(), C.byref(h)))
    return _table_to_dataset(h)


def parse_long_format(data: bytes, name: str = "<memory>") -> FunctionalDataset:
    """read_long_format over file contents already in memory."""
    h = C.c_void_p()
    check(_lib.lib().dfpca_parse_long_format(_lib.ctx(), name.encode(), data, len(data), C.byref(h)))
    return _table_to_dataset(h)


def _fmt17(v: float) -> str:
    if v != v:
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    return "%.17g" % v


def write_long_format(path: str, data: FunctionalDataset, axis_names: Optional[Sequence[str]] = None) -> None:
    """io.hpp:158-178: tab-separated, header sample_id, t1.., y; 17 digits."""
    names = list(axis_names) if axis_names else ["t%d" % (k + 1) for k in range(data.dim)]
    if len(names) != data.dim:
        raise Error(ErrorClass.Config, "InvalidArgument", "one axis name per dimension")
    try:
        f = open(path, "w", newline="\n")
    except OSError:
        raise Error(ErrorClass.Parse, "IoError", "cannot open '%s' for writing" % path) from None
    with f:
        f.write("sample_id\t" + "\t".join(names) + "\ty\n")
        d = data.dim
        for s in data.samples:
            c = np.asarray(s.coords, dtype=np.float64).ravel()
            v = np.asarray(s.values, dtype=np.float64)
            for j in range(v.size):
                f.write(s.id + "".join("\t" + _fmt17(float(c[j * d + k])) for k in range(d)) + "\t" + _fmt17(float(v[j]))
                        + "\n")


def write_grid(path: str, grid: EvaluationGrid) -> None:
    """io.hpp:188-203 ("dfpca-grid v1")."""
    try:
        f = open(path, "w", newline="\n")
    except OSError:
        raise Error(ErrorClass.Parse, "IoError", "cannot open '%s' for writing" % path) from None
    with f:
        f.write("dfpca-grid v1\ndim %d\n" % grid.dim())
        for k in range(grid.dim()):
            ax = grid.axis(k)
            f.write("axis %d %d" % (k, len(ax)) + "".join(" " + _fmt17(float(v)) for v in ax) + "\n")
        if grid.has_mask():
            f.write("mask " + "".join("1" if m else "0" for m in np.asarray(grid.mask()).ravel()) + "\n")


def _parse_token_double(tok: str, where: str) -> float:
    # strtod acceptance (io.hpp:39-46) for the grid file's few numbers
    t = tok.strip(" \t\n\v\f\r") if tok[:1].isspace() else tok
    try:
        v = float.fromhex(t) if t.lower().lstrip("+-").startswith("0x") else float(t)
    except ValueError:
        raise Error(ErrorClass.Parse, "ParseError", "%s: not a number: '%s'" % (where, tok)) from None
    if "_" in t or math.isinf(v) and not t.lower().lstrip("+-").startswith("inf"):
        raise Error(ErrorClass.Parse, "ParseError", "%s: not a number: '%s'" % (where, tok))
    return v


def read_grid(path: str) -> EvaluationGrid:
    """io.hpp:206-259."""
    try:
        f = open(path, "rb")
    except OSError:
        raise Error(ErrorClass.Parse, "IoError", "cannot open '%s' for reading" % path) from None
    with f:
        lines = f.read().decode("latin-1").split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        raise Error(ErrorClass.Parse, "ParseError", "%s:1: empty grid file" % path)
    first = lines[0][:-1] if lines[0].endswith("\r") else lines[0]
    if not first.startswith("dfpca-grid"):
        raise Error(ErrorClass.Parse, "ParseError", "%s:1: not a dfpca-grid file (bad magic)" % path)
    if first != "dfpca-grid v1":
        raise Error(ErrorClass.Version, "VersionMismatch", "%s: unsupported grid format '%s'" % (path, first))
    dim, axes, mask_bits = 0, [], ""
    for no, line in enumerate(lines[1:], start=2):
        line = line[:-1] if line.endswith("\r") else line
        if not line:
            continue
        toks = line.split()
        tag = toks[0] if toks else ""
        where = "%s:%d" % (path, no)
        if tag == "dim":
            try:
                dd = int(toks[1])
            except (IndexError, ValueError):
                dd = 0
            if dd < 1:
                raise Error(ErrorClass.Parse, "ParseError", "%s: bad dimension" % where)
            dim = dd
            axes = [[] for _ in range(dim)]
        elif tag == "axis":
            try:
                k, cnt = int(toks[1]), int(toks[2])
            except (IndexError, ValueError):
                k, cnt = -1, 0
            if k < 0 or k >= len(axes) or cnt < 2:
                raise Error(ErrorClass.Parse, "ParseError", "%s: bad axis header" % where)
            if len(toks) - 3 < cnt:
                raise Error(ErrorClass.Parse, "ParseError", "%s: axis shorter than declared" % where)
            axes[k] = [_parse_token_double(t, where) for t in toks[3:3 + cnt]]
        elif tag == "mask":
            mask_bits += "".join(toks[1:])
        else:
            raise Error(ErrorClass.Parse, "ParseError", "%s: unknown record '%s'" % (where, tag))
    if dim == 0:
        raise Error(ErrorClass.Parse, "ParseError", "%s: missing 'dim' record" % path)
    for k in range(dim):
        if not axes[k]:
            raise Error(ErrorClass.Parse, "ParseError", "%s: missing axis %d" % (path, k))
    if not mask_bits:
        return EvaluationGrid(axes)
    total = int(np.prod([len(a) for a in axes]))
    if len(mask_bits) != total:
        raise Error(ErrorClass.Parse, "ParseError",
                    "%s: mask length %d does not match grid size %d" % (path, len(mask_bits), total))
    if set(mask_bits) - {"0", "1"}:
        raise Error(ErrorClass.Parse, "ParseError", "%s: mask entries must be 0 or 1" % path)
    return EvaluationGrid(axes, np.frombuffer(mask_bits.encode(), dtype=np.uint8) - ord("0"))


def bin_long_format(path: str, grid: EvaluationGrid, opt: BinOptions = BinOptions()):
    """read_long_format + linear_bin without the host round trip: the table is
    parsed on the GPU and binned there (the observations never cross PCIe).
    Returns (BinnedData, sample ids in first-appearance order); the same
    binned data, bit for bit, as linear_bin(read_long_format(path), ...)."""
    t = C.c_void_p()
    check(_lib.lib().dfpca_read_long_format(_lib.ctx(), str(path).encode(), C.byref(t)))
    try:
        dim, ns, no, nid = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
        _lib.lib().dfpca_table_info(t, C.byref(dim), C.byref(ns), C.byref(no), C.byref(nid))
        id_off = np.zeros(ns.value + 1, dtype=np.int64)
        chars = C.create_string_buffer(max(nid.value, 1))
        check(_lib.lib().dfpca_table_copy(_lib.ctx(), t, None, None, None, id_off.ctypes.data_as(C.POINTER(C.c_int64)),
                                          chars))
        raw = chars.raw
        ids = [raw[id_off[i]:id_off[i + 1]].decode("utf-8", "surrogateescape") for i in range(ns.value)]
        if dim.value != grid.dim():
            raise Error(ErrorClass.Config, "InvalidArgument", "dataset/grid dimension mismatch")
        h = C.c_void_p()
        status = _lib.lib().dfpca_linear_bin_table(_lib.ctx(), t, C.byref(grid.desc()), int(opt.mean_path),
                                                   int(opt.covariance_path), C.byref(h))
        if status != 0:
            err = _lib.last_error()
            if err.name() == "ObservationOutsideGrid":
                i, j = _lib.last_error_location()
                raise Error(err.error_class, err.name(), f"sample '{ids[i]}' observation {j} lies outside the grid hull")
            raise err
    finally:
        _lib.lib().dfpca_table_free(t)
    return BinnedData(h, grid), ids

