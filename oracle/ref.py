"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_ref/libdfpca_ref.so,
the reference implementation (proj/include/dfpca, compiled unchanged by
oracle/Makefile).  Used by tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / reference arm as the checker; never by the product.

Inputs/outputs are plain numpy arrays so the same fixtures feed both the
GPU library and this oracle.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libdfpca_ref.so"

PD = C.POINTER(C.c_double)
PI = C.POINTER(C.c_int64)
PU8 = C.POINTER(C.c_uint8)
VP = C.c_void_p

_SIG = {
    "ref_last_error": (C.c_char_p, [C.POINTER(C.c_int)]),
    "ref_set_threads": (None, [C.c_int]),
    "ref_linear_bin": (C.c_int, [C.c_int, PI, PD, PU8, C.c_int64, PI, PD, PD, C.c_int, C.c_int, C.POINTER(VP)]),
    "ref_binned_from_host": (C.c_int, [C.c_int, PI, PD, PU8, C.c_int64, PI, C.c_int, PD, PD, PD, C.c_int,
                                       C.c_int64, PI, PD, PD, PD, PD, PD, C.POINTER(VP)]),
    "ref_binned_info": (C.c_int, [VP, PI, PI, PI, PI]),
    "ref_binned_download": (C.c_int, [VP, PD, PD, PD, PI, PD, PD, PD, PD, PD, PI]),
    "ref_binned_free": (None, [VP]),
    "ref_local_linear": (C.c_int, [VP, C.c_int, PI, PD, PU8, PD, C.c_int, C.c_int64, PD]),
    "ref_covariance": (C.c_int, [VP, C.c_int, PI, PD, PU8, PD, PD, C.c_int64, C.c_int, PD]),
    "ref_pair_grids": (C.c_int, [VP, C.c_int, PD, PD]),
    "ref_randomized_eig": (C.c_int, [C.c_int, PI, PD, PU8, PD, C.c_int64, C.c_int64, C.c_uint64, PD, PD, PD, PD, PI]),
    "ref_dense_eig": (C.c_int, [C.c_int, PI, PD, PU8, PD, C.c_int64, PD, PD, PD, PD, PI]),
    "ref_eig_residuals": (C.c_int, [C.c_int, PI, PD, PU8, PD, C.c_int64, PD, PD, PD]),
    "ref_estimate_mean": (C.c_int, [C.c_int, PI, PD, PU8, C.c_int64, PI, PD, PD, PD, C.c_int, PD]),
    "ref_estimate_covariance": (C.c_int, [C.c_int, PI, PD, PU8, C.c_int64, PI, PD, PD, PD, PD, PD]),
    "ref_estimate_sigma2": (C.c_int, [C.c_int, PI, PD, PU8, PD, PD, PD, PD]),
    "ref_scores": (C.c_int, [C.c_int, PI, PD, PU8, C.c_int64, PI, PD, PD, PD, C.c_int64, PD, PD, C.c_double,
                             C.c_int, PD, C.POINTER(C.c_int)]),
    "ref_reconstruct": (C.c_int, [C.c_int, PI, PD, PU8, PD, C.c_int64, PD, PD, PD, PD]),
    "ref_cv_score": (C.c_int, [C.c_int, PI, PD, PU8, C.c_int64, PI, PD, PD, C.c_int, C.c_int64, C.c_uint64, PD, PD,
                               PI]),
    "ref_read_long_format": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "ref_table_info": (None, [C.c_void_p, C.POINTER(C.c_int), PI, PI, PI]),
    "ref_table_copy": (None, [C.c_void_p, PI, PD, PD, PI, C.c_char_p]),
    "ref_table_free": (None, [C.c_void_p]),
    "ref_write_long_format": (C.c_int, [C.c_char_p, C.c_int, C.c_int64, PI, PD, PD, PI, C.c_char_p]),
    "ref_write_grid": (C.c_int, [C.c_char_p, C.c_int, PI, PD, PU8]),
    "ref_read_grid": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), PI, PD, PU8, C.POINTER(C.c_int)]),
    "ref_simulate": (C.c_int, [C.c_int, C.c_int, PI, PD, PU8, C.c_int64, C.c_int64, C.c_uint64, PI, PD, PD]),
    "ref_covariance_block": (C.c_int, [VP, C.c_int, PI, PD, PU8, PD, PD, PI, PI, PI, PI, PD]),
}

_lib = None


class RefError(RuntimeError):
    def __init__(self, cls: int, what: str):
        super().__init__(what)
        self.cls = cls
        self._name = what.split(":", 1)[0]

    def name(self) -> str:
        return self._name


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise ImportError(f"oracle not built: {LIB} (run make -C oracle)")
        l = C.CDLL(str(LIB))
        for n, (res, args) in _SIG.items():
            f = getattr(l, n)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def set_threads(n: int):
    lib().ref_set_threads(int(n))


def _chk(st):
    if st != 0:
        cls = C.c_int()
        msg = lib().ref_last_error(C.byref(cls)).decode()
        raise RefError(cls.value, msg)


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, (a.ctypes.data_as(PD) if a.size else None)


class _GridArgs:
    """(dim, shape*, axes*, mask*) for a grid given as (axes list, mask)."""

    def __init__(self, axes, mask=None):
        self.dim = len(axes)
        self.shape = np.array([len(a) for a in axes], dtype=np.int64)
        self.axes = np.ascontiguousarray(np.concatenate([np.asarray(a, dtype=np.float64) for a in axes]))
        self.mask = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        self.G = int(np.prod(self.shape))

    def args(self):
        return (self.dim, self.shape.ctypes.data_as(PI), self.axes.ctypes.data_as(PD),
                self.mask.ctypes.data_as(PU8) if self.mask is not None else None)


def grid_args(grid) -> _GridArgs:
    """Accepts the product's EvaluationGrid or (axes, mask)."""
    if hasattr(grid, "axes") and callable(grid.axes):
        return _GridArgs(grid.axes(), grid.mask())
    axes, mask = grid
    return _GridArgs(axes, mask)


@dataclass
class RefBinned:
    handle: int
    G: int
    codes: int
    n_samples: int
    n_pair: int

    def __del__(self):
        try:
            lib().ref_binned_free(self.handle)
        except Exception:
            pass

    def fields(self) -> dict:
        G, npair, codes, n = self.G, self.n_pair, self.codes, self.n_samples
        out = dict(mass=np.zeros(G), wvalue=np.zeros(G), wsquare=np.zeros(G),
                   sample_index=np.zeros(npair, dtype=np.int64), pair_weight=np.zeros(npair),
                   ps_mass=np.zeros(npair * G), ps_value=np.zeros(npair * G),
                   diag_mass=np.zeros(G * codes), diag_value=np.zeros(G * codes),
                   sample_sizes=np.zeros(n, dtype=np.int64))
        P = lambda a: a.ctypes.data_as(PD) if a.size else None
        Q = lambda a: a.ctypes.data_as(PI) if a.size else None
        lib().ref_binned_download(self.handle, P(out["mass"]), P(out["wvalue"]), P(out["wsquare"]),
                                  Q(out["sample_index"]), P(out["pair_weight"]), P(out["ps_mass"]),
                                  P(out["ps_value"]), P(out["diag_mass"]), P(out["diag_value"]),
                                  Q(out["sample_sizes"]))
        return out


def _wrap(h) -> RefBinned:
    n, npair, G, codes = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    lib().ref_binned_info(h, C.byref(n), C.byref(npair), C.byref(G), C.byref(codes))
    return RefBinned(h, G.value, codes.value, n.value, npair.value)


def linear_bin(grid, offsets, coords, values, mean_path=True, covariance_path=False) -> RefBinned:
    ga = grid_args(grid)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    c, cp = _d(coords)
    v, vp = _d(values)
    h = VP()
    _chk(lib().ref_linear_bin(*ga.args(), off.size - 1, off.ctypes.data_as(PI), cp, vp, int(mean_path),
                              int(covariance_path), C.byref(h)))
    return _wrap(h)


def binned_from_host(grid, sample_sizes, mass=None, wvalue=None, wsquare=None, per_sample=(),
                     diag_mass=None, diag_value=None, has_mean=True, has_cov=False) -> RefBinned:
    ga = grid_args(grid)
    G = ga.G
    codes = 3 ** ga.dim
    z = lambda a, n: np.ascontiguousarray(np.zeros(n) if a is None else a, dtype=np.float64)
    m, wv, ws = z(mass, G), z(wvalue, G), z(wsquare, G)
    dm, dv = z(diag_mass, G * codes), z(diag_value, G * codes)
    sizes = np.ascontiguousarray(sample_sizes, dtype=np.int64)
    si = np.array([p[0] for p in per_sample], dtype=np.int64)
    pw = np.array([p[1] for p in per_sample], dtype=np.float64)
    psm = np.ascontiguousarray(np.concatenate([p[2] for p in per_sample]) if per_sample else np.zeros(0))
    psv = np.ascontiguousarray(np.concatenate([p[3] for p in per_sample]) if per_sample else np.zeros(0))
    P = lambda a: a.ctypes.data_as(PD) if a.size else None
    Q = lambda a: a.ctypes.data_as(PI) if a.size else None
    h = VP()
    _chk(lib().ref_binned_from_host(*ga.args(), sizes.size, Q(sizes), int(has_mean), P(m), P(wv), P(ws),
                                    int(has_cov), si.size, Q(si), P(pw), P(psm), P(psv), P(dm), P(dv),
                                    C.byref(h)))
    return _wrap(h)


def fft_local_linear(binned: RefBinned, grid, h, target: int = 0, n_blocks: int = 0) -> np.ndarray:
    ga = grid_args(grid)
    hh, hp = _d(h)
    out = np.empty(ga.G)
    _chk(lib().ref_local_linear(binned.handle, *ga.args(), hp, int(target), int(n_blocks), out.ctypes.data_as(PD)))
    return out


def fft_covariance(binned: RefBinned, grid, h, mean, n_blocks: int = 0, mode: int = 0) -> np.ndarray:
    ga = grid_args(grid)
    hh, hp = _d(h)
    mu, mp = _d(mean)
    out = np.empty(ga.G * ga.G)
    _chk(lib().ref_covariance(binned.handle, *ga.args(), hp, mp, int(n_blocks), int(mode), out.ctypes.data_as(PD)))
    return out


def pair_grids(binned: RefBinned, mode: int = 1):
    G = binned.G
    pw = np.empty(G * G)
    pv = np.empty(G * G)
    _chk(lib().ref_pair_grids(binned.handle, int(mode), pw.ctypes.data_as(PD), pv.ctypes.data_as(PD)))
    return pw, pv


def _eig(fn, grid, cov, L_max, *extra):
    ga = grid_args(grid)
    cv, cp = _d(cov)
    ev = np.zeros(max(L_max, 1))
    ef = np.zeros(max(L_max, 1) * ga.G)
    fve = np.zeros(max(L_max, 1))
    tot = C.c_double()
    n = C.c_int64()
    _chk(fn(*ga.args(), cp, *extra, ev.ctypes.data_as(PD), ef.ctypes.data_as(PD), fve.ctypes.data_as(PD),
            C.byref(tot), C.byref(n)))
    L = n.value
    return dict(eigenvalues=ev[:L].copy(), eigenfunctions=ef[:L * ga.G].reshape(L, ga.G).copy(),
                fve=fve[:L].copy(), total_variance=tot.value)


def randomized_eig(grid, cov, q: int, L_max: int, seed: int):
    return _eig(lib().ref_randomized_eig, grid, cov, L_max, int(q), int(L_max), C.c_uint64(seed))


def dense_eig(grid, cov, L_max: int):
    return _eig(lib().ref_dense_eig, grid, cov, L_max, int(L_max))


def eig_residuals(grid, cov, evals, efuncs):
    ga = grid_args(grid)
    cv, cp = _d(cov)
    ev, evp = _d(evals)
    ef, efp = _d(np.ravel(efuncs))
    out = np.zeros(len(ev))
    _chk(lib().ref_eig_residuals(*ga.args(), cp, len(ev), evp, efp, out.ctypes.data_as(PD)))
    return out


def estimate_mean(grid, offsets, coords, values, h, squares=False) -> np.ndarray:
    ga = grid_args(grid)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    c, cp = _d(coords)
    v, vp = _d(values)
    hh, hp = _d(h)
    out = np.empty(ga.G)
    _chk(lib().ref_estimate_mean(*ga.args(), off.size - 1, off.ctypes.data_as(PI), cp, vp, hp, int(squares),
                                 out.ctypes.data_as(PD)))
    return out


def estimate_covariance(grid, offsets, coords, values, h, mean) -> np.ndarray:
    ga = grid_args(grid)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    c, cp = _d(coords)
    v, vp = _d(values)
    hh, hp = _d(h)
    mu, mp = _d(mean)
    out = np.empty(ga.G * ga.G)
    _chk(lib().ref_estimate_covariance(*ga.args(), off.size - 1, off.ctypes.data_as(PI), cp, vp, hp, mp,
                                       out.ctypes.data_as(PD)))
    return out


# ---- scores.hpp ------------------------------------------

def estimate_sigma2(grid, diag, cov, mean) -> float:
    """scores.hpp:82-108."""
    ga = grid_args(grid)
    a, ap = _d(diag)
    b, bp = _d(cov)
    c, cp = _d(mean)
    out = C.c_double()
    _chk(lib().ref_estimate_sigma2(*ga.args(), ap, bp, cp, C.byref(out)))
    return out.value


def scores(grid, offsets, coords, values, mean, evals, efuncs, sigma2, method: int):
    """compute_scores (scores.hpp:272-277) for every sample; method 0 = pace,
    1 = integration.  Returns (scores [n, L], sparse-warning flags [n])."""
    ga = grid_args(grid)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    n = off.size - 1
    c, cp = _d(coords)
    v, vp = _d(values)
    mu, mp = _d(mean)
    ev, evp = _d(evals)
    ef, efp = _d(np.ravel(efuncs))
    L = ev.size
    out = np.zeros(max(n * L, 1))
    sp = np.zeros(max(n, 1), dtype=np.int32)
    _chk(lib().ref_scores(*ga.args(), n, off.ctypes.data_as(PI), cp, vp, mp, L, evp, efp, float(sigma2),
                          int(method), out.ctypes.data_as(PD), sp.ctypes.data_as(C.POINTER(C.c_int))))
    return out[:n * L].reshape(n, L), sp[:n].astype(bool)


def reconstruct_on_grid(grid, mean, evals, efuncs, sc) -> np.ndarray:
    """scores.hpp:280-300."""
    ga = grid_args(grid)
    mu, mp = _d(mean)
    ev, evp = _d(evals)
    ef, efp = _d(np.ravel(efuncs))
    s, spp = _d(sc)
    out = np.empty(ga.G)
    _chk(lib().ref_reconstruct(*ga.args(), mp, ev.size, evp, efp, spp, out.ctypes.data_as(PD)))
    return out


def cv_score(grid, offsets, coords, values, target: int, h, max_units: int = 2000, seed: int = 0x5EED):
    """CvObjective(data, grid, target, {max_units, seed}) evaluated at h
    (bandwidth.hpp:56-163); target 0 mean, 1 covariance, 2 diag.
    Returns (score, n_units)."""
    ga = grid_args(grid)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    c, cp = _d(coords)
    v, vp = _d(values)
    hh, hp = _d(h)
    out = C.c_double()
    nu = C.c_int64()
    _chk(lib().ref_cv_score(*ga.args(), off.size - 1, off.ctypes.data_as(PI), cp, vp, int(target), int(max_units),
                            C.c_uint64(seed), hp, C.byref(out), C.byref(nu)))
    return out.value, nu.value


def read_long_format(path):
    """io.hpp:115-155 -> (dim, offsets, coords, values, ids)."""
    h = C.c_void_p()
    _chk(lib().ref_read_long_format(str(path).encode(), C.byref(h)))
    try:
        dim, ns, no, nid = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
        lib().ref_table_info(h, C.byref(dim), C.byref(ns), C.byref(no), C.byref(nid))
        off = np.zeros(ns.value + 1, dtype=np.int64)
        coords = np.zeros(no.value * dim.value)
        values = np.zeros(no.value)
        id_off = np.zeros(ns.value + 1, dtype=np.int64)
        chars = C.create_string_buffer(max(nid.value, 1))
        lib().ref_table_copy(h, off.ctypes.data_as(PI), coords.ctypes.data_as(PD), values.ctypes.data_as(PD),
                             id_off.ctypes.data_as(PI), chars)
    finally:
        lib().ref_table_free(h)
    raw = chars.raw
    ids = [raw[id_off[i]:id_off[i + 1]] for i in range(ns.value)]
    return dim.value, off, coords, values, ids


def write_long_format(path, dim, offsets, coords, values, ids):
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    blob = b"".join(i if isinstance(i, bytes) else i.encode() for i in ids)
    id_off = np.zeros(len(ids) + 1, dtype=np.int64)
    np.cumsum([len(i if isinstance(i, bytes) else i.encode()) for i in ids], out=id_off[1:])
    c, pc = _d(coords)
    v, pv = _d(values)
    _chk(lib().ref_write_long_format(str(path).encode(), int(dim), len(ids), off.ctypes.data_as(PI), pc, pv,
                                     id_off.ctypes.data_as(PI), blob))


def write_grid(path, grid):
    g = _GridArgs(*grid)
    _chk(lib().ref_write_grid(str(path).encode(), *g.args()))


def read_grid(path):
    """-> (axes list, mask or None)"""
    dim, has_mask = C.c_int(), C.c_int()
    shape = np.zeros(16, dtype=np.int64)
    _chk(lib().ref_read_grid(str(path).encode(), C.byref(dim), shape.ctypes.data_as(PI), None, None,
                             C.byref(has_mask)))
    n = shape[:dim.value]
    axes = np.zeros(int(n.sum()))
    mask = np.zeros(int(np.prod(n)), dtype=np.uint8)
    _chk(lib().ref_read_grid(str(path).encode(), C.byref(dim), shape.ctypes.data_as(PI), axes.ctypes.data_as(PD),
                             mask.ctypes.data_as(PU8), C.byref(has_mask)))
    out, o = [], 0
    for k in n:
        out.append(axes[o:o + k])
        o += k
    return out, (mask if has_mask.value else None)



def simulate(kind: int, grid, n: int, points_per_sample: int = 0, seed: int = 20260815):
    """The reference's generate() (simulate.hpp:163-245) for the models of
    ref_simulate: (offsets, coords, values)."""
    g = grid_args(grid)
    off = np.zeros(n + 1, dtype=np.int64)
    _chk(lib().ref_simulate(kind, *g.args(), n, points_per_sample, seed, off.ctypes.data_as(PI), None, None))
    N = int(off[-1])
    coords = np.empty(N * g.dim)
    values = np.empty(N)
    _chk(lib().ref_simulate(kind, *g.args(), n, points_per_sample, seed, off.ctypes.data_as(PI),
                            coords.ctypes.data_as(PD), values.ctypes.data_as(PD)))
    return off, coords, values


def covariance_block(binned: RefBinned, grid, h, mean, s_box, t_box) -> np.ndarray:
    """The reference's centered, symmetrized covariance restricted to the
    node boxes s_box x t_box (each ([lo...], [hi...]) per axis, hi exclusive):
    fft_covariance's block-pair loop body run for that pair (ref_capi.cpp)."""
    g = grid_args(grid)
    hh, hp = _d(h)
    m, mp = _d(mean)
    sl, sh, tl, th = (np.ascontiguousarray(x, dtype=np.int64) for x in (*s_box, *t_box))
    ns = int(np.prod(sh - sl))
    nt = int(np.prod(th - tl))
    out = np.empty(ns * nt)
    _chk(lib().ref_covariance_block(binned.handle, *g.args(), hp, mp, sl.ctypes.data_as(PI), sh.ctypes.data_as(PI),
                                    tl.ctypes.data_as(PI), th.ctypes.data_as(PI), out.ctypes.data_as(PD)))
    return out.reshape(ns, nt)
