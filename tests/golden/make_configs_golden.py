#!/usr/bin/env python3
"""Golden fixtures for BASELINE.json's configs, made by the REFERENCE itself
(oracle/_ref/libdfpca_ref.so) on inputs drawn by the reference's own
generator (simulate.hpp, through oracle/ref.simulate).  Run in the build
container (minutes; 8 host threads):

    make -C oracle && python tests/golden/make_configs_golden.py [cfg ...]

The inputs are NOT stored (cfg 3 alone is 197 MB): the GPU tests redraw them
with the library's restatement of the generator, which tests/test_simulate.py
pins bit for bit to the reference's generate(); each fixture stores a digest
of its inputs so a drift is caught before any comparison.  Outputs too large
to commit are stored as fixed samples (indices + values):

  cfg1  Sim I, n=200 x 100 points, 100 nodes, h=0.25: mean, squares, full
        covariance, randomized (q=99) and dense eigensystems, L=3.
  cfg2  images n=500, 32^2, h=0.1: mean, 65 536 sampled covariance entries,
        randomized eigensystem q=99, L=20.
  cfg3  images n=2000, 64^2, h=0.1: mean, squares, 8 full covariance rows +
        32 768 sampled entries, randomized eigensystem (M=4096, q=99, L=20)
        and the dense eigenvalues.
  cfg3w the same data at h=0.3 (R=20: the reference's FFT path, conv.hpp:73).
  cfg4  sparse masked n=2000, 64^2, h=0.15 (ladder): mean, sampled in-mask
        entries, randomized eigensystem q=99, L=20.
  cfg5  Sim II d=3, 32^3, n=100, h=0.1 (R=4): mean, and 48 full 32x32 blocks of
        the 1.07e9-point covariance (ref_capi.cpp:ref_covariance_block, the
        reference's block-pair loop body on 2x4x4 node boxes at corners, edges
        and the interior).
"""
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref as R  # noqa: E402
from paper_1510_04439_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent
SEED = 20260815
KIND = {1: synth.SIM_SIM1, 2: synth.SIM_IMAGES2, 3: synth.SIM_IMAGES2, 4: synth.SIM_SPARSE2, 5: synth.SIM_SIM2}


def digest(sd) -> str:
    h = hashlib.sha256()
    for a in (sd.offsets, sd.coords, sd.values):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def draw(cfg, n=None, h=None):
    """The config's inputs from the reference's generator (oracle side), with
    the grid of synth.config."""
    sd = synth.config(cfg, n=n, h=h)
    off, c, v = R.simulate(KIND[cfg], (sd.axes, sd.mask), sd.n_samples, 100 if cfg == 1 else 0, SEED)
    assert np.array_equal(off, sd.offsets) and np.array_equal(c, sd.coords) and np.array_equal(v, sd.values)
    sd.offsets, sd.coords, sd.values = off, c, v
    return sd


def header(cfg, sd, n):
    axes = np.concatenate([np.asarray(a, dtype=np.float64) for a in sd.axes])
    return dict(cfg=np.int64(cfg), n=np.int64(n), seed=np.uint64(SEED), h=np.asarray(sd.h), axes=axes,
                shape=np.array([len(a) for a in sd.axes], dtype=np.int64),
                mask=np.asarray(sd.mask if sd.mask is not None else [], dtype=np.uint8),
                input_digest=np.bytes_(digest(sd)))


def eig_fields(prefix, e):
    return {f"{prefix}_values": e["eigenvalues"], f"{prefix}_functions": e["eigenfunctions"],
            f"{prefix}_fve": e["fve"], f"{prefix}_total": np.float64(e["total_variance"])}


def sample_entries(cov, G, mask, count, rows, rng):
    C = cov.reshape(G, G)
    inside = np.ones(G, bool) if mask is None else np.asarray(mask, bool)
    nodes = np.flatnonzero(inside)
    a = rng.choice(nodes, count)
    b = rng.choice(nodes, count)
    idx = a.astype(np.int64) * G + b
    out = dict(cov_idx=idx, cov_val=cov[idx])
    if rows:
        r = np.asarray(rows, dtype=np.int64)
        out.update(cov_rows=r, cov_row_vals=C[r].copy())
    return out


def smooth_all(sd, with_squares=True):
    grid = (sd.axes, sd.mask)
    t0 = time.time()
    r = R.linear_bin(grid, sd.offsets, sd.coords, sd.values, True, True)
    mean = R.fft_local_linear(r, grid, sd.h, 0)
    sq = R.fft_local_linear(r, grid, sd.h, 1) if with_squares else None
    t1 = time.time()
    cov = R.fft_covariance(r, grid, sd.h, mean)
    print(f"  bin+mean {t1 - t0:.1f}s covariance {time.time() - t1:.1f}s", flush=True)
    return r, mean, sq, cov


def cfg1():
    sd = draw(1)
    r, mean, sq, cov = smooth_all(sd)
    grid = (sd.axes, None)
    out = header(1, sd, 200)
    out.update(mean=mean, squares=sq, cov=cov)
    out.update(eig_fields("reig", R.randomized_eig(grid, cov, 99, 3, SEED)))
    out.update(eig_fields("deig", R.dense_eig(grid, cov, 3)))
    return out


def cfg2():
    sd = draw(2)
    r, mean, sq, cov = smooth_all(sd, with_squares=False)
    out = header(2, sd, 500)
    out.update(mean=mean)
    out.update(sample_entries(cov, 1024, None, 65536, [0, 31, 527, 1023], np.random.default_rng(2)))
    out.update(eig_fields("reig", R.randomized_eig((sd.axes, None), cov, 99, 20, SEED)))
    return out


def cfg3(h=0.1, tag=3):
    sd = draw(3, h=h)
    r, mean, sq, cov = smooth_all(sd)
    out = header(3, sd, 2000)
    out.update(mean=mean, squares=sq)
    out.update(sample_entries(cov, 4096, None, 32768, [0, 63, 64, 2080, 2143, 4032, 4095, 1000],
                              np.random.default_rng(tag)))
    t0 = time.time()
    out.update(eig_fields("reig", R.randomized_eig((sd.axes, None), cov, 99, 20, SEED)))
    t1 = time.time()
    if h == 0.1:
        out.update(eig_fields("deig", R.dense_eig((sd.axes, None), cov, 20)))
    print(f"  randomized eig {t1 - t0:.1f}s dense {time.time() - t1:.1f}s", flush=True)
    return out


def cfg4():
    sd = draw(4)
    r, mean, sq, cov = smooth_all(sd, with_squares=False)
    out = header(4, sd, 2000)
    out.update(mean=mean)
    out.update(sample_entries(cov, 4096, sd.mask, 65536, [], np.random.default_rng(4)))
    out.update(eig_fields("reig", R.randomized_eig((sd.axes, sd.mask), cov, 99, 20, SEED)))
    return out


def cfg5_boxes():
    """48 (s box, t box) pairs of 2x4x4 node boxes: corners, edges, faces,
    interior, and the diagonal blocks among them."""
    lo_choices = [(0, 0, 0), (30, 28, 28), (0, 28, 14), (15, 14, 0), (14, 12, 12), (30, 0, 28)]
    boxes = [(np.array(l), np.array(l) + np.array([2, 4, 4])) for l in lo_choices]
    pairs = []
    for i, s in enumerate(boxes):
        for j, t in enumerate(boxes):
            pairs.append((s, t))
    rng = np.random.default_rng(5)
    while len(pairs) < 48:
        l1 = np.array([rng.integers(0, 31), rng.integers(0, 29), rng.integers(0, 29)])
        l2 = np.array([rng.integers(0, 31), rng.integers(0, 29), rng.integers(0, 29)])
        pairs.append(((l1, l1 + [2, 4, 4]), (l2, l2 + [2, 4, 4])))
    return pairs


def cfg5(n=100):
    sd = draw(5, n=n)
    grid = (sd.axes, None)
    t0 = time.time()
    r = R.linear_bin(grid, sd.offsets, sd.coords, sd.values, True, True)
    mean = R.fft_local_linear(r, grid, sd.h, 0)
    print(f"  bin+mean {time.time() - t0:.1f}s", flush=True)
    out = header(5, sd, n)
    out.update(mean=mean)
    pairs = cfg5_boxes()
    blocks = []
    t0 = time.time()
    for s, t in pairs:
        blocks.append(R.covariance_block(r, grid, sd.h, mean, s, t))
    print(f"  {len(pairs)} blocks {time.time() - t0:.1f}s", flush=True)
    out.update(block_s=np.array([np.concatenate(p[0]) for p in pairs], dtype=np.int64),
               block_t=np.array([np.concatenate(p[1]) for p in pairs], dtype=np.int64),
               block_vals=np.stack(blocks))
    return out


JOBS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg3w": lambda: cfg3(0.3, 33), "cfg4": cfg4, "cfg5": cfg5}


def main():
    R.set_threads(8)
    names = sys.argv[1:] or list(JOBS)
    for name in names:
        t0 = time.time()
        print(name, flush=True)
        out = JOBS[name]()
        np.savez_compressed(OUT / f"{name}.npz", **out)
        print(f"wrote {name}.npz in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
