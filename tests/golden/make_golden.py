#!/usr/bin/env python3
"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself
(oracle/_ref/libdfpca_ref.so = /root/reference/proj/include/dfpca compiled
unchanged against oracle/shim).  Run in the build container:

    make -C oracle && python tests/golden/make_golden.py

Each fixture stores its inputs (so no generator has to stay bit-stable) and
the reference outputs.  They pin the oracle build (tests/test_oracle.py), the
numpy restatement (oracle/restate.py) and the GPU path (tests/test_gpu_parity.py,
__graft_entry__.smoke()).
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref as R  # noqa: E402
from paper_1510_04439_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent


def save(name, sd, extra):
    axes = np.concatenate([np.asarray(a, dtype=np.float64) for a in sd.axes])
    shape = np.array([len(a) for a in sd.axes], dtype=np.int64)
    np.savez_compressed(OUT / f"{name}.npz", axes=axes, shape=shape,
                        mask=np.asarray(sd.mask if sd.mask is not None else [], dtype=np.uint8),
                        offsets=sd.offsets, coords=sd.coords, values=sd.values, h=np.asarray(sd.h), **extra)
    print("wrote", name)


def binned_fields(r):
    f = r.fields()
    return {f"bin_{k}": v for k, v in f.items()}


def main():
    cases = {
        "cov2d_random": synth.random_points(2, 9, 12, 10, 0.3, seed=11),
        "cov1d_random": synth.random_points(1, 26, 20, 8, 0.2, seed=12),
        "cov2d_nodes": synth.grid_nodes(2, 8, 10, 0.25, seed=13),
        "cov2d_masked": synth.sparse_masked(10, 60, 0.35, seed=14),
    }
    for name, sd in cases.items():
        grid = (sd.axes, sd.mask)
        r = R.linear_bin(grid, sd.offsets, sd.coords, sd.values, True, True)
        mean = R.fft_local_linear(r, grid, sd.h, 0)
        sq = R.fft_local_linear(r, grid, sd.h, 1)
        cov = R.fft_covariance(r, grid, sd.h, mean)
        pw, pv = R.pair_grids(r)
        extra = binned_fields(r)
        extra.update(mean=mean, squares=sq, cov=cov, pw=pw, pv=pv)
        M = int(np.prod([len(a) for a in sd.axes])) if sd.mask is None else int(np.count_nonzero(sd.mask))
        q = min(20, M)
        eig = R.randomized_eig(grid, cov, q, 3, 20260815)
        extra.update(eig_values=eig["eigenvalues"], eig_functions=eig["eigenfunctions"], eig_fve=eig["fve"],
                     eig_total=np.array([eig["total_variance"]]), eig_q=np.array([q]))
        # noise variance, scores (both methods), reconstruction,
        # dense eigendecomposition -- on the reference's own model surfaces
        s2 = R.estimate_sigma2(grid, sq, cov, mean)
        efs = eig["eigenfunctions"]
        pace, _ = R.scores(grid, sd.offsets, sd.coords, sd.values, mean, eig["eigenvalues"], efs, s2, 0)
        integ, warn = R.scores(grid, sd.offsets, sd.coords, sd.values, mean, eig["eigenvalues"], efs, s2, 1)
        rec = R.reconstruct_on_grid(grid, mean, eig["eigenvalues"], efs, integ[0])
        dense = R.dense_eig(grid, cov, 3)
        extra.update(sigma2=np.array([s2]), scores_pace=pace, scores_integration=integ,
                     scores_sparse_warning=warn.astype(np.uint8), reconstruct0=rec,
                     dense_values=dense["eigenvalues"], dense_functions=dense["eigenfunctions"],
                     dense_fve=dense["fve"], dense_total=np.array([dense["total_variance"]]))
        save(name, sd, extra)


if __name__ == "__main__":
    main()
