#!/usr/bin/env python3
"""dense_eig on the device: the hand-written path (csrc/dense_eig.cu) against
cuSOLVER syevd (DFPCA_DENSE_EIG=cusolver) on a symmetric M x M matrix with a
decaying spectrum, L = 20; per-kernel device times of the hand-written path
(events around every launch), one JSON line per M.

    python tools/time_dense_eig.py [M ...]
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1510_04439_b200 import _lib, api  # noqa: E402


def matrix(M):
    rng = np.random.default_rng(1)
    Q, _ = np.linalg.qr(rng.standard_normal((M, 40)))
    S = (Q * (10.0 * 0.6 ** np.arange(40))) @ Q.T + 1e-9 * np.eye(M)
    return 0.5 * (S + S.T)


def timed(mz, grid, mode):
    os.environ["DFPCA_DENSE_EIG"] = mode
    t0 = time.perf_counter()
    e = api.dense_eig(mz, 20, grid)
    return (time.perf_counter() - t0) * 1e3, e


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [512, 1024, 2048, 4096]
    for M in sizes:
        t = (np.arange(M) + 0.5) / M
        grid = api.EvaluationGrid([list(t)])
        mz = api.matrixize(api.SurfaceEstimate(grid, api.SurfaceKind.Covariance, values=matrix(M).ravel()))
        first = {m: timed(mz, grid, m)[0] for m in ("cusolver", "native")}
        warm = {m: min(timed(mz, grid, m)[0] for _ in range(3)) for m in ("cusolver", "native")}
        _, a = timed(mz, grid, "cusolver")
        _, b = timed(mz, grid, "native")
        _lib.profile(True)
        timed(mz, grid, "native")
        ks = {k: round(v[0], 3) for k, v in _lib.kernel_stats().items()}
        _lib.profile(False)
        lam_a, lam_b = np.asarray(a.eigenvalues), np.asarray(b.eigenvalues)
        print(json.dumps({
            "M": M, "L": 20,
            "native_ms_first": round(first["native"], 2), "native_ms_warm": round(warm["native"], 2),
            "cusolver_ms_first": round(first["cusolver"], 2), "cusolver_ms_warm": round(warm["cusolver"], 2),
            "native_kernels_ms": ks,
            "max_rel_eigenvalue_diff": float(np.max(np.abs(lam_a - lam_b) / np.abs(lam_a))),
            "rel_total_variance_diff": abs(a.total_variance - b.total_variance) / a.total_variance,
        }), flush=True)


if __name__ == "__main__":
    main()
