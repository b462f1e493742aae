#!/usr/bin/env python3
"""Times the 8(f) rank-1 stages (noise variance, scores, reconstruction) on the
GPU next to the reference (oracle/_ref, the reference's scores.hpp compiled
unchanged, host cores) on BASELINE configs 3 (dense, integration scores) and 4
(sparse masked, PACE scores), and checks parity on the same model.

    python tools/bench_scores.py [--reps 3]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1510_04439_b200 import api, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    from oracle import ref as R
    R.set_threads(os.cpu_count() or 1)
    for name, make, method in (("configs[2] d=2 64x64 n=2000 (integration)", lambda: synth.grid_nodes(2, 64, 2000, 0.1),
                                api.ScoreMethod.Integration),
                               ("configs[3] sparse masked 64x64 n=2000 (pace)", lambda: synth.sparse_masked(64, 2000, 0.15),
                                api.ScoreMethod.Pace)):
        sd = make()
        grid = sd.grid()
        b = api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
        h = api.Bandwidth(sd.h)
        mean = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean)
        diag = api.fft_local_linear(b, grid, h, api.MomentTarget.Squares)
        cov = api.fft_covariance(b, grid, h, mean)
        eig = api.randomized_eig(api.matrixize(cov), 99, 20, grid, 20260815)
        data = sd.dataset()
        t = []
        for _ in range(a.reps + 1):
            t0 = time.perf_counter()
            s2 = api.estimate_sigma2(diag, cov, mean)
            sc, _ = api.compute_scores_batch(data, grid, mean, eig, s2, method)
            rec = api.reconstruct_on_grid(mean, eig, sc)
            t.append(time.perf_counter() - t0)
        gpu_ms = 1e3 * float(np.median(t[1:]))
        efs = np.stack(eig.eigenfunctions)
        covv = cov.values
        t0 = time.perf_counter()
        rs2 = R.estimate_sigma2((sd.axes, sd.mask), diag.values, covv, mean.values)
        rsc, _ = R.scores((sd.axes, sd.mask), sd.offsets, sd.coords, sd.values, mean.values, eig.eigenvalues, efs,
                          rs2, method.value)
        rrec = np.stack([R.reconstruct_on_grid((sd.axes, sd.mask), mean.values, eig.eigenvalues, efs, rsc[i])
                         for i in range(rsc.shape[0])])
        cpu_ms = (time.perf_counter() - t0) * 1e3
        den = np.maximum(1.0, np.maximum(np.abs(sc), np.abs(rsc)))
        fin = ~np.isnan(rec)
        print(json.dumps({
            "workload": name, "n": int(sd.n_samples), "L": len(eig.eigenvalues), "G": grid.size(),
            "gpu_ms": gpu_ms, "cpu_reference_ms": cpu_ms, "cpu_cores": os.cpu_count(),
            "sigma2_bit_equal": bool(np.float64(s2).view(np.uint64) == np.float64(rs2).view(np.uint64)),
            "scores_max_rel_diff": float(np.max(np.abs(sc - rsc) / den)),
            "reconstruct_bit_equal": bool(np.array_equal(np.isnan(rec), np.isnan(rrec)) and
                                          np.array_equal(rec[fin].view(np.uint64), rrec[fin].view(np.uint64))),
        }), flush=True)


if __name__ == "__main__":
    main()
