"""Break the bench's end-to-end step (pinned host obs -> host covariance) into
its public-API calls, each bracketed by a device synchronize.

    python tools/time_e2e.py [--reps 5]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import bench
    from paper_1510_04439_b200 import _lib, api

    dev = torch.device("cuda", 0)
    sd = bench.make_data(seed=20260815)
    grid = sd.grid()
    h = api.Bandwidth(sd.h)
    data = sd.dataset()
    offsets, coords, values = data.csr()
    G2 = grid.size() ** 2
    host_cov = np.empty(G2)
    for a in (offsets, coords, values, host_cov):
        _lib.pin(a)
    rows = []
    for it in range(args.reps + 1):
        t = {}
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        b2 = api.linear_bin(data, grid, api.BinOptions(True, True))
        torch.cuda.synchronize(dev)
        t["linear_bin"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        m2 = api.fft_local_linear(b2, grid, h, api.MomentTarget.Mean)
        torch.cuda.synchronize(dev)
        t["mean"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        c2 = api.fft_covariance(b2, grid, h, m2)
        torch.cuda.synchronize(dev)
        t["covariance"] = time.perf_counter() - t0
        t["cov_device_total"] = _lib.stage_ms("total") / 1e3
        t0 = time.perf_counter()
        _lib.check(_lib.lib().dfpca_surface_download(_lib.ctx(), c2.device_handle(),
                                                     host_cov.ctypes.data_as(_lib.PD)))
        t["download"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        del b2, m2, c2
        torch.cuda.synchronize(dev)
        t["free"] = time.perf_counter() - t0
        if it > 0:
            rows.append(t)
    for k in rows[0]:
        print(f"{k:18s} {1e3 * np.mean([r[k] for r in rows]):9.3f} ms")


if __name__ == "__main__":
    main()
