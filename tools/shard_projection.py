#!/usr/bin/env python3
"""Per-rank device time of the slab-sharded covariance on ONE GPU: every rank
of a `world`-rank run computes its slab alone with the exchanges dropped
(dfpca_covariance_slab_dryrun), so max over ranks is the compute part of a
multi-GPU step; the exchange volumes of the schedule are printed beside it.
This is a projection for planning, not a multi-GPU measurement.

    python tools/shard_projection.py [--dim 2 --cells 64 --n 2000 --h 0.1] [--worlds 1,2,4,8]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1510_04439_b200 import _lib, api, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--cells", type=int, default=64)
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--h", type=float, default=0.1)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--stats", action="store_true", help="per-kernel times of the slowest rank")
    a = ap.parse_args()
    sd = synth.grid_nodes(a.dim, a.cells, a.n, a.h)
    grid = sd.grid()
    h = api.Bandwidth(sd.h)
    b = api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
    mean = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean)
    G = grid.size()
    n1 = a.cells
    rn = G // n1
    R = int(np.ceil(a.h / grid.spacing(0) - 1e-12))
    for _ in range(2):
        api.fft_covariance(b, grid, h, mean)
    ts = []
    for _ in range(a.reps):
        api.fft_covariance(b, grid, h, mean)
        ts.append(_lib.stage_ms("total"))
    one = min(ts)
    for world in [int(x) for x in a.worlds.split(",")]:
        per_rank = []
        for r in range(world):
            ts = []
            for _ in range(a.reps + 1):  # first call warms the allocator
                s = api.covariance_slab_dryrun(b, grid, h, mean, world, r)
                ts.append(_lib.stage_ms("total"))
                del s
            per_rank.append(min(ts[1:]))
        bl = api.shard_blocks(n1, rn, R, world, 0)
        b1 = api.shard_blocks(n1, rn, R, world, 1)

        def vol(blocks):
            v = np.zeros(world)
            for (src, dst, r0, r1, c0, c1, tr) in blocks:
                if src != dst:
                    v[dst] += 8.0 * (r1 - r0) * (c1 - c0)
            return v
        v0, v1 = vol(bl), vol(b1)
        print(json.dumps({"world": world, "bounds": api.shard_bounds(n1, rn, R, world),
                          "one_device_ms": one, "rank_ms": [round(x, 4) for x in per_rank],
                          "max_rank_ms": max(per_rank), "compute_efficiency": one / (world * max(per_rank)),
                          "recv_MB_pairs_max": float(v0.max() / 1e6), "recv_MB_cov_max": float(v1.max() / 1e6)}),
              flush=True)
        if a.stats:
            worst = int(np.argmax(per_rank))
            _lib.profile(True)
            s = api.covariance_slab_dryrun(b, grid, h, mean, world, worst)
            st = {k: round(v[0], 4) for k, v in sorted(_lib.kernel_stats().items(), key=lambda kv: -kv[1][0])}
            stages = {k: round(_lib.stage_ms(k), 4) for k in ("pairs", "exchange", "moments", "solve", "center")}
            _lib.profile(False)
            del s
            print(json.dumps({"world": world, "rank": worst, "kernels_ms": st, "stages_ms": stages}), flush=True)


if __name__ == "__main__":
    main()
