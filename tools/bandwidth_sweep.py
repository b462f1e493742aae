#!/usr/bin/env python3
"""Covariance step time against the kernel radius (the
reference switches AxisConv from direct taps to overlap-add FFT at 33 taps,
conv.hpp:73).  configs[2] geometry (d=2, 64^2, n=2000, GridNodes design from
the reference's generator); for each bandwidth: R, taps, device ms per
fft_covariance (median of --steps), the stage split and the moment-pass
kernels' time.  One JSON line per bandwidth.

    python tools/bandwidth_sweep.py [--h 0.05,0.1,...] [--steps 5]
"""
import argparse
import json
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1510_04439_b200 import _lib, api, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--h", default="0.05,0.1,0.15,0.2,0.25,0.3,0.35,0.4,0.5,0.6")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--cells", type=int, default=64)
    ap.add_argument("--n", type=int, default=2000)
    a = ap.parse_args()
    sd = synth.config(3, n=a.n, cells=a.cells)
    grid = sd.grid()
    data = sd.dataset()
    b = api.linear_bin(data, grid, api.BinOptions(True, True))
    for hs in a.h.split(","):
        hv = float(hs)
        h = api.Bandwidth([hv, hv])
        mean = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean)
        api.fft_covariance(b, grid, h, mean)  # warm (tables, allocations)
        ms, stages = [], {}
        for _ in range(a.steps):
            api.fft_covariance(b, grid, h, mean)
            ms.append(_lib.stage_ms("total"))
            for st in ("pairs", "moments", "solve", "fallback", "center"):
                stages[st] = stages.get(st, 0.0) + _lib.stage_ms(st) / a.steps
        _lib.profile(True)
        api.fft_covariance(b, grid, h, mean)
        ks = _lib.kernel_stats()
        _lib.profile(False)
        R = math.ceil(hv / grid.spacing(0) - 1e-9)
        moments_k = {k: round(v[0], 4) for k, v in ks.items() if k.startswith(("k_pass", "k_tphase", "k_conv"))}
        print(json.dumps({"h": hv, "R": R, "taps": 2 * R + 1, "reference_conv": "fft" if 2 * R + 1 >= 33 else "direct",
                          "ms": float(np.median(ms)), "gridpts_per_s": grid.size() ** 2 / (np.median(ms) / 1e3),
                          "stages_ms": {k: round(v, 4) for k, v in stages.items()}, "moment_kernels_ms": moments_k}),
              flush=True)


if __name__ == "__main__":
    main()
