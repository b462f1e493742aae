#!/usr/bin/env python3
"""One warm covariance step of the bench workload, for ncu captures.

    python tools/profile_step.py [--steps 2] [--cells 64] [--n 2000] [--h 0.1]

Runs linear_bin + fft_local_linear once, then `--steps` fft_covariance calls.
Under ncu use -s to skip the setup launches (see profiles/README.md).
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1510_04439_b200 import _lib, api, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--cells", type=int, default=64)
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--h", type=float, default=0.1)
    ap.add_argument("--dim", type=int, default=2)
    ap.add_argument("--stats", action="store_true", help="per-kernel device times (event-bracketed launches)")
    a = ap.parse_args()
    sd = synth.grid_nodes(a.dim, a.cells, a.n, a.h)
    grid = sd.grid()
    h = api.Bandwidth(sd.h)
    b = api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
    mean = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean)
    print("setup launches", _lib.kernel_launches(), flush=True)
    for i in range(a.steps):
        if a.stats and i == a.steps - 1:
            _lib.profile(True)
        c = api.fft_covariance(b, grid, h, mean)
        if a.stats and i == a.steps - 1:
            for k, (ms, cnt) in sorted(_lib.kernel_stats().items(), key=lambda kv: -kv[1][0]):
                print(f"  {k:40s} {cnt:5d} launches {ms:10.3f} ms", flush=True)
            _lib.profile(False)
        print("step total ms", _lib.stage_ms("total"), "launches", _lib.kernel_launches(), flush=True)
        del c


if __name__ == "__main__":
    main()
