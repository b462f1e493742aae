#!/usr/bin/env python3
"""Per-kernel device times (CUDA events around every launch) of one
randomized_eig on the bench covariance (q = 99, L = 20)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1510_04439_b200 import _lib, api, synth  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sd = synth.grid_nodes(2, cells, 2000, 0.1)
grid = sd.grid()
h = api.Bandwidth(sd.h)
b = api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
print("binning stage ms", _lib.stage_ms("binning"), "total", _lib.stage_ms("total"))
mean = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean)
cov = api.fft_covariance(b, grid, h, mean)
S = api.matrixize(cov)
api.randomized_eig(S, 99, 20, grid, 1)
for what in ("bin", "eig"):
    _lib.profile(True)
    if what == "bin":
        api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
    else:
        e = api.randomized_eig(S, 99, 20, grid, 20260815)
    st = _lib.kernel_stats()
    _lib.profile(False)
    print(f"--- {what}: total {_lib.stage_ms('total'):.3f} ms")
    for k, (ms, n) in sorted(st.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:32s} {n:5d} {ms:9.3f} ms")
print("eigenvalues", e.eigenvalues[:4])
