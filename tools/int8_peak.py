#!/usr/bin/env python3
"""Dense int8 tensor-core peak of this GPU, measured like MEASURED_PEAKS.json's
bf16 figure: torch._int_mm (cuBLASLt, int8 x int8 -> int32) on N^3 products,
best of 10 (burst), CUDA events, with the SM clock sampled during the run.
The roofline denominator of the Ozaki SYRK (k_oz_syrk: tcgen05.mma kind::i8).

    python tools/int8_peak.py [--n 8192]
"""
import argparse
import json
import subprocess

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    a = ap.parse_args()
    n = a.n
    x = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    y = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    for _ in range(3):
        torch._int_mm(x, y)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(x, y)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    # sustained, with the clock sampled under load
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    reps = 200
    for _ in range(reps):
        torch._int_mm(x, y)
    e.record()
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    torch.cuda.synchronize()
    sustained = s.elapsed_time(e) / reps
    ops = 2.0 * n ** 3
    print(json.dumps({"int8_tops_burst": ops / best / 1e9, "int8_tops_sustained": ops / sustained / 1e9,
                      "n": n, "ms_best": best, "ms_sustained": sustained, "sm_clock_mhz_now_max": clk,
                      "how": "torch._int_mm (cuBLASLt) int8 x int8 -> int32, 2 N^3 ops"}))


if __name__ == "__main__":
    main()
