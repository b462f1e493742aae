#!/usr/bin/env python3
"""Summaries of ncu output for profiles/.

    python tools/ncu_summary.py launches <launches.csv> [--skip N]
    python tools/ncu_summary.py full <report.ncu-rep>
"""
import csv
import io
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warp_latency_issue_stalled_barrier",
]


def clean(name: str) -> str:
    name = name.replace("(anonymous namespace)::", "").replace("void ", "").replace("dfpca_gpu::", "")
    return re.sub(r"\(.*$", "", name)


def launches(path, skip=0):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    seq = [(clean(r[ki]), float(r[vi].replace(",", "")) / 1e3) for r in rows[hdr + 1:] if len(r) > vi]
    seq = seq[skip:]
    agg = {}
    for n, t in seq:
        a = agg.setdefault(n, [0.0, 0])
        a[0] += t
        a[1] += 1
    tot = sum(t for _, t in seq)
    print(f"{'kernel':48s} {'launches':>8s} {'us':>10s} {'share':>6s}")
    for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k[:48]:48s} {c:8d} {t:10.1f} {t / tot:6.2f}")
    print(f"{'total':48s} {len(seq):8d} {tot:10.1f}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", clean(r[h.index("Kernel Name")]))
        for m in METRICS:
            if m in h:
                i = h.index(m)
                print(f"   {m:75s} {r[i]} {units[i]}".rstrip())


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
        launches(sys.argv[2], skip)
    else:
        full(sys.argv[2])
