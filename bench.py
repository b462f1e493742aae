#!/usr/bin/env python3
"""Benchmark of the binned FPCA covariance smoother on the GPU (libdfpca_cuda.so).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload = BASELINE.json configs[2]: d = 2, n = 2000 subjects observed at every
node of a 64 x 64 midpoint grid, h = 0.1 (R = 7, 15 taps), 4-D local-linear
covariance over G^2 = 16,777,216 grid points (synthetic data of that shape).

A "step" is one fft_covariance (reference fft_smoother.hpp:585): pair grids,
the 20 kernel-moment convolutions, the per-node 5x5 solves with the fallback
ladder, centering and symmetrization, from device-resident binned data to a
device-resident covariance.  value = G^2 / step time (gridpts/s).  N > 1 splits
the one covariance into s1-plane slabs, one per GPU (csrc/shard.hpp: SYRK over
each rank's row tiles, NCCL exchanges of the pair-grid windows and of the
covariance rows), step time = max over ranks ("scaling": "strong").
e2e: the same metric through the public API with host buffers, over the FPCA
core of SURVEY.md 8(d): pinned host observations -> linear_bin ->
fft_local_linear (Mean, Squares) -> fft_covariance -> randomized_eig (q=99,
L=20) -> EigenSystem (eigenvalues and eigenfunction surfaces) on the host,
every step.  The inputs are drawn by the reference's own generator.

--impl reference times the reference implementation itself (oracle/_ref: the
reference's headers compiled unchanged) on the host cores on the SAME
workload: one full FPCA run (~100 s; --ref-steps runs, --steps ignored), value
from its fft_covariance stage, e2e from the whole run.  Our line's
cpu_baseline is a bounded sample (first --cpu-subjects subjects).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CELLS, N_SUBJ, H = 64, 2000, 0.1
METRIC = "smoothed covariance gridpts/s (d=2 64², 4-D LL); end-to-end FPCA time vs CPU"
WORKLOAD = ("configs[2]: d=2 n=2000 on 64x64 midpoint grid, GridNodes design, h=0.1 (R=7), fft_covariance; "
            "inputs drawn by the reference's generator (simulate.hpp, seed 20260815)")
PEAKS = ROOT / "MEASURED_PEAKS.json"
# FP64 peak of this pool's B200 (DMMA m8n8k4 and DFMA both), measured with
# tools/fp64_peak.cu (profiles/fp64_peak_r01.txt); MEASURED_PEAKS.json has no FP64 entry.
FP64_PEAK_TFLOPS = 37.07
# Dense int8 tensor peak of this pool's B200, measured like MEASURED_PEAKS.json's
# bf16 figure (cuBLASLt int8 GEMM, 8192^3, best of 10; tools/int8_peak.py,
# profiles/r07_int8_peak.jsonl): the denominator of the Ozaki SYRK (k_oz_syrk).
INT8_PEAK_TOPS = 3126.7
OZ_SLICES = 8  # csrc/ozaki.cu kOzS


def rank_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    (every 2 ms, microsecond queries) when the driver's library is present,
    else nvidia-smi (every 0.1 s)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.query_s = []
        self.source = "nvidia-smi"
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._h = nv.nvmlDeviceGetHandleByIndex(device)
            self._max = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                          nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            self._nv = nv
            self.source = "nvml"
        except Exception:
            self._nv = None

    def _sample_nvml(self):
        nv = self._nv
        q0 = time.perf_counter()
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        self.query_s.append(time.perf_counter() - q0)
        self.rows.append([str(sm), str(self._max)] + ["Active" if rs & b else "Not Active" for b in self._bits])

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nv is not None:
                    self._sample_nvml()
                    self._stop.wait(0.002)
                    continue
                q0 = time.perf_counter()
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                self.query_s.append(time.perf_counter() - q0)
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "source": self.source}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "sm_min_mhz": min(sm) if sm else None, "reasons": reasons, "samples": len(self.rows),
                "source": self.source,
                "query_ms": float(1e3 * np.median(self.query_s)) if self.query_s else None}


# ------------------------------------------------------------------- data --
def make_data(seed=20260815):
    """configs[2] drawn by the reference's own generator (simulate.hpp's
    generate() restated bit for bit in the library: dfpca_simulate)."""
    from paper_1510_04439_b200 import synth
    return synth.config(3, n=N_SUBJ, h=H, cells=CELLS, seed=seed)


def cpu_sample(sd, n_sub: int):
    """Bounded reference sample: the same grid, bandwidth and design with the
    first n_sub subjects (the pair build is O(n), convolutions and solves are
    O(G^2) and unchanged)."""
    G = CELLS * CELLS
    off = sd.offsets[:n_sub + 1]
    return off, sd.coords[:off[-1] * 2], sd.values[:off[-1]]


# -------------------------------------------------------------- reference --
def reference_fpca(sd, threads: int):
    """One run of the reference's FPCA core on the host (oracle/_ref: the
    reference's headers compiled unchanged): the stages of fit_pipeline
    (pipeline.hpp:308-340) timed like its StageClock (pipeline.hpp:143-165):
    linear_bin, fft_local_linear(Mean), fft_local_linear(Squares),
    fft_covariance, matrixize + randomized_eig(q=99, L=20).  Seconds per stage."""
    from oracle import ref as R
    R.set_threads(threads)
    grid = (sd.axes, sd.mask)
    t = {}
    t0 = time.perf_counter()
    b = R.linear_bin(grid, sd.offsets, sd.coords, sd.values, True, True)
    t["linear_bin"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    mu = R.fft_local_linear(b, grid, sd.h, 0)
    t["mean"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    R.fft_local_linear(b, grid, sd.h, 1)
    t["squares"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    cov = R.fft_covariance(b, grid, sd.h, mu)
    t["covariance"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    eig = R.randomized_eig(grid, cov, 99, 20, 20260815)
    t["randomized_eig"] = time.perf_counter() - t0
    return t, eig


def run_reference(args, emit=True):
    """--impl reference: the reference's own CPU implementation of the path on
    the SAME workload as our arm (n = 2000, 64^2, h = 0.1), all host threads.
    One FPCA run is ~100 s of host time (its pair build is serial), so the
    arm runs --ref-steps of them (default 1) whatever --steps says: a
    same-config number rather than a same-step-count one.  value = G^2 / the
    fft_covariance time; e2e = G^2 / the whole FPCA (host observations ->
    EigenSystem), the same stages as our e2e."""
    rank, world, _ = rank_env()
    if rank != 0:
        return None
    cores = os.cpu_count() or 1
    sd = make_data()
    G2 = (CELLS * CELLS) ** 2
    n_steps = max(1, args.ref_steps if args.ref_steps else 1)
    for _ in range(args.ref_warmup if args.ref_warmup is not None else 0):
        reference_fpca(sd, cores)
    runs = [reference_fpca(sd, cores) for _ in range(n_steps)]
    t_cov = float(np.mean([r[0]["covariance"] for r in runs]))
    t_all = float(np.mean([sum(r[0].values()) for r in runs]))
    stages = {k: float(np.mean([r[0][k] for r in runs])) * 1e3 for k in runs[0][0]}
    val = G2 / t_cov
    sample = (f"the full workload: fft_covariance of all {N_SUBJ} subjects on the 64x64 grid "
              f"(16,777,216 gridpts), reference headers compiled unchanged (oracle/_ref), "
              f"set_max_threads({cores}); {n_steps} run(s), --steps ignored (one run is ~60 s)")
    line = {"metric": METRIC, "value": val, "unit": "gridpts/s", "n_gpus": args.gpus, "steps": n_steps,
            "warmup": 0, "ms_per_step": t_cov * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "cpu_sample": f"full config, n={N_SUBJ}", "same_config": True},
            "impl": "reference",
            "stages_ms": stages,
            "eig_top3": [float(x) for x in runs[-1][1]["eigenvalues"][:3]],
            "cpu_baseline": {"value": val, "unit": "gridpts/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": G2 / t_all, "unit": "gridpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                    "ms_per_step": t_all * 1e3,
                    "path": "host observations -> linear_bin -> mean -> squares -> fft_covariance -> "
                            "randomized_eig (q=99, L=20) -> EigenSystem"}}
    if emit:
        print(json.dumps(line), flush=True)
    return line


def reference_sample_baseline(args):
    """cpu_baseline of our line: the reference's fft_covariance on a bounded
    sample of the workload (the first --cpu-subjects subjects on the full
    64^2 grid: the pair build is O(n), convolutions and solves are O(G^2) and
    unchanged), so the default bench run stays within minutes."""
    from oracle import ref as R
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    sd = make_data()
    n_sub = args.cpu_subjects
    off, coords, values = cpu_sample(sd, n_sub)
    grid = (sd.axes, None)
    b = R.linear_bin(grid, off, coords, values, True, True)
    mu = R.fft_local_linear(b, grid, sd.h, 0)
    t0 = time.perf_counter()
    R.fft_covariance(b, grid, sd.h, mu)
    t = time.perf_counter() - t0
    return {"value": (CELLS * CELLS) ** 2 / t, "unit": "gridpts/s", "cores": cores, "kind": "reference",
            "sample": (f"fft_covariance on the full 64x64 grid (16,777,216 gridpts), first {n_sub} of {N_SUBJ} "
                       f"subjects, reference headers compiled unchanged (oracle/_ref), set_max_threads({cores}); "
                       f"the same-config reference is bench.py --impl reference")}


# ------------------------------------------------------ long-format tables --
IO_METRIC = "long-format observation rows/s (read_long_format, io.hpp:115)"
IO_WORKLOAD = ("configs[2] observations as a long-format table: 8,192,000 rows (d=2, n=2000 x 64^2 nodes), "
               "tab-separated %.17g, ids s<i> (SURVEY.md 8(f) rank 2)")


def io_table(sd, path, n_samples=None):
    from paper_1510_04439_b200 import synth
    with open(path, "wb") as f:
        f.write(synth.long_format_bytes(sd, n_samples))
    return os.path.getsize(path), int(sd.offsets[n_samples if n_samples else -1])


def run_io_reference(args, path_full=None, emit=True):
    """The reference's read_long_format (oracle/_ref: io.hpp compiled
    unchanged), single-threaded as in the reference, on the first
    --cpu-io-subjects subjects of the table."""
    import tempfile
    from oracle import ref as R
    rank, _, _ = rank_env()
    if rank != 0:
        return None
    sd = make_data()
    n_sub = args.cpu_io_subjects
    path = os.path.join(tempfile.mkdtemp(), "sample.tsv")
    size, rows = io_table(sd, path, n_sub)
    for _ in range(args.ref_warmup if args.ref_warmup is not None else 1):
        R.read_long_format(path)
    times = []
    for _ in range(max(1, args.ref_steps if args.ref_steps else 3)):
        t0 = time.perf_counter()
        R.read_long_format(path)
        times.append(time.perf_counter() - t0)
    os.unlink(path)
    t = float(np.mean(times))
    val = rows / t
    line = {"metric": IO_METRIC, "value": val, "unit": "rows/s", "n_gpus": args.gpus, "steps": len(times),
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": IO_WORKLOAD, "cpu_sample": f"first {n_sub} subjects: {rows} rows, {size} bytes"},
            "impl": "reference",
            "cpu_baseline": {"value": val, "unit": "rows/s", "cores": 1, "kind": "reference",
                             "sample": f"read_long_format of the first {n_sub} of {N_SUBJ} subjects ({rows} rows, "
                                       f"{size / 1e6:.1f} MB, page cache), reference io.hpp compiled unchanged"},
            "e2e": {"value": val, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if emit:
        print(json.dumps(line), flush=True)
    return line


def run_io(args):
    """A step = one read_long_format of the full table.  value: the device
    stages (text resident in HBM -> CSR table in HBM: newline scan, parse,
    grouping, scatter; CUDA-event timed); e2e: the public call from the file
    (page cache) to the host FunctionalDataset arrays, wall clock."""
    import ctypes as C
    import tempfile
    rank, world, local = rank_env()
    if rank != 0:
        return
    os.environ.setdefault("DFPCA_DEVICE", str(local))
    from paper_1510_04439_b200 import _lib, api
    sd = make_data()
    path = os.path.join(tempfile.mkdtemp(), "cfg3.tsv")
    size, rows = io_table(sd, path)
    L = _lib.lib()
    dev_stages = ("lines", "parse", "group", "scatter")

    def read_table():
        h = C.c_void_p()
        _lib.check(L.dfpca_read_long_format(_lib.ctx(), path.encode(), C.byref(h)))
        st = {k: _lib.stage_ms(k) for k in dev_stages + ("upload", "total")}
        return h, st

    for _ in range(args.warmup):
        h, _ = read_table()
        L.dfpca_table_free(h)
    launches0 = _lib.kernel_launches()
    dev_ms, stage_acc = [], {}
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            h, st = read_table()
            L.dfpca_table_free(h)
            dev_ms.append(sum(st[k] for k in dev_stages))
            for k, v in st.items():
                stage_acc[k] = stage_acc.get(k, 0.0) + v
    launches = _lib.kernel_launches() - launches0
    t_dev = float(np.mean(dev_ms)) / 1e3
    _lib.profile(True)
    h, _ = read_table()
    kstats = _lib.kernel_stats()
    L.dfpca_table_free(h)
    _lib.profile(False)
    e2e = []
    for it in range(args.e2e_steps + 1):
        t0 = time.perf_counter()
        ds = api.read_long_format(path)
        if it > 0:
            e2e.append(time.perf_counter() - t0)
    off, coords, values = ds.csr()
    assert int(off[-1]) == rows and np.array_equal(values.view(np.uint64), sd.values.view(np.uint64))
    d2h = off.nbytes + coords.nbytes + values.nbytes + sum(len(s.id) for s in ds.samples) + off.nbytes
    t_e2e = float(np.mean(e2e))
    # file -> binned data (the fit pipeline's first two stages): the table
    # parsed and binned on the device (bin_long_format) against the two public
    # calls with the dataset crossing to the host and back in between
    grid, bopt = sd.grid(), api.BinOptions(True, True)
    fused, split = [], []
    for it in range(args.e2e_steps + 1):
        # calls are synchronous at return; the binned data stays on the device
        t0 = time.perf_counter()
        b1, _ = api.bin_long_format(path, grid, bopt)
        t1 = time.perf_counter()
        b2 = api.linear_bin(api.read_long_format(path), grid, bopt)
        t2 = time.perf_counter()
        m1, m2 = np.asarray(b1.diag_value), np.asarray(b2.diag_value)
        if it > 0:
            fused.append(t1 - t0)
            split.append(t2 - t1)
    assert np.array_equal(m1.view(np.uint64), m2.view(np.uint64))
    del b1, b2
    os.unlink(path)
    # roofline of the dominant device kernel (HBM-bound byte work).  Algorithmic
    # bytes per launch: k_split_lines reads every text byte once plus two
    # newline offsets per line and writes the record flag, id start / length
    # and the F field bounds (8 + 8 + 4 + 8F B per line); k_parse_fields reads,
    # per number field, its bounds, the line start and its text, and writes the
    # value (the field text is ~ the text bytes minus ids and separators)
    F = 4
    models = {"k_split_lines": size + rows * (16 + 8 + 8 + 4 + 8 * F),
              "k_parse_fields": size + rows * 3 * (8 + 8 + 8)}
    top = max((k for k in models if k in kstats), key=lambda k: kstats[k][0], default=None)
    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm = peaks.get("hbm_gbs", 6548.8)
    roof = None
    if top:
        ms = kstats[top][0]
        alg = models[top]
        ach = alg / (ms / 1e3) / 1e9
        tr, tr_src = ncu_traffic(top, "io_r*_ncu_full_summary.txt")
        roof = {"kernel": top, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": tr, "traffic_source": tr_src,
                "algorithmic_bytes_per_launch": alg, "kernel_ms": ms,
                "model": {"k_split_lines": "text bytes + 16 B newline offsets + (28 + 8F) B outputs per row",
                          "k_parse_fields": "text bytes + 24 B (bounds, line start, value) per number field"},
                "share_of_device_stages": ms / (t_dev * 1e3),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}
    cpu = None
    if not args.no_cpu_baseline:
        try:
            ra = argparse.Namespace(**vars(args))
            ra.ref_steps, ra.ref_warmup = 2, 1
            cpu = run_io_reference(ra, emit=False)["cpu_baseline"]
        except Exception as e:
            cpu = {"value": None, "unit": "rows/s", "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}
    out = {"metric": IO_METRIC, "value": rows / t_dev, "unit": "rows/s", "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t_dev * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": IO_WORKLOAD, "rows": rows, "bytes": size,
                      "l2": "inputs larger than L2 (373 MB text)"},
           "stages_ms_per_step": {k: v / args.steps for k, v in stage_acc.items()},
           "e2e": {"value": rows / t_e2e, "unit": "rows/s", "h2d_bytes_per_step": int(size),
                   "d2h_bytes_per_step": int(d2h), "ms_per_step": t_e2e * 1e3,
                   "all_ms": [round(t * 1e3, 2) for t in e2e],
                   "path": "file (page cache) -> pinned slots -> HBM -> device parse/group -> host CSR arrays"},
           "file_to_binned": {"ms_bin_long_format": float(np.mean(fused)) * 1e3,
                              "ms_read_then_linear_bin": float(np.mean(split)) * 1e3,
                              "grid": [int(n) for n in grid.shape()], "mean_path": True, "covariance_path": True,
                              "path": "bin_long_format: file -> HBM -> parse/group -> binning, observations stay "
                                      "on the device; vs read_long_format -> host arrays -> linear_bin",
                              "bit_identical": True},
           "gpu_launches": int(launches),
           "kernels": {k: {"ms": v[0], "launches": v[1]} for k, v in sorted(kstats.items(), key=lambda kv: -kv[1][0])},
           "roofline": roof, "cpu_baseline": cpu, "clocks": clk.summary()}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------- ours --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-subjects", type=int, default=100)
    ap.add_argument("--ref-steps", type=int, default=None)
    ap.add_argument("--ref-warmup", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--workload", choices=["covariance", "io"], default="covariance",
                    help="io: the long-format table reader (SURVEY.md 8(f) rank 2)")
    ap.add_argument("--cpu-io-subjects", type=int, default=200)
    ap.add_argument("--h", type=float, default=None,
                    help="bandwidth override (configs[2] is quoted at h = 0.1; SURVEY.md 8(d) also times 0.3, "
                         "R = 20, the reference's FFT path)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.h is not None:
        global H, WORKLOAD
        H = args.h
        WORKLOAD = WORKLOAD.replace("h=0.1 (R=7)", f"h={H} (R={int(np.ceil(H * CELLS))})")

    if args.workload == "io":
        if args.impl == "reference":
            run_io_reference(args)
        else:
            run_io(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return

    rank, world, local = rank_env()
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    os.environ.setdefault("DFPCA_DEVICE", str(local))

    from paper_1510_04439_b200 import _lib, api
    sharded = world > 1
    if sharded:
        # this process's rank of the slab-sharded covariance (csrc/shard.hpp):
        # our own NCCL communicator, its unique id broadcast over torch's
        def bcast(uid):
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            return obj[0]
        api.init_distributed(world, rank, broadcast=bcast)
    cov_fn = api.fft_covariance_sharded if sharded else api.fft_covariance
    # every rank holds the same data: one covariance split across the GPUs
    sd = make_data(seed=20260815)
    grid = sd.grid()
    h = api.Bandwidth(sd.h)
    G = grid.size()
    G2 = G * G
    data = sd.dataset()

    binned = api.linear_bin(data, grid, api.BinOptions(True, True))
    mean = api.fft_local_linear(binned, grid, h, api.MomentTarget.Mean)

    # L2 flush buffer (> 126 MB L2) written between timed steps through torch
    import torch
    dev = torch.device("cuda", local)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MB

    def one_step():
        cov = cov_fn(binned, grid, h, mean)
        return _lib.stage_ms("total"), cov

    for _ in range(args.warmup):
        one_step()

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()

    launches0 = _lib.kernel_launches()
    dev_ms = []
    stage_acc = {}
    barrier()
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize(dev)
            ms, cov = one_step()
            dev_ms.append(ms)
            for st in ("pairs", "moments", "solve", "fallback", "center"):
                stage_acc[st] = stage_acc.get(st, 0.0) + _lib.stage_ms(st)
            del cov
        wall = time.perf_counter() - wall0
    barrier()
    launches = _lib.kernel_launches() - launches0
    t_step = float(np.sum(dev_ms)) / args.steps / 1e3
    if dist is not None:
        tt = torch.tensor([t_step], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    value = G2 / t_step  # one covariance per step, split across the ranks

    # ---- per-kernel profile pass (outside the timed region) ----
    _lib.profile(True)
    one_step()
    kstats = _lib.kernel_stats()
    _lib.profile(False)

    # ---- e2e through the public API with pinned host buffers ----
    # host observations -> EigenSystem on the host, the stages
    # of fit_pipeline (pipeline.hpp:308-340): linear_bin, fft_local_linear
    # (Mean, Squares), fft_covariance, matrixize + randomized_eig (q=99,
    # L=20); the eigenvalues and eigenfunction surfaces come back every step.
    offsets, coords, values = data.csr()
    probe = cov_fn(binned, grid, h, mean)
    slab_row0, slab_rows = probe.rows()
    del probe
    host_cov = np.empty(slab_rows * G)
    pinned = [_lib.pin(a) for a in (offsets, coords, values, host_cov)]
    Q_SKETCH, L_MAX = 99, 20

    def fpca(stage_times=None):
        def mark(name, t_prev):
            if stage_times is not None:
                torch.cuda.synchronize(dev)
                now = time.perf_counter()
                stage_times[name] = stage_times.get(name, 0.0) + (now - t_prev)
                return now
            return t_prev
        t = time.perf_counter()
        b2 = api.linear_bin(data, grid, api.BinOptions(True, True))
        t = mark("linear_bin", t)
        m2 = api.fft_local_linear(b2, grid, h, api.MomentTarget.Mean)
        t = mark("mean", t)
        api.fft_local_linear(b2, grid, h, api.MomentTarget.Squares)
        t = mark("squares", t)
        c2 = cov_fn(b2, grid, h, m2)
        t = mark("covariance", t)
        es = api.randomized_eig(api.matrixize(c2), Q_SKETCH, L_MAX, grid, 20260815)
        mark("randomized_eig", t)
        return es

    e2e_t = []
    for it in range(args.e2e_steps + 1):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        es = fpca()
        t1 = time.perf_counter()
        if it > 0:
            e2e_t.append(t1 - t0)
    e2e_step = float(np.mean(e2e_t))
    eig_top3 = [float(x) for x in es.eigenvalues[:3]]
    n_comp = len(es.eigenvalues)
    d2h = 8 * n_comp * (G + 2) + 8  # eigenvalues, FVE, eigenfunction surfaces, total variance
    # one more pass, synchronised per stage, for the breakdown (not timed above)
    brk = {}
    fpca(brk)
    eig_ms = _lib.stage_ms("eigen")
    # the previous e2e scope, kept for comparison: observations -> covariance
    # copied back to pinned host memory
    cov_t = []
    for it in range(3):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        b2 = api.linear_bin(data, grid, api.BinOptions(True, True))
        m2 = api.fft_local_linear(b2, grid, h, api.MomentTarget.Mean)
        c2 = cov_fn(b2, grid, h, m2)
        _lib.check(_lib.lib().dfpca_surface_download(_lib.ctx(), c2.device_handle(),
                                                     host_cov.ctypes.data_as(_lib.PD)))
        if it > 0:
            cov_t.append(time.perf_counter() - t0)
        del b2, m2, c2
    if dist is not None:
        tt = torch.tensor([e2e_step], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_step = float(tt.item())
    h2d = offsets.nbytes + coords.nbytes + values.nbytes

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ----
    roof = roofline(kstats, G, binned, slab=(slab_row0, slab_rows) if sharded else None)

    # ---- CPU baseline (reference, rank 0, N = 1) ----
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = reference_sample_baseline(args)
        except Exception as e:  # oracle missing on this box
            cpu = {"value": None, "unit": "gridpts/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    out = {
        "metric": METRIC, "value": value, "unit": "gridpts/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "grid": [CELLS, CELLS], "n_subjects": N_SUBJ, "h": H,
                   "gridpts": G2, "l2": "flushed (256 MB write) before every timed step",
                   "parallelism": (f"slab-sharded s1 planes over {world} GPUs (NCCL exchanges of pair-grid "
                                   f"windows and covariance rows), rank 0 rows [{slab_row0}, {slab_row0 + slab_rows})"
                                   if sharded else "single GPU")},
        "stages_ms_per_step": {k: v / args.steps for k, v in stage_acc.items()},
        "wall_ms_per_step": wall / args.steps * 1e3,
        "e2e": {"value": G2 / e2e_step, "unit": "gridpts/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_step * 1e3,
                "breakdown_ms": {k: v * 1e3 for k, v in brk.items()},
                "all_ms": [round(t * 1e3, 3) for t in e2e_t],
                "path": ("pinned host obs -> linear_bin -> fft_local_linear (Mean, Squares) -> fft_covariance -> "
                         f"randomized_eig (q={Q_SKETCH}, L={L_MAX}) -> EigenSystem on the host"),
                "pinned": all(pinned),
                "to_covariance_ms": float(np.mean(cov_t)) * 1e3},
        "eigen_ms": eig_ms, "eig_top3": eig_top3, "eig_components": n_comp,
        "gpu_launches": int(launches),
        "kernels": {k: {"ms": v[0], "launches": v[1]} for k, v in sorted(kstats.items(), key=lambda kv: -kv[1][0])},
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def tri_fractions(cells: int, R: int, tile: int = 64):
    """Row fractions of the upper-triangle s-phase (csrc/conv.cuh View::tri):
    for each column tile, the s1 pass reads s1 < min(n1, s1_out + R) rows and
    writes s1 < s1_out rows, the in-plane pass works on those; the solve and
    the centering touch s <= t."""
    n1 = cells
    G = cells * cells
    rows_in = rows_out = 0
    for c0 in range(0, G, tile):
        tmax = min(c0 + tile, G) - 1
        s1_out = tmax // cells + 1
        rows_in += min(n1, s1_out + R) * (min(c0 + tile, G) - c0)
        rows_out += s1_out * (min(c0 + tile, G) - c0)
    upper = (G * (G + 1) / 2) / (G * G)
    return rows_in / (n1 * G), rows_out / (n1 * G), upper


def tphase_fractions(cells: int, R: int):
    """Fractions of the t-planes the trimmed t-phase reads and writes
    (csrc/smooth.cu: row s computes the t1 planes >= plane(s) - t1_margin,
    t1_margin = R + ceil(64 / cells), and reads R more planes below them):
    averaged over the pair-grid rows s."""
    margin = R + (64 + cells - 1) // cells
    rd = wr = 0.0
    for s1 in range(cells):
        lo = max(0, s1 - margin)
        wr += (cells - lo) / cells
        rd += (cells - max(0, lo - R)) / cells
    return rd / cells, wr / cells


def kernel_model(G: int, n_pair: int, shared: bool):
    """Algorithmic work per step of every kernel of the d = 2 covariance step
    (DESIGN.md 'Roofline model'); one array = G^2 doubles.

    pairs   k_gemm_tn     SYRK of the pair-weighted value grids: n G^2 FMAs
                          (the symmetric half of 2 n G^2 flops)    -> FP64 tensor
            k_rank_one    pw = W M(s) M(t): write 1 array          -> HBM
            k_scale_rows  w_i V_i: read + write n G doubles
    t-phase k_tphase2(v)  read pw, pv; write 9 t-partials -- the planes the
                          trimmed kernel actually moves (tphase_fractions:
                          0.71 of the input planes read, 0.62 of the output
                          planes written at cfg 3: 347 MB, ncu 293 MB)
    s-phase k_pass_cols   s1 pass first: 9 in (rows s1 < s1_out + R) + 14 out
                          (rows s1 < s1_out); s2 pass: 14 in + 20 out on those rows
    solve   k_solve       20 moments in + 1 out at s <= t
    center  k_center_mirror  read s <= t, write both triangles

    shared: the shared-constant design (every subject observed at every node,
    the bench's GridNodes workload): the mass moments are closed-form
    (k_solve_sep_tri), pw is never built, only pv is convolved:
    t-phase   read pv, write 3 value t-partials (trimmed as above)
    s-phase   s1: 3 in (trimmed + R rows) + 4 out; s2: 4 in + 5 out (s <= t rows)
    solve     5 value moments in + 1 out at s <= t
    """
    cells = int(round(G ** 0.5))
    R = int(np.ceil(H * cells))
    f_in, f_out, upper = tri_fractions(cells, R)
    t_rd, t_wr = tphase_fractions(cells, R)
    arr = 8.0 * G * G
    # Ozaki SYRK (csrc/ozaki.cu): the S(S+1)/2 slice-pair int8 products over
    # the upper triangle, 2 ops per MAC (the kernel also multiplies the zero
    # padding of K to a multiple of 64 and whole 128 x 128 diagonal tiles);
    # slicing reads the value grids once and writes 2 S bytes per entry
    S = OZ_SLICES
    ozaki = {
        "k_oz_syrk": ("int8", 2.0 * S * (S + 1) / 2 * n_pair * G * (G + 1) / 2),
        "k_oz_slice": ("hbm", 8.0 * n_pair * G + 2.0 * S * n_pair * G),
        "k_oz_colmax": ("hbm", 8.0 * n_pair * G),
    }
    if shared:
        return {
            **ozaki,
            "k_gemm_tn": ("tensor", 2.0 * n_pair * G * G / 2.0),
            "k_scale_rows": ("hbm", 2 * 8.0 * n_pair * G),
            "k_tphase2": ("hbm", (1 * t_rd + 3 * t_wr) * arr),
            "k_tphase2v": ("hbm", (1 * t_rd + 3 * t_wr) * arr),
            "k_pass_cols": ("hbm", (3 * f_in + 4 * f_out + (4 + 5) * f_out) * arr),
            "k_solve_sep_tri": ("hbm", 6 * upper * arr),
            "k_solve_shared_tri": ("hbm", 6 * upper * arr),
            "k_center_mirror": ("hbm", (upper + 1.0) * arr),
        }
    return {
        **ozaki,
        "k_gemm_tn": ("tensor", 2.0 * n_pair * G * G / 2.0),
        "k_rank_one": ("hbm", 1 * arr),
        "k_scale_rows": ("hbm", 2 * 8.0 * n_pair * G),
        "k_tphase2": ("hbm", (2 * t_rd + 9 * t_wr) * arr),
        "k_tphase2v": ("hbm", (2 * t_rd + 9 * t_wr) * arr),
        "k_pass_cols": ("hbm", (9 * f_in + 14 * f_out + (14 + 20) * f_out) * arr),
        "k_solve_tri": ("hbm", 21 * upper * arr),
        "k_center_mirror": ("hbm", (upper + 1.0) * arr),
    }


def ncu_traffic(kernel: str, pattern: str = "r*_ncu_full_summary.txt"):
    """dram__bytes_read.sum + dram__bytes_write.sum (bytes) of one launch of
    `kernel` from the newest committed `ncu --set full` summary
    (profiles/rNN_ncu_full_summary.txt, written by tools/ncu_summary.py full;
    values in Mbyte as ncu reports them), or (None, None)."""
    files = sorted((ROOT / "profiles").glob(pattern))
    if not files:
        return None, None
    cur, vals = None, {}
    for line in files[-1].read_text().splitlines():
        if line.startswith("== "):
            cur = line[3:].strip()
            continue
        parts = line.split()
        if cur and len(parts) in (2, 3) and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            base = cur.split("::")[-1].split("<")[0]
            # values in ncu's unit (third column when recorded; older files: Mbyte)
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(parts[2] if len(parts) == 3 else "Mbyte")
            if base == kernel and (cur, parts[0]) not in vals and scale:
                vals[(cur, parts[0])] = float(parts[1].replace(",", "")) * scale
    if not vals:
        return None, None
    return sum(vals.values()), f"{files[-1].relative_to(ROOT)} (first launch of {kernel})"


def roofline(kstats, G, binned, slab=None):
    """Dominant kernel (largest device time in one profiled step) against its
    bound, plus the same figure for every modelled kernel."""
    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm = peaks.get("hbm_gbs")
    if not kstats:
        return None
    model = kernel_model(G, N_SUBJ, shared=("k_solve_shared_tri" in kstats or "k_solve_sep_tri" in kstats))
    slab_share = 1.0
    if slab is not None:  # one rank's share: its rows of the upper triangle
        r0, nr = slab
        share = (sum(G - s for s in range(r0, r0 + nr))) / (G * (G + 1) / 2)
        model = {k: (bnd, work * share) for k, (bnd, work) in model.items()}
        slab_share = 1.0 / share
    total_ms = sum(v[0] for v in kstats.values())
    table = {}
    for name, (ms, cnt) in kstats.items():
        if name not in model:
            continue
        bound, work = model[name]
        secs = ms / 1e3
        if bound == "tensor":
            ach = work / secs / 1e12
            table[name] = {"bound": "tensor", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                           "frac": ach / FP64_PEAK_TFLOPS, "ms": ms, "launches": cnt,
                           "share_of_step": ms / total_ms}
        elif bound == "int8":
            ach = work / secs / 1e12
            table[name] = {"bound": "tensor", "achieved": ach, "peak": INT8_PEAK_TOPS, "unit": "TOP/s (int8)",
                           "frac": ach / INT8_PEAK_TOPS, "ms": ms, "launches": cnt,
                           "share_of_step": ms / total_ms,
                           # the FP64 product it replaces, n G^2 flops over the same time
                           "fp64_equiv_tflops": N_SUBJ * G * G / secs / 1e12 / (slab_share if slab else 1.0)}
        else:
            ach = work / secs / 1e9
            table[name] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                           "frac": ach / hbm if hbm else None, "ms": ms, "launches": cnt,
                           "share_of_step": ms / total_ms}
    dom = max(table, key=lambda k: table[k]["ms"])
    d = dict(table[dom])
    d["kernel"] = dom
    d["traffic"], d["traffic_source"] = ncu_traffic(dom)
    d["algorithmic_per_launch"] = model[dom][1] / table[dom]["launches"]
    d["peak_source"] = ("measured dense int8 peak (cuBLASLt 8192^3, tools/int8_peak.py, profiles/r07_int8_peak.jsonl)"
                        if model[dom][0] == "int8" else
                        "measured FP64 DMMA peak (tools/fp64_peak.cu, profiles/fp64_peak_r01.txt)"
                        if d["bound"] == "tensor" else "MEASURED_PEAKS.json hbm_gbs (measured copy)")
    d["all_kernels"] = table
    return d


if __name__ == "__main__":
    main()
