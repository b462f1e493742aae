#!/usr/bin/env python3
"""The reference's FPCA core on the host, stage by stage (the StageClock of
pipeline.hpp:143-165 over the stages of fit_pipeline, pipeline.hpp:308-340),
at set_max_threads(1) and at set_max_threads(nproc) (SURVEY.md
8(d)): configs[2] (d=2 64^2, n=2000, h=0.1, inputs from the reference's own
generator), randomized_eig q=99, L=20.  One JSON line per thread count.

    python tools/time_reference_stages.py [--threads 1,16] [--n 2000]
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", default=f"1,{os.cpu_count() or 1}")
    ap.add_argument("--n", type=int, default=bench.N_SUBJ)
    a = ap.parse_args()
    bench.N_SUBJ = a.n
    sd = bench.make_data()
    for th in [int(x) for x in a.threads.split(",")]:
        t, eig = bench.reference_fpca(sd, th)
        print(json.dumps({"threads": th, "cores": os.cpu_count(), "n": a.n,
                          "stages_ms": {k: round(v * 1e3, 1) for k, v in t.items()},
                          "total_ms": round(sum(t.values()) * 1e3, 1),
                          "eig_top3": [float(x) for x in eig["eigenvalues"][:3]]}), flush=True)


if __name__ == "__main__":
    main()
