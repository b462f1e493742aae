#!/usr/bin/env python3
"""Times the CV bandwidth objective (reference
bandwidth.hpp CvObjective / cv_score) on the GPU next to the reference
(oracle/_ref: bandwidth.hpp compiled unchanged, host cores), max_units = 2000.

    python tools/bench_cv.py
"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1510_04439_b200 import api, synth  # noqa: E402


def main():
    from oracle import ref as R
    R.set_threads(os.cpu_count() or 1)
    cases = [
        ("configs[3] sparse masked 64x64 n=2000", lambda: synth.sparse_masked(64, 2000, 0.15), 2000),
        ("configs[2] dense 64x64 n=2000 (8.2 M observations)", lambda: synth.grid_nodes(2, 64, 2000, 0.1), 2000),
    ]
    for name, make, units in cases:
        sd = make()
        targets = [api.CvTarget.Mean, api.CvTarget.DiagPlusNoise]
        if max(sd.offsets[1:] - sd.offsets[:-1]) <= 64:
            targets.append(api.CvTarget.Covariance)
        for t in targets:
            obj = api.CvObjective(sd.dataset(), sd.grid(), t, max_units=units)
            h = api.Bandwidth(sd.h)
            obj(h)  # warm
            reps = []
            for _ in range(3):
                t0 = time.perf_counter()
                got = obj(h)
                reps.append(time.perf_counter() - t0)
            gpu_ms = 1e3 * min(reps)
            # the reference on the same units (dense: a 100-unit sample, scaled)
            ru = units if sd.offsets[-1] < 1_000_000 else 100
            t0 = time.perf_counter()
            want, _ = R.cv_score((sd.axes, sd.mask), sd.offsets, sd.coords, sd.values, t.value, sd.h, max_units=ru)
            cpu_ms = (time.perf_counter() - t0) * 1e3 * units / ru
            line = {"workload": name, "target": t.name, "units": obj.n_units(), "used": obj.last_used,
                    "gpu_ms_per_evaluation": gpu_ms, "cpu_reference_ms_per_evaluation": cpu_ms,
                    "cpu_cores": os.cpu_count(), "cpu_sample_units": ru}
            if ru == units:
                line["rel_diff_vs_reference"] = abs(got - want) / abs(want)
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
