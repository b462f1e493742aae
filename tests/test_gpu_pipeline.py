"""The reference's own fit_pipeline (pipeline.hpp: grid, bandwidths, mean,
diagonal and covariance smoothers, noise variance, eigensolver, FVE
selection, scores) run unchanged against the drop-in headers -- every hot-path
call going to the GPU -- and against the reference alone, from one driver
source (tests/cpp/pipeline_run.cpp, built by __graft_entry__.build() through
tests/cpp/build_harness.py).  Bars: the reference tests' own (eigenvalues
1e-6 relative, test_eigensolve.cpp:349), noise variance and FVE alike, and the
leading scores and eigenfunction to 1e-6."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BIN = Path(__file__).resolve().parent / "cpp" / "_bin"


def _run(name, *args):
    exe = BIN / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (needs the reference sources: __graft_entry__.build())")
    r = subprocess.run([str(exe), *args], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("eig", ["randomized", "dense"])
@pytest.mark.parametrize("sim", ["sim1", "grid2d", "random2d"])
def test_fit_pipeline_dropin_matches_reference(sim, eig):
    got = _run("pipeline_dropin", sim, eig)
    want = _run("pipeline_ref", sim, eig)
    assert got["ok"] and want["ok"]
    assert got["n_components"] == want["n_components"]
    assert got["score_method"] == want["score_method"]
    assert got["h_cov"] == want["h_cov"]
    np.testing.assert_allclose(got["eigenvalues"], want["eigenvalues"], rtol=1e-6, atol=0)
    np.testing.assert_allclose(got["fve"], want["fve"], rtol=1e-6, atol=0)
    assert abs(got["sigma2"] - want["sigma2"]) <= 1e-8 * abs(want["sigma2"])
    assert abs(got["total_variance"] - want["total_variance"]) <= 1e-8 * abs(want["total_variance"])
    a, b = np.asarray(got["phi0"]), np.asarray(want["phi0"])
    m = ~np.isnan(b)
    assert np.array_equal(np.isnan(a), np.isnan(b))
    assert np.max(np.abs(a[m] - b[m])) <= 1e-6 * np.max(np.abs(b[m]))
    sa, sb = np.asarray(got["scores_head"]), np.asarray(want["scores_head"])
    assert np.max(np.abs(sa - sb)) <= 1e-6 * max(1.0, np.max(np.abs(sb)))
