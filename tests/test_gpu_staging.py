"""Large pageable host buffers cross PCIe through the pinned staging slots
(csrc/longfmt.cu copy_h2d / copy_d2h); pinned buffers are copied directly.
Both routes must give the same bytes: binning inputs, surface upload and
download, BinnedData download."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_1510_04439_b200 import api as A
    return A


def _bits(a):
    return np.asarray(a).view(np.uint64)


def test_surface_round_trip_pageable_and_pinned(api):
    from paper_1510_04439_b200 import _lib
    grid = api.EvaluationGrid.uniform([0.0, 0.0], [1.0, 1.0], [41, 39])   # 1599^2 doubles = 20.5 MB
    G = grid.size()
    rng = np.random.default_rng(3)
    vals = rng.standard_normal(G * G)
    vals[::977] = np.nan
    s = api.SurfaceEstimate(grid, api.SurfaceKind.Covariance, values=vals.copy())
    h = s.device_handle()
    back = api.SurfaceEstimate(grid, api.SurfaceKind.Covariance, handle=h)
    s._h = None  # one owner
    assert np.array_equal(_bits(back.values), _bits(vals))
    # the same download into pinned memory
    out = np.empty(G * G)
    assert _lib.pin(out)
    try:
        import ctypes as C
        _lib.check(_lib.lib().dfpca_surface_download(_lib.ctx(), h, out.ctypes.data_as(C.POINTER(C.c_double))))
    finally:
        _lib.unpin(out)
    assert np.array_equal(_bits(out), _bits(vals))


def test_linear_bin_pageable_equals_pinned(api):
    from paper_1510_04439_b200 import _lib, synth
    sd = synth.random_points(2, 24, 300, 4000, 0.2)   # ~1.2 M observations, coords ~19 MB
    grid = sd.grid()
    opt = api.BinOptions(True, True)
    a = api.linear_bin(api.FunctionalDataset.from_csr(2, sd.offsets, sd.coords, sd.values), grid, opt)
    off, co, va = (np.array(x, copy=True) for x in (sd.offsets, sd.coords, sd.values))
    assert co.nbytes > (8 << 20)
    pins = [_lib.pin(x) for x in (off, co, va)]
    try:
        assert all(pins)
        b = api.linear_bin(api.FunctionalDataset.from_csr(2, off, co, va), grid, opt)
        for f in ("mass", "wvalue", "wsquare", "diag_mass", "diag_value"):
            assert np.array_equal(_bits(getattr(a, f)), _bits(getattr(b, f))), f
        for x, y in zip(a.per_sample, b.per_sample):
            assert np.array_equal(_bits(x.mass), _bits(y.mass))
            assert np.array_equal(_bits(x.value), _bits(y.value))
    finally:
        for x in (off, co, va):
            _lib.unpin(x)
