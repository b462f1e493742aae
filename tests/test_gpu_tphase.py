"""The fused d = 2 t-phase on zero-padded planes (k_tphase2v, the default)
against the double-buffered unpadded kernel (k_tphase2, DFPCA_TPHASE_2BUF=1):
the same products in the same order, so the covariance must be bit-identical,
for the shared design (value planes only) and the general design (mass
orders too), with and without the upper-triangle trims."""
import numpy as np
import pytest

from helpers import bit_equal

pytestmark = pytest.mark.gpu

CASES = {
    "shared_64_h01": (lambda s: s.grid_nodes(2, 64, 8, 0.1), False),
    "general_64_h01": (lambda s: s.grid_nodes(2, 64, 8, 0.1), True),
    "shared_48_wide": (lambda s: s.grid_nodes(2, 48, 6, 0.3), False),
    "random_40": (lambda s: s.random_points(2, 40, 20, 30, 0.2), False),
    "masked_sparse": (lambda s: s.sparse_masked(32, 200, 0.25), False),
}


def _cov(api, sd, general, monkeypatch, two_buf):
    if two_buf:
        monkeypatch.setenv("DFPCA_TPHASE_2BUF", "1")
    else:
        monkeypatch.delenv("DFPCA_TPHASE_2BUF", raising=False)
    if general:
        monkeypatch.setenv("DFPCA_GENERAL_PAIRS", "1")
    grid = sd.grid()
    b = api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
    h = api.Bandwidth(sd.h)
    mean = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean)
    return np.asarray(api.fft_covariance(b, grid, h, mean).values)


@pytest.mark.parametrize("case", list(CASES))
def test_padded_tphase_bit_identical(case, monkeypatch):
    from paper_1510_04439_b200 import api, synth
    make, general = CASES[case]
    sd = make(synth)
    a = _cov(api, sd, general, monkeypatch, False)
    b = _cov(api, sd, general, monkeypatch, True)
    assert np.isfinite(a).any()
    assert bit_equal(a, b)
