"""The pair-grid SYRK by the Ozaki scheme on the int8 tensor cores
(csrc/ozaki.cu, the default) against the FP64 DMMA SYRK (DFPCA_SYRK=dmma):
pw and pv within 1e-14 of the largest entry (the bound test_pair_grids holds
against the reference; exact zeros are the reference's own business there,
a near-cancelling sum can round to 0 in one FP64 order and not another), the
same NaNs; the covariance within 1e-10 and exactly symmetric.  Grid sizes
that are not multiples of the 128-node tiles, and a NaN observation (its row
and column of the pair grid must come out NaN, as the FP64 sum's do)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DESIGNS = {
    "nodes_10x10": lambda s: s.grid_nodes(2, 10, 25, 0.2),
    "nodes_37x37": lambda s: s.grid_nodes(2, 37, 60, 0.15),
    "random2d_30": lambda s: s.random_points(2, 30, 40, 25, 0.2),
    "random1d_300": lambda s: s.random_points(1, 300, 50, 40, 0.05),
    "random3d_9": lambda s: s.random_points(3, 9, 30, 20, 0.35),
}


def _pairs(api, sd, mode, monkeypatch):
    monkeypatch.setenv("DFPCA_SYRK", mode)
    monkeypatch.setenv("DFPCA_PAIRS", "dense")
    grid = sd.grid()
    b = api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
    pw, pv = api.pair_grids(b)
    h = api.Bandwidth(sd.h)
    mean = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean)
    cov = api.fft_covariance(b, grid, h, mean).values
    return grid.size(), pw, pv, np.asarray(cov)


@pytest.mark.parametrize("case", list(DESIGNS))
def test_ozaki_matches_dmma(case, monkeypatch):
    from paper_1510_04439_b200 import api, synth
    sd = DESIGNS[case](synth)
    G, pw0, pv0, c0 = _pairs(api, sd, "dmma", monkeypatch)
    _, pw1, pv1, c1 = _pairs(api, sd, "ozaki", monkeypatch)
    for a, b in ((pw0, pw1), (pv0, pv1)):
        scale = max(1e-300, float(np.max(np.abs(a))))
        assert np.max(np.abs(a - b)) <= 1e-14 * scale
    fin = np.isfinite(c0)
    assert np.array_equal(fin, np.isfinite(c1))
    assert np.max(np.abs(c0[fin] - c1[fin])) <= 1e-10 * max(1.0, float(np.max(np.abs(c0[fin]))))
    m = c1.reshape(G, G)
    assert np.array_equal(m.view(np.uint64), m.T.view(np.uint64))


def test_ozaki_nan_observation_poisons_its_row_and_column(monkeypatch):
    from paper_1510_04439_b200 import api, synth
    sd = synth.grid_nodes(2, 12, 20, 0.2)
    sd.values = np.array(sd.values, dtype=np.float64, copy=True)
    sd.values[7] = np.nan
    _, pw0, pv0, _ = _pairs(api, sd, "dmma", monkeypatch)
    G, pw1, pv1, _ = _pairs(api, sd, "ozaki", monkeypatch)
    assert np.isnan(pv0).any()
    assert np.array_equal(np.isnan(pv0), np.isnan(pv1))
    assert np.array_equal(np.isnan(pw0), np.isnan(pw1))
    fin = np.isfinite(pv0)
    assert np.max(np.abs(pv0[fin] - pv1[fin])) <= 1e-14 * max(1e-300, float(np.max(np.abs(pv0[fin]))))
