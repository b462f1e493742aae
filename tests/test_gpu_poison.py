"""The covariance with every t-partial NaN-filled before the t-phase
(DFPCA_POISON=1): the upper-triangle trims of the t-phase and s-phase must
never read an entry that was not written -- any such read would turn the
result into NaN.  Compared with the reference (1e-10) and, for slabs, with
the one-GPU bits."""
import numpy as np
import pytest

from helpers import bit_equal, rel_surface_diff

pytestmark = pytest.mark.gpu

CASES = {
    "2d_nodes_64": lambda s: s.grid_nodes(2, 64, 6, 0.1),
    "2d_nodes_48_wide": lambda s: s.grid_nodes(2, 48, 5, 0.3),
    "2d_random_40": lambda s: s.random_points(2, 40, 20, 30, 0.2),
    "2d_masked_sparse": lambda s: s.sparse_masked(32, 200, 0.25),
    "2d_aniso_small_rn": lambda s: s.random_points(2, 12, 30, 20, 0.3),
    "3d_random": lambda s: s.random_points(3, 8, 20, 30, 0.35),
}


@pytest.mark.parametrize("case", list(CASES))
def test_poisoned_partials_never_read(ref, case, monkeypatch):
    from paper_1510_04439_b200 import api, synth
    monkeypatch.setenv("DFPCA_POISON", "1")
    sd = CASES[case](synth)
    grid = sd.grid()
    b = api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
    h = api.Bandwidth(sd.h)
    mean = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean)
    cov = api.fft_covariance(b, grid, h, mean).values
    r = ref.linear_bin((sd.axes, sd.mask), sd.offsets, sd.coords, sd.values, True, True)
    mr = ref.fft_local_linear(r, (sd.axes, sd.mask), sd.h, 0)
    assert rel_surface_diff(mean.values, mr) <= 1e-10
    cr = ref.fft_covariance(r, (sd.axes, sd.mask), sd.h, mr)
    assert rel_surface_diff(cov, cr) <= 1e-10
    many = api.fft_covariance_emulated(b, grid, h, mean, 3)
    assert bit_equal(many.values, cov)
