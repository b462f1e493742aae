"""GPU parity: libdfpca_cuda.so (through the Python mirror of the C-ABI) against
the reference implementation compiled unchanged (oracle/_ref) on identical
seeded inputs.

Bars (BASELINE.json north_star):
  * binning: every BinnedData field bit-equal;
  * pair grids: pw entries carrying a self-pair band bit-equal (they decide
    empty kernel windows), everything else within 1e-14 relative (reordered
    FP64 sum over samples);
  * smoothed mean / squares / covariance: max |a-b|/max(1,|a|,|b|) <= 1e-10,
    identical NaN pattern, covariance exactly symmetric;
  * randomized eig (same seed): eigenvalues within 1e-6 relative,
    sign-aligned ISE <= 1e-8, Riemann orthonormality 1e-10.
"""
import numpy as np
import pytest

from helpers import aligned_ise, bit_equal, rel_surface_diff

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def api():
    from paper_1510_04439_b200 import api as A
    return A


def _bin_both(api, ref, sd, mean_path=True, cov_path=True):
    grid = sd.grid()
    data = sd.dataset()
    g = api.linear_bin(data, grid, api.BinOptions(mean_path, cov_path))
    r = ref.linear_bin((sd.axes, sd.mask), sd.offsets, sd.coords, sd.values, mean_path, cov_path)
    return grid, g, r


def _same_or_absent(got, want):
    # the reference leaves fields of a disabled path empty; the oracle binding
    # hands those back zero-filled
    if np.asarray(got).size == 0:
        return not np.any(want)
    return bit_equal(got, want)


def _assert_binned_equal(g, r):
    f = r.fields()
    assert _same_or_absent(g.mass, f["mass"])
    assert _same_or_absent(g.wvalue, f["wvalue"])
    assert _same_or_absent(g.wsquare, f["wsquare"])
    assert g.sample_sizes == [int(x) for x in f["sample_sizes"]]
    G = g.grid.size()
    assert len(g.per_sample) == f["sample_index"].size
    for i, sg in enumerate(g.per_sample):
        assert sg.sample_index == int(f["sample_index"][i])
        assert sg.pair_weight == f["pair_weight"][i]
        assert bit_equal(sg.mass, f["ps_mass"][i * G:(i + 1) * G])
        assert bit_equal(sg.value, f["ps_value"][i * G:(i + 1) * G])
    assert _same_or_absent(g.diag_mass, f["diag_mass"])
    assert _same_or_absent(g.diag_value, f["diag_value"])


# ---------------------------------------------------------------- binning --

@pytest.mark.parametrize("case", ["nodes2d", "random1d", "random2d", "random3d", "sparse_masked", "nodes3d"])
def test_binning_bit_exact(api, ref, case):
    from paper_1510_04439_b200 import synth
    sd = {
        "nodes2d": lambda: synth.grid_nodes(2, 12, 30, 0.2),
        "random1d": lambda: synth.random_points(1, 41, 25, 15, 0.15),
        "random2d": lambda: synth.random_points(2, 13, 20, 25, 0.3),
        "random3d": lambda: synth.random_points(3, 7, 10, 30, 0.4),
        "sparse_masked": lambda: synth.sparse_masked(20, 60, 0.2),
        "nodes3d": lambda: synth.grid_nodes(3, 6, 8, 0.3),
    }[case]()
    grid, g, r = _bin_both(api, ref, sd)
    _assert_binned_equal(g, r)


def test_binning_mean_only_and_empty_samples(api, ref):
    from paper_1510_04439_b200 import synth
    sd = synth.random_points(2, 9, 6, 5, 0.3)
    # make sample 2 empty and sample 4 a single observation
    counts = np.diff(sd.offsets)
    counts[2] = 0
    counts[4] = 1
    keep = np.concatenate([np.arange(sd.offsets[i], sd.offsets[i] + counts[i]) for i in range(counts.size)])
    sd.offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    sd.values = np.ascontiguousarray(sd.values[keep])
    sd.coords = np.ascontiguousarray(sd.coords.reshape(-1, 2)[keep].ravel())
    for mp, cp in [(True, False), (True, True), (False, True)]:
        grid, g, r = _bin_both(api, ref, sd, mp, cp)
        _assert_binned_equal(g, r)


@pytest.mark.parametrize("chunk", ["1", "37", "1000"])
@pytest.mark.parametrize("case", ["nodes2d", "random2d", "empty_samples"])
def test_binning_chunked_bit_exact(api, ref, case, chunk, monkeypatch):
    """Sample-aligned chunks (copy of chunk c + 1 overlapping the binning of
    chunk c) with carry-in sums: still bit-identical to the reference."""
    from paper_1510_04439_b200 import synth
    monkeypatch.setenv("DFPCA_BIN_CHUNK_OBS", chunk)
    sd = {"nodes2d": lambda: synth.grid_nodes(2, 12, 30, 0.2),
          "random2d": lambda: synth.random_points(2, 13, 40, 25, 0.3),
          "empty_samples": lambda: synth.random_points(2, 9, 30, 5, 0.3)}[case]()
    if case == "empty_samples":
        counts = np.diff(sd.offsets)
        counts[[0, 7, 8, 29]] = 0
        keep = np.concatenate([np.arange(sd.offsets[i], sd.offsets[i] + counts[i]) for i in range(counts.size)])
        sd.offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        sd.values = np.ascontiguousarray(sd.values[keep])
        sd.coords = np.ascontiguousarray(sd.coords.reshape(-1, 2)[keep].ravel())
    grid, g, r = _bin_both(api, ref, sd)
    _assert_binned_equal(g, r)
    # an observation outside the hull in a later chunk: same error, context reusable
    bad = sd.dataset()
    last = max(i for i, smp in enumerate(bad.samples) if smp.n_obs() > 0)
    bad.samples[last].coords = np.array(bad.samples[last].coords, copy=True)
    bad.samples[last].coords[-1] = 7.0
    bad.invalidate()
    with pytest.raises(api.Error) as ei:
        api.linear_bin(bad, grid)
    assert ei.value.name() == "ObservationOutsideGrid"
    _assert_binned_equal(api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True)), r)


def test_binning_boundary_and_outside(api):
    grid = api.EvaluationGrid.uniform([0.0], [1.0], [5])
    data = api.FunctionalDataset(1, [api.Sample("a", np.array([0.0, 1.0, 0.125]), np.array([1.0, 2.0, 3.0]))])
    b = api.linear_bin(data, grid)
    # boundary nodes get full mass; 0.125 splits 0.5/0.5 between nodes 0 and 1
    w = 1.0 / 3.0
    assert np.allclose(b.mass, [w + 0.5 * w, 0.5 * w, 0, 0, w], rtol=0, atol=1e-15)
    bad = api.FunctionalDataset(1, [api.Sample("ok", np.array([0.5]), np.array([1.0])),
                                    api.Sample("bad id", np.array([0.2, 1.5]), np.array([1.0, 2.0]))])
    with pytest.raises(api.Error) as ei:
        api.linear_bin(bad, grid)
    assert ei.value.name() == "ObservationOutsideGrid"
    assert "'bad id' observation 1" in str(ei.value)


# ------------------------------------------------------------- pair grids --

@pytest.mark.parametrize("case", ["nodes2d", "random2d", "random1d"])
def test_pair_grids(api, ref, case):
    from paper_1510_04439_b200 import synth
    sd = {"nodes2d": lambda: synth.grid_nodes(2, 10, 25, 0.2),
          "random2d": lambda: synth.random_points(2, 9, 30, 12, 0.3),
          "random1d": lambda: synth.random_points(1, 21, 12, 7, 0.2)}[case]()
    grid, g, r = _bin_both(api, ref, sd)
    pw, pv = api.pair_grids(g)
    rpw, rpv = ref.pair_grids(r)
    f = r.fields()
    band = (f["diag_mass"] != 0) | (f["diag_value"] != 0)
    # entries carrying a band: bit-equal
    G = grid.size()
    codes = 3 ** grid.dim()
    shape = grid.shape()
    for e in np.flatnonzero(band):
        u, code = divmod(int(e), codes)
        offs = []
        for k in range(grid.dim() - 1, -1, -1):
            offs.append(code % 3 - 1)
            code //= 3
        offs = offs[::-1]
        idx = np.unravel_index(u, shape)
        tt = [idx[k] + offs[k] for k in range(grid.dim())]
        if any(t < 0 or t >= shape[k] for k, t in enumerate(tt)):
            continue
        t = int(np.ravel_multi_index(tt, shape))
        assert pw[u * G + t] == rpw[u * G + t]  # exact: decides empty windows
        assert abs(pv[u * G + t] - rpv[u * G + t]) <= 1e-14 * max(1e-300, np.max(np.abs(rpv)))
    scale_w = max(1e-300, np.max(np.abs(rpw)))
    scale_v = max(1e-300, np.max(np.abs(rpv)))
    assert np.max(np.abs(pw - rpw)) <= 1e-14 * scale_w
    assert np.max(np.abs(pv - rpv)) <= 1e-14 * scale_v
    assert np.array_equal(pw == 0, rpw == 0)


@pytest.mark.parametrize("case", ["sparse_masked", "random2d", "random1d", "random3d"])
def test_pair_grids_sparse_route_bit_exact(api, ref, case, monkeypatch):
    """The sparse route (per-sample nonzeros, (s, t) records sorted stably,
    terms added in sample order, then the band) reproduces the reference's
    pair grids bit for bit -- both of them, every entry."""
    from paper_1510_04439_b200 import synth
    monkeypatch.setenv("DFPCA_PAIRS", "sparse")
    sd = {"sparse_masked": lambda: synth.sparse_masked(24, 150, 0.3),
          "random2d": lambda: synth.random_points(2, 11, 25, 12, 0.3),
          "random1d": lambda: synth.random_points(1, 21, 12, 7, 0.2),
          "random3d": lambda: synth.random_points(3, 5, 10, 8, 0.4)}[case]()
    grid, g, r = _bin_both(api, ref, sd)
    pw, pv = api.pair_grids(g)
    rpw, rpv = ref.pair_grids(r)
    assert bit_equal(pw, rpw) and bit_equal(pv, rpv)


@pytest.mark.parametrize("route", ["sparse", "dense"])
@pytest.mark.parametrize("case", ["2d_random", "2d_masked_sparse", "1d"])
def test_covariance_both_pair_routes(api, ref, case, route, monkeypatch):
    from paper_1510_04439_b200 import synth
    monkeypatch.setenv("DFPCA_PAIRS", route)
    sd = COV_CASES[case](synth)
    grid, g, r = _bin_both(api, ref, sd, True, True)
    h = api.Bandwidth(sd.h)
    mean_r = ref.fft_local_linear(r, (sd.axes, sd.mask), sd.h, 0)
    mean_g = api.fft_local_linear(g, grid, h, api.MomentTarget.Mean)
    cov_g = api.fft_covariance(g, grid, h, mean_g).values
    cov_r = ref.fft_covariance(r, (sd.axes, sd.mask), sd.h, mean_r)
    assert rel_surface_diff(cov_g, cov_r) <= TOL


def test_pair_grids_two_observations_exact(api):
    # tests/test_fft_smoother.cpp:161-186
    grid = api.EvaluationGrid.uniform([0.0], [1.0], [5])
    data = api.FunctionalDataset(1, [api.Sample("a", np.array([0.25, 0.75]), np.array([2.0, 5.0]))])
    b = api.linear_bin(data, grid, api.BinOptions(True, True))
    pw, pv = api.pair_grids(b)
    for s in range(5):
        for t in range(5):
            if (s, t) in ((1, 3), (3, 1)):
                assert abs(pw[s * 5 + t] - 0.5) <= 0.5e-15 and abs(pv[s * 5 + t] - 5.0) <= 5e-15
            else:
                assert pw[s * 5 + t] == 0.0 and pv[s * 5 + t] == 0.0


# --------------------------------------------------------------- smoothers --

MEAN_CASES = {
    "1d_nodes": lambda s: s.random_points(1, 41, 25, 15, 0.15, uniform_grid=True),
    "1d_fft_taps": lambda s: s.random_points(1, 101, 15, 25, 0.2),  # 41 taps: reference FFT path
    "2d_aniso": lambda s: s.random_points(2, 17, 20, 20, 0.3),
    "2d_nodes": lambda s: s.grid_nodes(2, 16, 20, 0.14),
    "3d_nodes": lambda s: s.grid_nodes(3, 8, 6, 0.3),
    "masked": lambda s: s.sparse_masked(24, 40, 0.25),
    # wide windows: radius 27 / 40 run the zero-padded radius-32 / 48 kernels
    "1d_wide_r32": lambda s: s.random_points(1, 61, 15, 20, 0.45),
    "1d_wide_r48": lambda s: s.random_points(1, 101, 15, 25, 0.4),
    # 48-node axis: 48 KB dynamic + static shared memory needs the opt-in
    "2d_n48_wide": lambda s: s.grid_nodes(2, 48, 4, 0.6),
}


@pytest.mark.parametrize("case", list(MEAN_CASES))
@pytest.mark.parametrize("target", [0, 1])
def test_local_linear(api, ref, case, target):
    from paper_1510_04439_b200 import synth
    sd = MEAN_CASES[case](synth)
    grid, g, r = _bin_both(api, ref, sd, True, False)
    h = api.Bandwidth(sd.h)
    got = api.fft_local_linear(g, grid, h, api.MomentTarget(target)).values
    want = ref.fft_local_linear(r, (sd.axes, sd.mask), sd.h, target)
    assert rel_surface_diff(got, want) <= TOL


COV_CASES = {
    "1d": lambda s: s.random_points(1, 26, 30, 8, 0.2),
    "1d_fft_taps": lambda s: s.random_points(1, 61, 12, 10, 0.3),
    "1d_nodes": lambda s: s.grid_nodes(1, 40, 30, 0.1),
    "2d_nodes": lambda s: s.grid_nodes(2, 12, 25, 0.2),
    # h < spacing: only the centre tap is positive, so the diagonal windows of
    # the shared design are empty and go through the fallback ladder
    "2d_nodes_narrow": lambda s: s.grid_nodes(2, 8, 20, 0.1),
    "2d_random": lambda s: s.random_points(2, 10, 40, 15, 0.3),
    "2d_masked_sparse": lambda s: s.sparse_masked(14, 120, 0.3),
    "3d_nodes": lambda s: s.grid_nodes(3, 5, 10, 0.45),
    "1d_wide_r32": lambda s: s.random_points(1, 61, 12, 10, 0.5),
    "2d_wide_r32": lambda s: _narrow_second_axis(s.random_points(2, 26, 30, 20, 1.0), 6, 0.3),
}


def _narrow_second_axis(sd, cells, h):
    """Anisotropic variant: axis 2 coarsened to `cells` nodes and bandwidth h
    (axis 1 keeps its wide window, radius 25 -> the radius-32 kernels)."""
    sd.axes = [sd.axes[0], [float(i) / float(cells - 1) for i in range(cells)]]
    sd.h = [sd.h[0], h]
    return sd


@pytest.mark.parametrize("case", list(COV_CASES))
def test_covariance(api, ref, case):
    from paper_1510_04439_b200 import synth
    sd = COV_CASES[case](synth)
    grid, g, r = _bin_both(api, ref, sd, True, True)
    h = api.Bandwidth(sd.h)
    mean_g = api.fft_local_linear(g, grid, h, api.MomentTarget.Mean)
    mean_r = ref.fft_local_linear(r, (sd.axes, sd.mask), sd.h, 0)
    assert rel_surface_diff(mean_g.values, mean_r) <= TOL
    cov_g = api.fft_covariance(g, grid, h, mean_g).values
    cov_r = ref.fft_covariance(r, (sd.axes, sd.mask), sd.h, mean_r)
    assert rel_surface_diff(cov_g, cov_r) <= TOL
    G = grid.size()
    M = cov_g.reshape(G, G)
    fin = ~np.isnan(M)
    assert np.array_equal(M[fin], M.T[fin])  # exact symmetry (test_fft_smoother.cpp:154-158)


@pytest.mark.parametrize("dim,cells,n,h", [(1, 50, 20, 0.1), (2, 12, 25, 0.2), (3, 5, 8, 0.45)])
def test_shared_design_closed_form_matches_general_path(api, dim, cells, n, h, monkeypatch):
    """GridNodes designs take the closed-form mass moments (k_solve_shared);
    DFPCA_GENERAL_PAIRS=1 forces the pair-grid convolution path on the same
    input.  Both must agree to the parity bar and the shared path must be the
    one that ran."""
    from paper_1510_04439_b200 import _lib, synth
    sd = synth.grid_nodes(dim, cells, n, h)
    grid = sd.grid()
    b = api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
    hh = api.Bandwidth(sd.h)
    mean = api.fft_local_linear(b, grid, hh, api.MomentTarget.Mean)
    _lib.profile(True)
    fast = api.fft_covariance(b, grid, hh, mean).values
    names = set(_lib.kernel_stats())
    _lib.profile(False)
    assert any(k.startswith(("k_solve_shared", "k_solve_sep")) for k in names), names
    monkeypatch.setenv("DFPCA_GENERAL_PAIRS", "1")
    _lib.profile(True)
    general = api.fft_covariance(b, grid, hh, mean).values
    names = set(_lib.kernel_stats())
    _lib.profile(False)
    assert not any(k.startswith("k_solve_shared") for k in names), names
    assert rel_surface_diff(fast, general) <= TOL


def test_block_plans_are_invariant(api):
    from paper_1510_04439_b200 import synth
    sd = synth.random_points(1, 101, 15, 25, 0.2)
    grid = sd.grid()
    b = api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
    h = api.Bandwidth([0.2])
    one = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean, api.single_block_plan(grid, h)).values
    four = api.blockwise_apply(api.make_block_plan(grid, h, 4), b, grid, h, api.MomentTarget.Mean).values
    assert bit_equal(one, four)


def test_plan_and_input_errors(api):
    from paper_1510_04439_b200 import synth
    sd = synth.random_points(1, 101, 5, 30, 0.2)
    grid = sd.grid()
    b = api.linear_bin(sd.dataset(), grid)
    h = api.Bandwidth([0.2])
    plan = api.make_block_plan(grid, h, 2)
    plan.halo[0] -= 1
    with pytest.raises(api.Error) as e:
        api.fft_local_linear(b, grid, h, api.MomentTarget.Mean, plan)
    assert e.value.name() == "HaloTooSmall"
    with pytest.raises(api.Error) as e:
        api.fft_local_linear(b, grid, h, api.MomentTarget.Mean, api.make_block_plan(grid, h, 6))
    assert e.value.name() == "BlockTooSmall"
    uneven = api.EvaluationGrid([[0.0, 0.1, 0.25, 0.6, 1.0]])
    tiny = api.FunctionalDataset(1, [api.Sample("a", np.array([0.1, 0.6]), np.array([1.0, 2.0]))])
    ub = api.linear_bin(tiny, uneven)
    with pytest.raises(api.Error) as e:
        api.fft_local_linear(ub, uneven, api.Bandwidth([0.5]), api.MomentTarget.Mean)
    assert e.value.name() == "GridNotEquispaced"
    solo = api.FunctionalDataset(1, [api.Sample("one", np.array([0.5]), np.array([1.0]))])
    sb = api.linear_bin(solo, grid, api.BinOptions(True, True))
    mean = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean)
    with pytest.raises(api.Error) as e:
        api.fft_covariance(sb, grid, h, mean)
    assert e.value.name() == "NoPairs"
    with pytest.raises(api.Error) as e:
        api.fft_local_linear(b, grid, api.Bandwidth([2.0]), api.MomentTarget.Mean)
    assert e.value.name() == "InvalidBandwidth"


def test_impulse_and_constant(api):
    # tests/test_fft_smoother.cpp:60-100
    grid = api.EvaluationGrid.uniform([0.0], [1.0], [21])
    y = 2.75
    mass = np.zeros(21)
    wv = np.zeros(21)
    ws = np.zeros(21)
    mass[10], wv[10], ws[10] = 1.0, y, y * y
    b = api.BinnedData.from_host(grid, mass=mass, wvalue=wv, wsquare=ws, sample_sizes=[1])
    est = api.fft_local_linear(b, grid, api.Bandwidth([1.0]), api.MomentTarget.Mean).values
    assert np.max(np.abs(est - y)) <= 1e-10
    rng = np.random.default_rng(3)
    samples = [api.Sample(str(i), 2.0 * rng.random(12), np.full(12, -1.5)) for i in range(8)]
    g2 = api.EvaluationGrid.uniform([0.0], [2.0], [33])
    b2 = api.linear_bin(api.FunctionalDataset(1, samples), g2)
    est2 = api.fft_local_linear(b2, g2, api.Bandwidth([0.4]), api.MomentTarget.Mean).values
    # Catch::Approx(-1.5).margin(1e-10) also allows the default relative
    # epsilon of 100 float ulps (the ridge biases b0 by ~1e-10 cond)
    assert np.all(np.abs(est2 + 1.5) <= np.maximum(1e-10, 1.5 * 100 * np.finfo(np.float32).eps))


def test_empty_window_ladder(api, ref):
    # two far-apart clusters: nodes between them have empty windows at h and
    # are recovered by the 1.5x enlargements (fft_smoother.hpp:471-487)
    grid_axes = [[i / 40.0 for i in range(41)]]
    rng = np.random.default_rng(5)
    coords = np.concatenate([rng.random(30) * 0.2, 0.8 + rng.random(30) * 0.2])
    values = np.sin(coords * 6) + rng.standard_normal(60) * 0.1
    offsets = np.array([0, 20, 40, 60], dtype=np.int64)
    from paper_1510_04439_b200.synth import SynthData
    sd = SynthData(1, grid_axes, None, offsets, coords, values, [0.18])
    grid, g, r = _bin_both(api, ref, sd, True, True)
    h = api.Bandwidth(sd.h)
    got = api.fft_local_linear(g, grid, h, api.MomentTarget.Mean).values
    want = ref.fft_local_linear(r, (sd.axes, None), sd.h, 0)
    assert rel_surface_diff(got, want) <= TOL
    # too narrow for the ladder: BandwidthTooSmall
    with pytest.raises(api.Error) as e:
        api.fft_local_linear(g, grid, api.Bandwidth([0.05]), api.MomentTarget.Mean)
    assert e.value.name() == "BandwidthTooSmall"
    with pytest.raises(ref.RefError) as e2:
        ref.fft_local_linear(r, (sd.axes, None), [0.05], 0)
    assert e2.value.name() == "BandwidthTooSmall"


# ------------------------------------------------------------------ eigen --

def _spectral_cov(grid_n=200, lam=(5.0, 2.0, 0.5)):
    t = (np.arange(grid_n) + 0.5) / grid_n
    seeds = [1.0 + t, np.sin(2 * np.pi * t), np.cos(5 * np.pi * t) + 0.3 * t]
    cv = 1.0 / grid_n
    phi = []
    for s in seeds[:len(lam)]:
        v = s.copy()
        for u in phi:
            v -= cv * np.dot(u, v) * u
        v /= np.sqrt(cv * np.dot(v, v))
        phi.append(v)
    cov = sum(l * np.outer(p, p) for l, p in zip(lam, phi))
    return [list(t)], cov.ravel()


@pytest.mark.parametrize("q,L", [(10, 3), (99, 3), (3, 3)])
def test_randomized_eig(api, ref, q, L):
    axes, cov = _spectral_cov()
    grid = api.EvaluationGrid(axes)
    surf = api.SurfaceEstimate(grid, api.SurfaceKind.Covariance, values=cov)
    S = api.matrixize(surf)
    got = api.randomized_eig(S, q, L, grid, 20260815)
    want = ref.randomized_eig((axes, None), cov, q, L, 20260815)
    dense = ref.dense_eig((axes, None), cov, L)
    cv = grid.cell_volume()
    assert len(got.eigenvalues) == len(want["eigenvalues"]) == L
    for l in range(L):
        assert abs(got.eigenvalues[l] - want["eigenvalues"][l]) <= 1e-6 * abs(want["eigenvalues"][l])
        assert abs(got.eigenvalues[l] - dense["eigenvalues"][l]) <= 1e-6 * abs(dense["eigenvalues"][l])
        assert aligned_ise(cv, got.eigenfunctions[l], want["eigenfunctions"][l]) < 1e-8
        # canonical sign must agree exactly in sign
        assert np.dot(got.eigenfunctions[l], want["eigenfunctions"][l]) > 0
    for a in range(L):
        for b in range(L):
            d = cv * np.dot(got.eigenfunctions[a], got.eigenfunctions[b])
            assert abs(d - (1.0 if a == b else 0.0)) <= 1e-10
    assert np.allclose(got.fve, want["fve"], rtol=1e-6, atol=0)
    res = api.eig_residuals(S, got, grid)
    assert all(r < 1e-8 * got.eigenvalues[0] for r in res)


def test_randomized_eig_reproducible_and_errors(api):
    axes, cov = _spectral_cov(60, (3.0, 1.0))
    grid = api.EvaluationGrid(axes)
    S = api.matrixize(api.SurfaceEstimate(grid, api.SurfaceKind.Covariance, values=cov))
    a = api.randomized_eig(S, 8, 2, grid, 7)
    b = api.randomized_eig(S, 8, 2, grid, 7)
    assert a.eigenvalues == b.eigenvalues
    for x, y in zip(a.eigenfunctions, b.eigenfunctions):
        assert bit_equal(x, y)
    with pytest.raises(api.Error) as e:
        api.randomized_eig(S, 1, 2, grid, 1)
    assert e.value.name() == "SketchTooSmall"
    assert api.default_sketch_size(3, 1000) == 99
    assert api.default_sketch_size(60, 1000) == 130
    assert api.default_sketch_size(3, 40) == 40


def test_masked_eig(api, ref):
    from paper_1510_04439_b200 import synth
    sd = synth.sparse_masked(12, 200, 0.3)
    grid, g, r = _bin_both(api, ref, sd, True, True)
    h = api.Bandwidth(sd.h)
    mean = api.fft_local_linear(g, grid, h, api.MomentTarget.Mean)
    cov = api.fft_covariance(g, grid, h, mean)
    S = api.matrixize(cov)
    got = api.randomized_eig(S, 40, 4, grid, 11)
    want = ref.randomized_eig((sd.axes, sd.mask), cov.values, 40, 4, 11)
    cv = grid.cell_volume()
    for l in range(len(want["eigenvalues"])):
        assert abs(got.eigenvalues[l] - want["eigenvalues"][l]) <= 1e-6 * abs(want["eigenvalues"][0])
        assert np.array_equal(np.isnan(got.eigenfunctions[l]), np.isnan(want["eigenfunctions"][l]))
