"""GPU: the slab-sharded covariance (csrc/shard.cu) is bit-identical to the
one-device covariance for any rank count (SURVEY.md 8(e) invariance target).

The ranks run as threads of this process on one GPU, each with its own
context and stream, exchanging the schedule's blocks device to device
(LocalTransport); they meet only at host-side barriers, no kernel waits on
another rank.  The NCCL transport moves the same packed blocks between
processes.  The schedule itself is checked between processes on CPU
(tests/test_shard_plan.py).
"""
import numpy as np
import pytest

from helpers import bit_equal

pytestmark = pytest.mark.gpu

CASES = {
    # shared design (closed-form mass moments), d = 2, 4 units of 128 rows
    "2d_nodes": lambda s: s.grid_nodes(2, 32, 60, 0.1),
    # general design (pw and pv both from the SYRK and both exchanged)
    "2d_random": lambda s: s.random_points(2, 24, 80, 40, 0.25),
    "2d_masked_sparse": lambda s: s.sparse_masked(32, 400, 0.3),
    # d = 3: generic tree passes and chunked columns
    "3d_nodes": lambda s: s.grid_nodes(3, 8, 12, 0.3),
    "3d_random": lambda s: s.random_points(3, 8, 30, 40, 0.35),
    # d = 1: one unit of 128 nodes per slab
    "1d_random": lambda s: s.random_points(1, 512, 30, 40, 0.05),
    # 96-node planes: pass kernels above 48 KB of shared memory, launched by
    # concurrent rank threads with different sizes (the attribute must only grow)
    "2d_nodes_96": lambda s: s.grid_nodes(2, 96, 6, 0.1),
}


@pytest.fixture(scope="module")
def api():
    from paper_1510_04439_b200 import api as A
    return A


def _setup(api, sd):
    grid = sd.grid()
    b = api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
    h = api.Bandwidth(sd.h)
    mean = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean)
    return grid, b, h, mean


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_covariance_bit_identical(api, case, world):
    from paper_1510_04439_b200 import synth
    sd = CASES[case](synth)
    grid, b, h, mean = _setup(api, sd)
    one = api.fft_covariance(b, grid, h, mean).values
    many = api.fft_covariance_emulated(b, grid, h, mean, world)
    assert many.rows() == (0, grid.size())
    assert bit_equal(many.values, one), f"{case} x{world}"


def test_sharded_general_path_forced(api, monkeypatch):
    """GridNodes input through the general pair path (pw from the SYRK and
    exchanged as well) -- DFPCA_GENERAL_PAIRS=1."""
    from paper_1510_04439_b200 import synth
    sd = synth.grid_nodes(2, 32, 40, 0.1)
    grid, b, h, mean = _setup(api, sd)
    monkeypatch.setenv("DFPCA_GENERAL_PAIRS", "1")
    one = api.fft_covariance(b, grid, h, mean).values
    many = api.fft_covariance_emulated(b, grid, h, mean, 4)
    assert bit_equal(many.values, one)


@pytest.mark.parametrize("route", ["sparse", "dense"])
def test_sharded_pair_routes(api, route, monkeypatch):
    """Both pair-grid routes on slabs: the sparse one builds every window
    whole (no exchange, idle ranks skip it too), bit-identical to one GPU."""
    from paper_1510_04439_b200 import synth
    monkeypatch.setenv("DFPCA_PAIRS", route)
    sd = synth.sparse_masked(32, 300, 0.3)
    grid, b, h, mean = _setup(api, sd)
    one = api.fft_covariance(b, grid, h, mean).values
    for world in (3, 9):
        many = api.fft_covariance_emulated(b, grid, h, mean, world)
        assert bit_equal(many.values, one), f"{route} x{world}"


def test_sharded_with_idle_ranks(api):
    """More ranks than 128-row units: the surplus ranks hold empty slabs and
    still take part in both exchanges."""
    from paper_1510_04439_b200 import synth
    sd = synth.grid_nodes(2, 12, 30, 0.2)  # G = 144: three 64-row units (rn = 12 -> 16-plane units)
    grid, b, h, mean = _setup(api, sd)
    bounds = api.shard_bounds(12, 12, 3, 5)
    assert sum(1 for r in range(5) if bounds[r] == bounds[r + 1]) >= 3
    one = api.fft_covariance(b, grid, h, mean).values
    many = api.fft_covariance_emulated(b, grid, h, mean, 5)
    assert bit_equal(many.values, one)


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("case", ["nodes_small_h", "masked_sparse"])
def test_sharded_ladder_bit_identical(api, world, case):
    """Empty kernel windows need the enlarged-window ladder
    (fft_smoother.hpp:471-487), whose windows reach past the slab halo: every
    rank takes the same branch and the sharded result is still bit-identical
    to the one-device covariance (whose ladder handles them)."""
    from paper_1510_04439_b200 import synth
    sd = (synth.grid_nodes(2, 16, 20, 0.05) if case == "nodes_small_h"  # h < spacing: empty diagonal windows
          else synth.config(4, n=300, cells=32, h=0.12))                  # sparse masked design (config 4)
    grid, b, h, mean = _setup(api, sd)
    one = api.fft_covariance(b, grid, h, mean).values  # one device: the ladder handles them
    many = api.fft_covariance_emulated(b, grid, h, mean, world)
    assert bit_equal(many.values, one)


def test_single_rank_sharded_entry_is_the_plain_covariance(api):
    from paper_1510_04439_b200 import synth
    sd = synth.grid_nodes(2, 16, 30, 0.2)
    grid, b, h, mean = _setup(api, sd)
    one = api.fft_covariance(b, grid, h, mean).values
    s = api.fft_covariance_sharded(b, grid, h, mean)  # no communicator: one rank
    assert s.rows() == (0, grid.size())
    assert bit_equal(s.values, one)


@pytest.mark.parametrize("case,world", [("2d_nodes", 3), ("2d_masked_sparse", 4), ("3d_nodes", 2),
                                        ("1d_random", 4)])
def test_sharded_randomized_eig_bit_identical(api, case, world):
    """Row-sharded projection (per-rank products with Sigma, all-gathered;
    QR, Rayleigh-Ritz and finalization replicated): every rank returns the
    one-device eigensystem bit for bit."""
    from paper_1510_04439_b200 import synth
    sd = CASES[case](synth)
    grid, b, h, mean = _setup(api, sd)
    M = grid.size() if sd.mask is None else int(np.count_nonzero(sd.mask))
    q, L = min(40, M), 5
    one = api.randomized_eig(api.matrixize(api.fft_covariance(b, grid, h, mean)), q, L, grid, 20260815)
    many, agree = api.fpca_emulated(b, grid, h, mean, world, q, L, 20260815)
    assert agree
    assert bit_equal(many.eigenvalues, one.eigenvalues)
    assert bit_equal(np.concatenate(many.eigenfunctions), np.concatenate(one.eigenfunctions))
    assert many.fve == one.fve and many.total_variance == one.total_variance


def test_nccl_transport_binding(api):
    """The NCCL transport (libnccl loaded at run time) on a one-rank
    communicator: grouped send/recv, all-gather and the max all-reduce move the
    data unchanged.  (Multi-rank NCCL needs one GPU per rank.)"""
    import ctypes as C
    from paper_1510_04439_b200 import _lib
    bad = C.c_int64(-1)
    _lib.check(_lib.lib().dfpca_nccl_selftest(_lib.ctx(), C.byref(bad)))
    assert bad.value == 0
