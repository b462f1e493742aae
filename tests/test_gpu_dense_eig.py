"""dense_eig (eigensolve.hpp:205-228) through the hand-written device
eigensolver (csrc/dense_eig.cu: Householder tridiagonalization, Sturm
multisection, inverse iteration, back-transformation) against LAPACK
(numpy.linalg.eigh, the reference's dsyevd family) on matrices of known
spectrum, and against the cuSOLVER path (DFPCA_DENSE_EIG=cusolver) on
smoothed covariances.

Bars (the reference's own test_eigensolve.cpp and test_gpu_scores.py's):
eigenvalues within 1e-10 relative (plus n eps ||A|| for the ones far below
lambda_1, the backward error any dsyevd carries), eigenfunctions by
sign-aligned ISE <= 1e-8 where the relative gap exceeds 1e-3, the pair
orthonormal under the Riemann product to 1e-10, total variance and FVE to
1e-10; repeated eigenvalues by the principal angle of their subspace.
"""
import numpy as np
import pytest

from helpers import aligned_ise, max_principal_angle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_1510_04439_b200 import api as A
    return A


def _matrix(M, spectrum, seed):
    """A symmetric M x M matrix (exactly symmetric in floating point) with
    the given eigenvalues (of the operator: the matrix's are spectrum / cv)."""
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((M, M)))
    cv = 1.0 / M
    lam = np.zeros(M)
    lam[:len(spectrum)] = spectrum
    S = (Q * (lam / cv)) @ Q.T
    S = 0.5 * (S + S.T)
    return S


def _expected(S, L, cv):
    w, U = np.linalg.eigh(S)
    tilde = w[::-1]
    U = U[:, ::-1]
    cut = max(0.0, tilde[0]) * 1e-12
    total = float(np.sum(tilde[tilde > cut])) * cv
    keep = [l for l in range(min(L, len(tilde))) if tilde[l] > cut]
    vals = tilde[keep] * cv
    return vals, [U[:, l] / np.sqrt(cv) for l in keep], total, np.cumsum(vals) / total, tilde * cv


def _run(api, S, L, monkeypatch=None, mode=None):
    M = S.shape[0]
    t = (np.arange(M) + 0.5) / M
    grid = api.EvaluationGrid([list(t)])
    if monkeypatch is not None and mode is not None:
        monkeypatch.setenv("DFPCA_DENSE_EIG", mode)
    surf = api.SurfaceEstimate(grid, api.SurfaceKind.Covariance, values=S.ravel())
    return grid, api.dense_eig(api.matrixize(surf), L, grid)


def _check(got, S, L, cv):
    vals, funcs, total, fve, all_vals = _expected(S, L, cv)
    assert len(got.eigenvalues) == len(vals)
    lam1 = abs(all_vals[0])
    n = S.shape[0]
    for l, (g, w) in enumerate(zip(got.eigenvalues, vals)):
        assert abs(g - w) <= 1e-10 * abs(w) + 4 * n * 2.2e-16 * lam1, (l, g, w)
    for l in range(len(vals)):
        gaps = [abs(all_vals[l] - all_vals[k]) for k in range(n) if k != l]
        if min(gaps) / lam1 > 1e-3:
            assert aligned_ise(cv, got.eigenfunctions[l], funcs[l]) <= 1e-8, l
    F = np.stack(got.eigenfunctions) if got.eigenfunctions else np.zeros((0, n))
    assert np.max(np.abs(cv * F @ F.T - np.eye(len(F))), initial=0.0) <= 1e-10
    assert abs(got.total_variance - total) <= 1e-10 * abs(total)
    assert np.allclose(got.fve, fve, rtol=1e-10, atol=1e-12)
    # the canonical sign: positive integral (eigensolve.hpp's rule)
    for f in F:
        s = cv * np.sum(f)
        if abs(s) > 1e-8:
            assert s > 0


SPECTRA = {
    "decaying": lambda: [10.0 * 0.5 ** l for l in range(30)],
    "with_negatives": lambda: [4.0, 2.0, 1.0, 0.5, -0.3, -1e-3] + [1e-7] * 5,
    "close_pair": lambda: [3.0, 1.0 + 1e-6, 1.0, 0.2, 0.1],
    "rank_two": lambda: [2.0, 0.7],
    "flat_tail": lambda: [5.0, 4.0, 3.0] + [1e-3] * 40,
}


@pytest.mark.parametrize("M", [3, 4, 7, 64, 333, 1000])
@pytest.mark.parametrize("spec", list(SPECTRA))
def test_dense_eig_known_spectrum(api, M, spec):
    s = SPECTRA[spec]()[:M]
    S = _matrix(M, s, seed=M * 7 + len(spec))
    L = min(6, M)
    _, got = _run(api, S, L)
    _check(got, S, L, 1.0 / M)


def test_dense_eig_repeated_eigenvalue_subspace(api):
    M = 256
    S = _matrix(M, [6.0, 2.0, 2.0, 2.0, 0.5], seed=11)
    cv = 1.0 / M
    _, got = _run(api, S, 5)
    vals, funcs, *_ = _expected(S, 5, cv)
    assert np.allclose(got.eigenvalues, vals, rtol=1e-10, atol=0)
    F = np.stack(got.eigenfunctions)
    assert abs(cv * F @ F.T - np.eye(5)).max() <= 1e-10
    assert max_principal_angle(cv, F[1:4], np.stack(funcs[1:4])) <= 1e-8


def test_dense_eig_zero_matrix(api):
    """All eigenvalues zero: nothing passes the cut (lambda_1 = 0 keeps none)."""
    M = 50
    _, got = _run(api, np.zeros((M, M)), 3)
    assert len(got.eigenvalues) == 0
    assert got.total_variance == 0.0


CASES = {
    "sparse_masked_2d": lambda s: s.sparse_masked(24, 150, 0.3),
    "random_1d": lambda s: s.random_points(1, 60, 80, 12, 0.15),
    "nodes_2d": lambda s: s.grid_nodes(2, 30, 40, 0.25),
}


@pytest.mark.parametrize("case", list(CASES))
def test_dense_eig_matches_cusolver(api, case, monkeypatch):
    from paper_1510_04439_b200 import synth
    sd = CASES[case](synth)
    grid = sd.grid()
    b = api.linear_bin(sd.dataset(), grid, api.BinOptions(True, True))
    h = api.Bandwidth(sd.h)
    mean = api.fft_local_linear(b, grid, h, api.MomentTarget.Mean)
    cov = api.fft_covariance(b, grid, h, mean)
    S = api.matrixize(cov)
    L = 8
    monkeypatch.setenv("DFPCA_DENSE_EIG", "cusolver")
    want = api.dense_eig(S, L, grid)
    monkeypatch.setenv("DFPCA_DENSE_EIG", "native")
    got = api.dense_eig(S, L, grid)
    lam = np.asarray(want.eigenvalues)
    assert len(got.eigenvalues) == len(lam)
    assert np.allclose(got.eigenvalues, lam, rtol=1e-10, atol=0)
    cv = grid.cell_volume()
    for l in range(len(lam)):
        gap = min([abs(lam[l] - lam[k]) for k in range(len(lam)) if k != l] + [np.inf]) / lam[0]
        if gap > 1e-3:
            assert aligned_ise(cv, got.eigenfunctions[l], want.eigenfunctions[l]) <= 1e-8
    assert abs(got.total_variance - want.total_variance) <= 1e-10 * abs(want.total_variance)
    assert np.allclose(got.fve, want.fve, rtol=1e-10, atol=1e-12)
