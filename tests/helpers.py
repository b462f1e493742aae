"""Shared comparison metrics, mirroring the reference tests' own metrics."""
import numpy as np


def rel_surface_diff(a, b) -> float:
    """max |a-b| / max(1, |a|, |b|) over finite entries (tests/acceptance.cpp:236-243);
    the NaN (outside) pattern must be identical."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape
    na, nb = np.isnan(a), np.isnan(b)
    assert np.array_equal(na, nb), f"outside pattern differs at {np.count_nonzero(na != nb)} entries"
    m = ~na
    if not m.any():
        return 0.0
    den = np.maximum(1.0, np.maximum(np.abs(a[m]), np.abs(b[m])))
    return float(np.max(np.abs(a[m] - b[m]) / den))


def bit_equal(a, b) -> bool:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def aligned_ise(cv, a, b) -> float:
    """Sign-aligned Riemann ISE of two eigenfunctions (test_eigensolve.cpp)."""
    a = np.asarray(a)
    b = np.asarray(b)
    m = ~np.isnan(a)
    d1 = np.sum((a[m] - b[m]) ** 2) * cv
    d2 = np.sum((a[m] + b[m]) ** 2) * cv
    return float(min(d1, d2))


def max_principal_angle(cv, A, B) -> float:
    """Largest principal angle (radians) between span(A) and span(B), rows
    = functions on the grid, under the Riemann inner product cv * <f, g>
    (SURVEY.md 8(c)); NaN (masked) nodes are dropped."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    m = ~np.isnan(A[0])
    Qa, _ = np.linalg.qr((np.sqrt(cv) * A[:, m]).T)
    Qb, _ = np.linalg.qr((np.sqrt(cv) * B[:, m]).T)
    s = np.linalg.svd(Qa.T @ Qb, compute_uv=False)
    # sin of the largest angle from the projection residual is accurate for small angles
    r = Qb - Qa @ (Qa.T @ Qb)
    sin_max = np.linalg.norm(r, 2)
    return float(np.arcsin(min(1.0, sin_max))) if s.min() > 0.7 else float(np.arccos(max(-1.0, min(1.0, s.min()))))
