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
