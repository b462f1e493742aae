"""TEST INFRASTRUCTURE ONLY -- an independent numpy / pure-Python restatement
of the reference's binned FPCA hot path, for small cases.

It cross-checks the compiled reference (oracle/_ref, via tests/golden/) and
gives the GPU tests a second, library-free checker.  Every function follows
the reference line by line in its evaluation order (file:line relative to
/root/reference/proj/include/dfpca); only tests/ and __graft_entry__.smoke()
import it.
"""
from __future__ import annotations

import math

import numpy as np

# ------------------------------------------------------------------ grid --


def locate_cell(axis, x):
    """surface.hpp:42-66"""
    n = len(axis)
    if x <= axis[0]:
        return 0, 0.0
    if x >= axis[-1]:
        return n - 2, 1.0
    lo, hi = 0, n - 1
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if axis[mid] <= x:
            lo = mid
        else:
            hi = mid
    return lo, (x - axis[lo]) / (axis[lo + 1] - axis[lo])


def strides_of(shape):
    """grid.hpp:48-54"""
    s = [1] * len(shape)
    for k in range(len(shape) - 2, -1, -1):
        s[k] = s[k + 1] * shape[k + 1]
    return s


def linear_bin(axes, offsets, coords, values, mean_path=True, cov_path=True):
    """binning.hpp:82-183, sequential in (sample, observation, corner) order."""
    d = len(axes)
    shape = [len(a) for a in axes]
    st = strides_of(shape)
    G = int(np.prod(shape))
    codes = 3 ** d
    out = dict(mass=np.zeros(G), wvalue=np.zeros(G), wsquare=np.zeros(G),
               diag_mass=np.zeros(G * codes), diag_value=np.zeros(G * codes),
               per_sample=[], sample_sizes=[])
    corners = 1 << d
    for i in range(len(offsets) - 1):
        a, b = int(offsets[i]), int(offsets[i + 1])
        n = b - a
        out["sample_sizes"].append(n)
        mean_w = 1.0 / n if n > 0 else 0.0
        sg = None
        if cov_path and n >= 2:
            sg = dict(sample_index=i, pair_weight=1.0 / (float(n) * float(n - 1)), mass=np.zeros(G),
                      value=np.zeros(G))
            out["per_sample"].append(sg)
        pw = sg["pair_weight"] if sg else 0.0
        for j in range(a, b):
            x = coords[j * d:(j + 1) * d]
            for k in range(d):
                tol = 1e-12 * (axes[k][-1] - axes[k][0])
                if x[k] < axes[k][0] - tol or x[k] > axes[k][-1] + tol:
                    raise ValueError(f"ObservationOutsideGrid: sample {i} observation {j - a}")
            cf = [locate_cell(axes[k], x[k]) for k in range(d)]
            cflat, cmass = [], []
            for c in range(corners):
                m, flat = 1.0, 0
                for k in range(d):
                    up = (c >> k) & 1
                    m *= cf[k][1] if up else (1.0 - cf[k][1])
                    flat += (cf[k][0] + up) * st[k]
                cflat.append(flat)
                cmass.append(m)
            y = float(values[j])
            if mean_path:
                for c in range(corners):
                    f = cflat[c]
                    wm = mean_w * cmass[c]
                    out["mass"][f] += wm
                    out["wvalue"][f] += wm * y
                    out["wsquare"][f] += wm * y * y
            if sg is not None:
                for c in range(corners):
                    sg["mass"][cflat[c]] += cmass[c]
                    sg["value"][cflat[c]] += cmass[c] * y
                for c1 in range(corners):
                    if cmass[c1] == 0.0:
                        continue
                    for c2 in range(corners):
                        if cmass[c2] == 0.0:
                            continue
                        code = 0
                        for k in range(d):
                            code = code * 3 + (((c2 >> k) & 1) - ((c1 >> k) & 1) + 1)
                        band = cflat[c1] * codes + code
                        mm = pw * cmass[c1] * cmass[c2]
                        out["diag_mass"][band] += mm
                        out["diag_value"][band] += mm * y * y
    return out


# ------------------------------------------------------------- smoothers --


def kernel_axis(u, h):
    """kernel.hpp:37-43"""
    z = u / h
    t = 1.0 - z * z
    return 0.75 * t / h if t > 0.0 else 0.0


def taps_for(h, spacing, order):
    """fft_smoother.hpp:199-207"""
    R = int(math.ceil(h / spacing))
    out = np.zeros(2 * R + 1)
    for o in range(-R, R + 1):
        u = -float(o) * spacing
        out[o + R] = kernel_axis(u, h) * u ** order
    return out


def conv_axis(arr, axis, taps):
    """Direct path of AxisConv::run_line (conv.hpp:165-173), zero extension."""
    R = len(taps) // 2
    a = np.moveaxis(arr, axis, -1)
    n = a.shape[-1]
    out = np.zeros_like(a)
    for j in range(n):
        acc = np.zeros(a.shape[:-1])
        for o in range(max(-R, -j), min(R, n - 1 - j) + 1):
            acc = acc + taps[o + R] * a[..., j + o]
        out[..., j] = acc
    return np.moveaxis(out, -1, axis)


def moment_basis(p):
    """local_fit.hpp:34-47: engine orders, constant, e_k, then (k<=l) row-major."""
    eng = [[0] * p]
    for k in range(p):
        o = [0] * p
        o[k] = 1
        eng.append(o)
    for k in range(p):
        for l in range(k, p):
            o = [0] * p
            o[k] += 1
            o[l] += 1
            eng.append(o)
    return eng


def ldlt_solve_local(S, T, p):
    """local_fit.hpp:63-100 with Eigen's LDLT (diagonal pivoting on the
    not-yet-factored diagonal, left-looking, lower storage).  Returns (b0, status)."""
    N = p + 1
    s0, t0 = S[0], T[0]
    if not s0 > 0.0:
        return 0.0, "Empty"
    A = np.zeros((N, N))
    rhs = np.zeros(N)
    A[0, 0] = S[0]
    rhs[0] = T[0]
    q = 1 + p
    for k in range(p):
        A[0, k + 1] = A[k + 1, 0] = S[1 + k]
        rhs[k + 1] = T[1 + k]
        for l in range(k, p):
            A[k + 1, l + 1] = A[l + 1, k + 1] = S[q]
            q += 1
    eps = 1e-10 * np.trace(A)
    A = A + eps * np.eye(N)
    trans = list(range(N))
    ret, fzp = True, False
    for k in range(N):
        piv = k + int(np.argmax(np.abs(np.diag(A)[k:])))
        trans[k] = piv
        if piv != k:
            A[[k, piv], :k] = A[[piv, k], :k]
            A[piv + 1:, [k, piv]] = A[piv + 1:, [piv, k]]
            A[k, k], A[piv, piv] = A[piv, piv], A[k, k]
            for i in range(k + 1, piv):
                A[i, k], A[piv, i] = A[piv, i], A[i, k]
        if k > 0:
            temp = np.diag(A)[:k] * A[k, :k]
            A[k, k] -= A[k, :k] @ temp
            A[k + 1:, k] -= A[k + 1:, :k] @ temp
        akk = A[k, k]
        valid = abs(akk) > 0.0
        if k == 0 and not valid:
            ret = False
            trans = list(range(N))
            break
        if valid:
            A[k + 1:, k] /= akk
        else:
            ret = ret and bool(np.all(A[k + 1:, k] == 0.0))
        if fzp and valid:
            ret = False
        elif not valid:
            fzp = True
    D = np.diag(A).copy()
    ok = ret and np.max(np.abs(D)) > 0.0 and np.min(D) > 0.0 and np.min(np.abs(D)) > 1e-8 * np.max(np.abs(D))
    if ok:
        x = rhs.copy()
        for k in range(N):
            x[k], x[trans[k]] = x[trans[k]], x[k]
        for j in range(N):
            x[j + 1:] -= A[j + 1:, j] * x[j]
        x = np.where(np.abs(D) > np.finfo(float).tiny, x / np.where(D == 0, 1, D), 0.0)
        for j in range(N - 1, -1, -1):
            x[:j] -= A[j, :j] * x[j]
        for k in range(N - 1, -1, -1):
            x[k], x[trans[k]] = x[trans[k]], x[k]
        if np.all(np.isfinite(x)):
            return float(x[0]), "Ok"
    return t0 / s0, "LocalConstant"


def _moments(mass_like, value_like, hs, spacings):
    p = mass_like.ndim
    eng = moment_basis(p)
    S, T = [], []
    for i, o in enumerate(eng):
        a = mass_like
        for k in range(p):
            a = conv_axis(a, k, taps_for(hs[k], spacings[k], o[k]))
        S.append(a)
    for o in eng[:1 + p]:
        a = value_like
        for k in range(p):
            a = conv_axis(a, k, taps_for(hs[k], spacings[k], o[k]))
        T.append(a)
    return np.stack([s.ravel() for s in S], 1), np.stack([t.ravel() for t in T], 1)


def fft_local_linear(axes, mask, binned, h, squares=False):
    """fft_smoother.hpp:498-575 (single block; direct convolution; no ladder)."""
    shape = [len(a) for a in axes]
    sp = [(a[-1] - a[0]) / (len(a) - 1) for a in axes]
    value = binned["wsquare" if squares else "wvalue"].reshape(shape)
    S, T = _moments(binned["mass"].reshape(shape), value, h, sp)
    out = np.full(S.shape[0], np.nan)
    for f in range(S.shape[0]):
        if mask is not None and not mask[f]:
            continue
        b0, st = ldlt_solve_local(S[f], T[f], len(shape))
        if st == "Empty":
            raise ValueError("BandwidthTooSmall")
        out[f] = b0
    return out


def pair_grids(binned, G, shape):
    """PairGridSource::build_into over the full box (fft_smoother.hpp:362-437)."""
    d = len(shape)
    codes = 3 ** d
    pw = np.zeros((G, G))
    pv = np.zeros((G, G))
    for sg in binned["per_sample"]:
        nz = np.flatnonzero(sg["mass"])
        for a in nz:
            for b in nz:
                pw[a, b] += sg["pair_weight"] * sg["mass"][a] * sg["mass"][b]
                pv[a, b] += sg["pair_weight"] * sg["value"][a] * sg["value"][b]
    st = strides_of(shape)
    for u in range(G):
        idx = np.unravel_index(u, shape)
        for code in range(codes):
            dm = binned["diag_mass"][u * codes + code]
            dv = binned["diag_value"][u * codes + code]
            if dm == 0.0 and dv == 0.0:
                continue
            offs, c = [], code
            for _ in range(d):
                offs.append(c % 3 - 1)
                c //= 3
            offs = offs[::-1]
            tt = [idx[k] + offs[k] for k in range(d)]
            if any(t < 0 or t >= shape[k] for k, t in enumerate(tt)):
                continue
            t = sum(tt[k] * st[k] for k in range(d))
            pw[u, t] -= dm
            pv[u, t] -= dv
    return pw, pv


def fft_covariance(axes, mask, binned, h, mean):
    """fft_smoother.hpp:585-744 (single block, direct convolution, no ladder):
    pair grids, 2d-dim moments, solves, centering, symmetrization."""
    shape = [len(a) for a in axes]
    d = len(shape)
    G = int(np.prod(shape))
    sp = [(a[-1] - a[0]) / (len(a) - 1) for a in axes]
    pw, pv = pair_grids(binned, G, shape)
    S, T = _moments(pw.reshape(shape + shape), pv.reshape(shape + shape), list(h) * 2, sp * 2)
    out = np.full(G * G, np.nan)
    for e in range(G * G):
        s, t = divmod(e, G)
        if mask is not None and not (mask[s] and mask[t]):
            continue
        b0, st = ldlt_solve_local(S[e], T[e], 2 * d)
        if st == "Empty":
            raise ValueError("BandwidthTooSmall")
        out[e] = b0
    for a in range(G):
        if mask is not None and not mask[a]:
            continue
        for b in range(G):
            if mask is not None and not mask[b]:
                continue
            out[a * G + b] -= mean[a] * mean[b]
    for a in range(G):
        for b in range(a + 1, G):
            if np.isnan(out[a * G + b]):
                continue
            avg = 0.5 * (out[a * G + b] + out[b * G + a])
            out[a * G + b] = avg
            out[b * G + a] = avg
    return out


# ----------------------------------------------------------------- eigen --

MASK64 = (1 << 64) - 1


def splitmix64(x):
    """rng.hpp:12-17"""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


class MT19937_64:
    """std::mt19937_64 (the engine of RandomStream, rng.hpp:30-33)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & MASK64
        self.idx = 312

    def __call__(self):
        if self.idx >= 312:
            for i in range(312):
                x = (self.mt[i] & 0xFFFFFFFF80000000) | (self.mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[i] = self.mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64


class RandomStream:
    """rng.hpp:30-78 (uniform + cached Box-Muller normal)."""

    def __init__(self, seed):
        self.eng = MT19937_64(splitmix64(seed))
        self.spare = None

    def uniform(self):
        return (float(self.eng() >> 11) + 0.5) * 2.0 ** -53

    def normal(self):
        if self.spare is not None:
            v, self.spare = self.spare, None
            return v
        u1, u2 = self.uniform(), self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        a = 6.283185307179586476925286766559 * u2
        self.spare = r * math.sin(a)
        return r * math.cos(a)


def randomized_eig(axes, mask, cov, q, L_max, seed):
    """matrixize + randomized_eig + finalize (eigensolve.hpp:71-103, 245-279, 148-194)."""
    shape = [len(a) for a in axes]
    G = int(np.prod(shape))
    cv = float(np.prod([(a[-1] - a[0]) / (len(a) - 1) for a in axes]))
    rows = [f for f in range(G) if mask is None or mask[f]]
    M = len(rows)
    Sig = np.asarray(cov).reshape(G, G)[np.ix_(rows, rows)]
    q = min(q, M)
    rng = RandomStream(seed)
    sd = 1.0 / math.sqrt(q)
    om = np.zeros((M, q))
    for j in range(q):
        for i in range(M):
            om[i, j] = sd * rng.normal()
    Y = Sig @ om
    Q, _ = np.linalg.qr(Y)
    small = Q.T @ (Sig @ Q)
    small = 0.5 * (small + small.T)
    w, V = np.linalg.eigh(small)
    tilde = w[::-1]
    lifted = Q @ V[:, ::-1]
    cut = max(0.0, tilde[0]) * 1e-12 if len(tilde) else 0.0
    total = float(sum(t for t in tilde if t > cut)) * cv
    kept, vals = [], []
    for l in range(len(tilde)):
        if len(vals) >= L_max or not tilde[l] > cut:
            break
        v = lifted[:, l].copy()
        for u in kept:
            v -= cv * (u @ v) * u
        nrm = math.sqrt(cv * (v @ v))
        if not nrm > 1e-10:
            continue
        v /= nrm
        s = cv * v.sum()
        if abs(s) < 1e-12 * math.sqrt(cv * v.size):
            nz = np.flatnonzero(v)
            s = v[nz[0]] if nz.size else 0.0
        if s < 0:
            v = -v
        kept.append(v)
        vals.append(tilde[l] * cv)
    funcs = []
    for v in kept:
        f = np.full(G, np.nan)
        f[rows] = v
        funcs.append(f)
    fve = list(np.cumsum(vals) / total) if total > 0 else [1.0] * len(vals)
    return dict(eigenvalues=np.array(vals), eigenfunctions=np.array(funcs), fve=np.array(fve),
                total_variance=total)
