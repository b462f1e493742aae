// Binned local-linear smoothers on the device: the d-dimensional mean /
// squares smoother (reference fft_local_linear, fft_smoother.hpp:498-575) and
// the 2d-dimensional covariance smoother (fft_covariance, :585-744).
//
// Moment engine.  The reference runs one full separable convolution per
// moment multi-index (nm + nl engines, fft_smoother.hpp:191-230, 639-646).
// Convolution is linear and the stencils are products of per-axis taps
// K(u) u^order, so the device factors the engines as a tree over the axes:
// every pass reads one partial once and emits all orders the remaining budget
// allows (|r| <= 2 for S, <= 1 for T).  The 2d axes of the covariance are
// split into t-axes (contiguous) and s-axes:
//   phase T: t-axis passes over row chunks of the pair grids, writing the
//            t-partials (multi-indices on the t axes only);
//   phase S: s-axis passes over column chunks of the t-partials, writing the
//            final moments of one chunk, followed by the per-node solve.
// The mean smoother is the same machinery with every axis a "t-axis".
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <array>
#include <functional>
#include <memory>
#include <cmath>
#include <cstdlib>
#include <map>
#include <string>

#include "conv.cuh"
#include "solve.cuh"

namespace dfpca_gpu {

DevGrid upload_grid_axes(dfpca_context* ctx, const Grid& g, DevBuf<double>& storage);
}  // namespace dfpca_gpu
#include "pairs.cuh"
#include "shard_exec.hpp"
namespace dfpca_gpu {

namespace {

using Orders = std::array<int, kMaxP>;

struct Basis {
  int p = 0;
  int nm = 0, nl = 0;
  std::vector<Orders> engine;  // engine index -> per-axis orders (local_fit.hpp:34-47)
  explicit Basis(int vars) : p(vars) {
    nm = 1 + p + p * (p + 1) / 2;
    nl = 1 + p;
    engine.assign(nm, Orders{});
    for (int k = 0; k < p; ++k) engine[1 + k][k] = 1;
    for (int k = 0; k < p; ++k)
      for (int l = k; l < p; ++l) {
        Orders o{};
        o[k] += 1;
        o[l] += 1;
        engine[quad_index(p, k, l)] = o;
      }
  }
  int find(const Orders& o) const {
    for (int i = 0; i < nm; ++i)
      if (engine[i] == o) return i;
    return -1;
  }
};

int order_sum(const Orders& o) {
  int s = 0;
  for (int v : o) s += v;
  return s;
}

// Per-axis taps for orders 0..2 (MomentEngineBank::taps_for,
// fft_smoother.hpp:199-207), computed on the host with std::pow so the taps
// are bit-identical to the reference's.
struct AxisTaps {
  int R = 0;
  std::vector<double> t[3];
};

AxisTaps make_taps(double h, double spacing) {
  AxisTaps a;
  a.R = static_cast<int>(std::ceil(h / spacing));
  for (int order = 0; order < 3; ++order) {
    a.t[order].assign(2 * a.R + 1, 0.0);
    for (int o = -a.R; o <= a.R; ++o) {
      const double u = -static_cast<double>(o) * spacing;
      a.t[order][o + a.R] = kernel_axis_value(u, h) * std::pow(u, order);
    }
  }
  return a;
}

// A partial array of the tree: orders used so far and where it lives.
struct Partial {
  Orders ord{};
  int budget_max = 2;  // 2: mass-like (S), 1: value-like (T)
  DevBuf<double>* buf = nullptr;
  double* ptr = nullptr;
};

// Runs passes for a list of axes (processed in the given order) over a chunk
// of `rows` contiguous outer rows; every array in the chunk has shape
// [rows][shape[ax_first..]] flattened.  `leaf_ptr` maps a finished partial to
// the destination pointer of its last pass (or nullptr to allocate).
struct ChunkDims {
  i64 rows;                // leading extent (outer rows of the chunk)
  std::vector<i64> shape;  // extents of the axes of this phase, in memory order
  i64 tail;                // trailing contiguous extent after these axes
  // upper-triangle restriction (View::tri) for the passes of tree level i
  std::vector<int> tri;
  View tri_params{};
  // output window [win_lo, win_hi) along view axis win_k (the s1 pass of a
  // covariance slab); win_k < 0: none
  int win_k = -1;
  i64 win_lo = 0, win_hi = -1;
  // s-phase order s1, then the in-plane axes: the first pass reads roots
  // whose axis is the outermost memory dimension ([s1][rest][cols]) and
  // writes compact [s1][rest][cols] buffers; with a window on axis 0 the
  // later passes cover only the written planes [win_lo, win_hi)
  bool axis0_first = false;
};

View make_view(double* p, const ChunkDims& cd, int k, i64 row_stride_override = -1) {
  // Axis k of cd.shape; memory is [rows][shape...][tail].
  i64 before = cd.rows;
  for (int a = 0; a < k; ++a) before *= cd.shape[a];
  i64 after = cd.tail;
  for (std::size_t a = k + 1; a < cd.shape.size(); ++a) after *= cd.shape[a];
  View v;
  v.p = p;
  v.outer = before;
  v.n = cd.shape[k];
  v.inner = after;
  v.js = after;
  v.os = row_stride_override >= 0 ? row_stride_override : cd.shape[k] * after;
  return v;
}

}  // namespace

// ---------------------------------------------------------------------------
// Solve kernel over a chunk of points with compact moment arrays.
struct MomPtrs {
  const double* S[kMaxNm];
  const double* T[kMaxNl];
};

struct SolveGeom {
  i64 npts;        // points in the chunk
  i64 tc;          // chunk width (columns); point e -> (e / tc, t0 + e % tc)
  i64 t0;
  i64 gt;          // full column extent (t grid size); 1-D mean: gt = tc = G
  int cov;         // 1: mask both s and t nodes
  int upper;       // covariance: solve only s <= t (the rest is mirrored)
  const std::uint8_t* mask;  // device mask (nullable)
  const double* mean;        // covariance: centered later; unused here
  // covariance slab (tiled solve only): moment rows [row_lo, npts / tc) are
  // solved; local row r is global s node r + row0 and lands in out row
  // r + row0 - out_row0
  i64 row_lo = 0;
  i64 row0 = 0;
  i64 out_row0 = 0;
};

template <int N>
__global__ void __launch_bounds__(128) k_solve(MomPtrs mp, SolveGeom g, double* __restrict__ out,
                                               unsigned long long* __restrict__ empty_count,
                                               i64* __restrict__ empty_list, i64 list_cap) {
  pdl_wait();
  constexpr int p = N - 1;
  constexpr int nm = 1 + p + p * (p + 1) / 2;
  constexpr int nl = 1 + p;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < g.npts;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 row = e / g.tc;
    const i64 col = g.t0 + e % g.tc;
    const i64 dst = g.cov ? row * g.gt + col : col + row * g.gt;
    if (g.upper && row > col) continue;
    bool inside = true;
    if (g.mask) inside = g.cov ? (g.mask[row] != 0 && g.mask[col] != 0) : (g.mask[dst] != 0);
    if (!inside) {
      out[dst] = __longlong_as_double(0x7ff8000000000000ll);
      continue;
    }
    double S[nm], T[nl];
#pragma unroll
    for (int i = 0; i < nm; ++i) S[i] = mp.S[i][e];
#pragma unroll
    for (int i = 0; i < nl; ++i) T[i] = mp.T[i][e];
    double b0;
    const int st = solve_local_dev<N>(S, T, b0);
    if (st == kFitEmpty) {
      const unsigned long long slot = atomicAdd(empty_count, 1ull);
      if (static_cast<i64>(slot) < list_cap) empty_list[slot] = dst;
      out[dst] = __longlong_as_double(0x7ff8000000000000ll);
    } else {
      out[dst] = b0;
    }
  }
}

// Shared-design covariance solve.  With pw(u,v) = sw - dm0 [u == v] (every
// subject's mass grid equal to the constant M0 and a diagonal-only band, see
// dfpca_binned::shared_const), every mass moment is closed-form:
//   S_ab(s,t) = sw P_a(s) P_b(t) - dm0 D_ab(s,t),
//   P_a(s)    = prod_k A^k_{a_k}(s_k),  A^k_r(j) = sum_o taps_r[o+R]  (0 <= j+o < n_k)
//   D_ab(s,t) = prod_k D^k_{a_k b_k}(s_k, t_k),
//   D^k_ab(x, y) = sum_u taps_a[u-x+R] taps_b[u-y+R],
// the separable convolution of the constant and of the diagonal, so only the
// nl value moments come from the convolution pipeline.
struct SharedMoments {
  const double* A[kMaxDim];  // [3][n_k]
  const double* D[kMaxDim];  // [3][3][n_k][n_k]
  int n[kMaxDim];
  int band[kMaxDim];         // D_k(x, y) == 0 exactly when |x - y| > band[k] (= R_s + R_t)
  float inv_n[kMaxDim];      // 1 / n_k for fast_divmod
  double sw, dm0;
  // per-node tables for k_solve_sep_tri (null when an axis exceeds kCoordMask)
  const double* P = nullptr;         // [SepIdx<d>::n][G]: P_a(u) = prod_k A^k_{a_k}(u_k)
  const unsigned* coord = nullptr;   // [G]: axis coordinates, kCoordBits each
  i64 G = 0;
};
constexpr int kCoordBits = 10;
#ifndef DFPCA_SEP_LOOP
#define DFPCA_SEP_LOOP 4
#endif
constexpr int kSepLoop = DFPCA_SEP_LOOP;  // tiles per CTA of k_solve_sep_tri
constexpr unsigned kCoordMask = (1u << kCoordBits) - 1;

template <int P>
__device__ __forceinline__ double shared_moment(const int (&o)[P], const double (&As)[P / 2][3],
                                                const double (&At)[P / 2][3], const double (&Dst)[P / 2][3][3],
                                                double sw, double dm0) {
  constexpr int d = P / 2;
  double pa = 1.0, pd = 1.0;
#pragma unroll
  for (int k = 0; k < d; ++k) {
    pa *= As[k][o[k]] * At[k][o[d + k]];
    pd *= Dst[k][o[k]][o[d + k]];
  }
  return sw * pa - dm0 * pd;
}

template <int N>
__global__ void __launch_bounds__(128) k_solve_shared(SharedMoments sh, MomPtrs mp, SolveGeom g,
                                                      double* __restrict__ out,
                                                      unsigned long long* __restrict__ empty_count,
                                                      i64* __restrict__ empty_list, i64 list_cap) {
  pdl_wait();
  constexpr int p = N - 1;
  constexpr int d = p / 2;
  constexpr int nm = 1 + p + p * (p + 1) / 2;
  constexpr int nl = 1 + p;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < g.npts; e += (i64)gridDim.x * blockDim.x) {
    const i64 row = e / g.tc;
    const i64 col = g.t0 + e % g.tc;
    const i64 dst = row * g.gt + col;
    if (g.upper && row > col) continue;
    if (g.mask && !(g.mask[row] != 0 && g.mask[col] != 0)) {
      out[dst] = __longlong_as_double(0x7ff8000000000000ll);
      continue;
    }
    // per-axis node coordinates, last axis fastest
    int sk[d], tk[d];
    i64 rs = row, rt = col;
#pragma unroll
    for (int k = d - 1; k >= 0; --k) {
      sk[k] = static_cast<int>(rs % sh.n[k]);
      rs /= sh.n[k];
      tk[k] = static_cast<int>(rt % sh.n[k]);
      rt /= sh.n[k];
    }
    double As[d][3], At[d][3], Dst[d][3][3];
#pragma unroll
    for (int k = 0; k < d; ++k) {
      const int n = sh.n[k];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        As[k][r] = __ldg(sh.A[k] + r * n + sk[k]);
        At[k][r] = __ldg(sh.A[k] + r * n + tk[k]);
      }
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          Dst[k][a][b] = a + b <= 2 ? __ldg(sh.D[k] + ((static_cast<i64>(a * 3 + b) * n + sk[k]) * n + tk[k])) : 0.0;
    }
    double S[nm], T[nl];
    {
      int o[p] = {};
      S[0] = shared_moment<p>(o, As, At, Dst, sh.sw, sh.dm0);
    }
#pragma unroll
    for (int k = 0; k < p; ++k) {
      int o[p] = {};
      o[k] = 1;
      S[1 + k] = shared_moment<p>(o, As, At, Dst, sh.sw, sh.dm0);
    }
#pragma unroll
    for (int k = 0; k < p; ++k)
#pragma unroll
      for (int l = k; l < p; ++l) {
        int o[p] = {};
        o[k] += 1;
        o[l] += 1;
        S[quad_index(p, k, l)] = shared_moment<p>(o, As, At, Dst, sh.sw, sh.dm0);
      }
#pragma unroll
    for (int i = 0; i < nl; ++i) T[i] = mp.T[i][e];
    double b0;
    const int st = solve_local_dev<N>(S, T, b0);
    if (st == kFitEmpty) {
      const unsigned long long slot = atomicAdd(empty_count, 1ull);
      if (static_cast<i64>(slot) < list_cap) empty_list[slot] = dst;
      out[dst] = __longlong_as_double(0x7ff8000000000000ll);
    } else {
      out[dst] = b0;
    }
  }
}

// Upper-triangle covariance solve, tiled: CTA (row, 128-column chunk) with
// 32-bit index math.  The s node is uniform across the CTA (its coordinates,
// P_a(s) and the D rows are broadcast loads), the t nodes are consecutive
// (coalesced moment loads and stores); CTAs whose chunk lies left of the
// diagonal exit at once.  Same per-point arithmetic as k_solve /
// k_solve_shared.
constexpr int kSolveTile = 128;

template <int N, bool SHARED>
__device__ __forceinline__ void solve_tri_body(const SharedMoments& sh, const MomPtrs& mp, const SolveGeom& g,
                                               int nch, double* __restrict__ out,
                                               unsigned long long* __restrict__ empty_count,
                                               i64* __restrict__ empty_list, i64 list_cap) {
  constexpr int p = N - 1;
  constexpr int d = p / 2;
  constexpr int nm = 1 + p + p * (p + 1) / 2;
  constexpr int nl = 1 + p;
  const int lrow = static_cast<int>(blockIdx.x / nch);
  const int ch = static_cast<int>(blockIdx.x - static_cast<unsigned>(lrow) * nch);
  const int tc = static_cast<int>(g.tc);
  const int t0 = static_cast<int>(g.t0);
  const int mrow = lrow + static_cast<int>(g.row_lo);  // moment row
  const int row = mrow + static_cast<int>(g.row0);     // global s node
  if (t0 + (ch + 1) * kSolveTile <= row) return;       // whole chunk below the diagonal
  const int c = ch * kSolveTile + static_cast<int>(threadIdx.x);
  const int col = t0 + c;
  if (c >= tc || col < row) return;
  const i64 e = static_cast<i64>(mrow) * tc + c;
  const i64 dst = static_cast<i64>(row - g.out_row0) * g.gt + col;
  if (g.mask && !(g.mask[row] != 0 && g.mask[col] != 0)) {
    out[dst] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  double S[nm], T[nl];
  if constexpr (SHARED) {
    int sk[d], tk[d];
    int rs = row, rt = col;
#pragma unroll
    for (int k = d - 1; k >= 0; --k) {
      const int n = sh.n[k];
      const int qs = rs / n, qt = rt / n;
      sk[k] = rs - qs * n;
      tk[k] = rt - qt * n;
      rs = qs;
      rt = qt;
    }
    double As[d][3], At[d][3], Dst[d][3][3];
#pragma unroll
    for (int k = 0; k < d; ++k) {
      const int n = sh.n[k];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        As[k][r] = __ldg(sh.A[k] + r * n + sk[k]);
        At[k][r] = __ldg(sh.A[k] + r * n + tk[k]);
      }
      const double* Dk = sh.D[k] + sk[k] * n + tk[k];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) Dst[k][a][b] = a + b <= 2 ? __ldg(Dk + (a * 3 + b) * n * n) : 0.0;
    }
    {
      int o[p] = {};
      S[0] = shared_moment<p>(o, As, At, Dst, sh.sw, sh.dm0);
    }
#pragma unroll
    for (int k = 0; k < p; ++k) {
      int o[p] = {};
      o[k] = 1;
      S[1 + k] = shared_moment<p>(o, As, At, Dst, sh.sw, sh.dm0);
    }
#pragma unroll
    for (int k = 0; k < p; ++k)
#pragma unroll
      for (int l = k; l < p; ++l) {
        int o[p] = {};
        o[k] += 1;
        o[l] += 1;
        S[quad_index(p, k, l)] = shared_moment<p>(o, As, At, Dst, sh.sw, sh.dm0);
      }
  } else {
#pragma unroll
    for (int i = 0; i < nm; ++i) S[i] = mp.S[i][e];
  }
#pragma unroll
  for (int i = 0; i < nl; ++i) T[i] = mp.T[i][e];
  double b0;
  __shared__ double sm_solve[(nm + nl) * kSolveTile];
  const int st = solve_local_perm<N>(S, T, sm_solve + threadIdx.x, kSolveTile, b0);
  if (st == kFitEmpty) {
    const unsigned long long slot = atomicAdd(empty_count, 1ull);
    if (static_cast<i64>(slot) < list_cap) empty_list[slot] = dst;
    out[dst] = __longlong_as_double(0x7ff8000000000000ll);
  } else {
    out[dst] = b0;
  }
}
template <int N>
__global__ void __launch_bounds__(kSolveTile) k_solve_tri(MomPtrs mp, SolveGeom g, int nch, double* __restrict__ out,
                                                          unsigned long long* __restrict__ empty_count,
                                                          i64* __restrict__ empty_list, i64 list_cap) {
  pdl_wait();
  solve_tri_body<N, false>(SharedMoments{}, mp, g, nch, out, empty_count, empty_list, list_cap);
}
#ifndef DFPCA_SOLVE5_MIN_CTAS
#define DFPCA_SOLVE5_MIN_CTAS 8
#endif
#ifndef DFPCA_SOLVE_MIN_CTAS
#define DFPCA_SOLVE_MIN_CTAS 1
#endif
// d = 2 (N = 5): 8 CTAs per SM (64 registers, 72 B of spills) measured
// 0.309 ms vs 0.324 ms at the natural 78 registers / 6 CTAs (cfg-3 step)
template <int N>
__global__ void __launch_bounds__(kSolveTile, N == 5 ? 8 : DFPCA_SOLVE_MIN_CTAS)
    k_solve_shared_tri(SharedMoments sh, MomPtrs mp, SolveGeom g, int nch, double* __restrict__ out,
                       unsigned long long* __restrict__ empty_count, i64* __restrict__ empty_list, i64 list_cap) {
  pdl_wait();
  solve_tri_body<N, true>(sh, mp, g, nch, out, empty_count, empty_list, list_cap);
}

// Shared-design covariance solve, tiled like k_solve_tri (CTA = one s row x
// 128 consecutive t).  The closed-form mass moments are separable:
//   S_o(s, t) = sw P_{o_s}(s) P_{o_t}(t) - dm0 prod_k D_k[o_sk][o_tk](s_k, t_k),
// where o = (o_s, o_t) is the moment's multi-index split into its s and t
// axes, P_{o_s}(s) = prod_k A_k[o_sk](s_k) and D_k vanishes exactly unless
// |s_k - t_k| <= R_k(s) + R_k(t).  So each thread forms the (d+1)(d+2)/2
// products of its t node once, the s products are CTA-uniform, a moment is
// one multiply, and the band tables are read only inside the band.  The
// normal matrix then goes through Eigen's pivoted LDLT; when the ridged
// diagonal is already in pivot order (the common case: the constant moment
// dominates and interior second moments tie, first index wins), the
// factorisation runs unpermuted in registers -- exactly the operations
// solve_local_perm performs with the identity permutation -- and only the
// other nodes take the shared-memory gather.
template <int D>
struct SepIdx {  // index of multi-index e_k (deg 1) / e_k + e_l (deg 2) among the (D+1)(D+2)/2
  static constexpr int n = (D + 1) * (D + 2) / 2;
  __host__ __device__ static constexpr int one(int k) { return 1 + k; }
  __host__ __device__ static constexpr int two(int k, int l) {  // k <= l
    return 1 + D + k * D - k * (k - 1) / 2 + (l - k);
  }
};

template <int N>
__device__ __forceinline__ void sep_products(const double (&a)[(N - 1) / 2][3], double (&P)[SepIdx<(N - 1) / 2>::n],
                                             double scale) {
  constexpr int d = (N - 1) / 2;
  using I = SepIdx<d>;
  double z = scale;
#pragma unroll
  for (int k = 0; k < d; ++k) z *= a[k][0];
  P[0] = z;
#pragma unroll
  for (int k = 0; k < d; ++k) {
    double v = scale;
#pragma unroll
    for (int m = 0; m < d; ++m) v *= a[m][m == k ? 1 : 0];
    P[I::one(k)] = v;
  }
#pragma unroll
  for (int k = 0; k < d; ++k)
#pragma unroll
    for (int l = k; l < d; ++l) {
      double v = scale;
#pragma unroll
      for (int m = 0; m < d; ++m) v *= a[m][(m == k) + (m == l)];
      P[I::two(k, l)] = v;
    }
}

// x = q n + r for 0 <= x < 2^24 without an integer division (float
// reciprocal estimate, one correction step).
__device__ __forceinline__ void fast_divmod(int x, int n, float inv_n, int& q, int& r) {
  q = __float2int_rz(__int2float_rn(x) * inv_n);
  r = x - q * n;
  if (r < 0) {
    --q;
    r += n;
  } else if (r >= n) {
    ++q;
    r -= n;
  }
}

// S (MomentBasis order, local_fit.hpp:34-47: covariates 0..d-1 are the s
// axes, d..2d-1 the t axes) of node pair (s, t) from the per-node products
// Ps = P(s), Pt = P(t) and packed axis coordinates cs, ct.  Raw products, the
// weight applied last: S = sw (P_s P_t), so moments that are mirror images of
// each other (s <-> t, or axis k <-> l at interior nodes) round identically
// and tie exactly in the exact path's pivot order.
// kExactOrder: the rounding the exact pass replays (sw applied last, so
// mirror-image moments tie exactly); otherwise Ps arrives pre-scaled by sw
// (one multiply per moment; the certified fast path needs no ties).
template <int N, bool kExactOrder = true>
__device__ __forceinline__ void sep_assemble(const SharedMoments& sh, const double (&Ps)[SepIdx<(N - 1) / 2>::n],
                                             const double (&Pt)[SepIdx<(N - 1) / 2>::n], unsigned cs, unsigned ct,
                                             double (&S)[1 + (N - 1) + (N - 1) * N / 2]) {
  constexpr int p = N - 1;
  constexpr int d = p / 2;
  using I = SepIdx<d>;
  const double sw = sh.sw;
  auto sc = [&](double v) { return kExactOrder ? sw * v : v; };
  S[0] = sc(Ps[0] * Pt[0]);
#pragma unroll
  for (int k = 0; k < p; ++k) S[1 + k] = sc(k < d ? Ps[I::one(k)] * Pt[0] : Ps[0] * Pt[I::one(k - d)]);
#pragma unroll
  for (int k = 0; k < p; ++k)
#pragma unroll
    for (int l = k; l < p; ++l) {
      double v;
      if (l < d) v = Ps[I::two(k, l)] * Pt[0];
      else if (k >= d) v = Ps[0] * Pt[I::two(k - d, l - d)];
      else v = Ps[I::one(k)] * Pt[I::one(l - d)];
      S[quad_index(p, k, l)] = sc(v);
    }
  int sk[d], tk[d];
  bool near = true;
#pragma unroll
  for (int k = 0; k < d; ++k) {
    sk[k] = static_cast<int>((cs >> (kCoordBits * k)) & kCoordMask);
    tk[k] = static_cast<int>((ct >> (kCoordBits * k)) & kCoordMask);
    const int dist = sk[k] > tk[k] ? sk[k] - tk[k] : tk[k] - sk[k];
    near = near && dist <= sh.band[k];
  }
  if (near) {
    // the same-observation band (exact zero outside it)
    double Dst[d][3][3];
#pragma unroll
    for (int k = 0; k < d; ++k) {
      const int n = sh.n[k];
      const double* Dk = sh.D[k] + sk[k] * n + tk[k];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) Dst[k][a][b] = a + b <= 2 ? __ldg(Dk + (a * 3 + b) * n * n) : 0.0;
    }
    auto band = [&](const int (&o)[p]) {
      double pd = sh.dm0;
#pragma unroll
      for (int k = 0; k < d; ++k) pd *= Dst[k][o[k]][o[d + k]];
      return pd;
    };
    {
      int o[p] = {};
      S[0] -= band(o);
    }
#pragma unroll
    for (int k = 0; k < p; ++k) {
      int o[p] = {};
      o[k] = 1;
      S[1 + k] -= band(o);
    }
#pragma unroll
    for (int k = 0; k < p; ++k)
#pragma unroll
      for (int l = k; l < p; ++l) {
        int o[p] = {};
        o[k] += 1;
        o[l] += 1;
        S[quad_index(p, k, l)] -= band(o);
      }
  }
}

// The per-node product table is interleaved, [G][sep_stride(d)] with the row
// padded to whole 16-byte pairs: one node's products are sep_stride / 2
// 128-bit loads (uniform for the row node, lane-contiguous for the columns).
__host__ __device__ constexpr int sep_stride(int d) { return ((d + 1) * (d + 2) / 2 + 1) & ~1; }

template <int N>
__device__ __forceinline__ void sep_load(const SharedMoments& sh, int node, double (&P)[SepIdx<(N - 1) / 2>::n]) {
  constexpr int np = SepIdx<(N - 1) / 2>::n;
  constexpr int ns = sep_stride((N - 1) / 2);
  const double2* q = reinterpret_cast<const double2*>(sh.P + static_cast<i64>(node) * ns);
#pragma unroll
  for (int i = 0; i < ns / 2; ++i) {
    const double2 v = __ldg(q + i);
    P[2 * i] = v.x;
    if (2 * i + 1 < np) P[2 * i + 1] = v.y;
  }
}

// Node of the tiled upper-triangle solve handled by thread `tid` of CTA
// (ch, lrow); false when the thread has no node.  Index arithmetic in 32
// bits (the launch guarantees rows * gt < 2^32 and npts < 2^32).
struct SepNode {
  unsigned row, col, c;
  unsigned e, dst;
};
__device__ __forceinline__ bool sep_node(const SolveGeom& g, unsigned lrow, unsigned ch, unsigned tid, SepNode& n) {
  const unsigned tc = static_cast<unsigned>(g.tc);
  const unsigned mrow = lrow + static_cast<unsigned>(g.row_lo);
  n.row = mrow + static_cast<unsigned>(g.row0);
  n.c = ch * kSolveTile + tid;
  n.col = static_cast<unsigned>(g.t0) + n.c;
  if (n.c >= tc || n.col < n.row) return false;
  n.e = mrow * tc + n.c;
  n.dst = (n.row - static_cast<unsigned>(g.out_row0)) * static_cast<unsigned>(g.gt) + n.col;
  return true;
}

// First column chunk of local row lrow holding a node with col >= row.
__host__ __device__ __forceinline__ unsigned sep_first_chunk(const SolveGeom& g, unsigned lrow, unsigned nch) {
  const long long row = static_cast<long long>(lrow) + g.row_lo + g.row0;
  const long long off = row - g.t0;
  const unsigned ch = off > 0 ? static_cast<unsigned>(off / kSolveTile) : 0u;
  return ch < nch ? ch : nch;
}

// Paired-row grid of the tiled triangle: grid row y holds the chunks of
// local rows y and rows-1-y back to back (their counts sum to ~nch + 1 on
// the full square), so no CTA is launched below the diagonal.
__device__ __forceinline__ bool sep_cta(const SolveGeom& g, unsigned rows, unsigned nch, unsigned x, unsigned& lrow,
                                        unsigned& ch) {
  const unsigned y = blockIdx.y;
  const unsigned c0 = sep_first_chunk(g, y, nch), cnt0 = nch - c0;
  if (x < cnt0) {
    lrow = y;
    ch = c0 + x;
    return true;
  }
  const unsigned y1 = rows - 1 - y;
  if (y1 <= y) return false;
  const unsigned c1 = sep_first_chunk(g, y1, nch);
  if (x - cnt0 >= nch - c1) return false;
  lrow = y1;
  ch = c1 + (x - cnt0);
  return true;
}

// Streaming load that does not allocate in L1 (the value moments are read
// once; L1 keeps the product- and band-table lines instead).
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// The ridged diagonal (eps = kRidgeScale trace, local_fit.hpp:70-71).
template <int N>
__device__ __forceinline__ void ridged_diagonal(const double (&S)[1 + (N - 1) + (N - 1) * N / 2], double (&dg)[N]) {
  constexpr int p = N - 1;
  dg[0] = S[0];
#pragma unroll
  for (int k = 0; k < p; ++k) dg[k + 1] = S[quad_index(p, k, k)];
  double tr = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) tr += dg[i];
  const double eps = 1e-10 * tr;
#pragma unroll
  for (int i = 0; i < N; ++i) dg[i] += eps;
}

// Shared-design covariance solve over the upper triangle, one CTA per
// (row, 128-column chunk): the mass moments are assembled from the per-node
// product table (uniform for the row, 128-bit loads for the columns), the
// value moments read from the pipeline, and the ridged system solved by the
// certified fast path (ldlt_certified).  Windows it cannot certify
// (near-singular, empty, non-SPD) are queued for k_solve_sep_exact as
// (word, lane bits) entries, word = lrow * ceil(tc / 32) + c / 32, one per
// warp with misses (pending[0] = count, zeroed by the caller; entries from
// pending[2]), so this kernel carries no register or code for them.
template <int N>
__global__ void __launch_bounds__(kSolveTile, N == 5 ? DFPCA_SOLVE5_MIN_CTAS : DFPCA_SOLVE_MIN_CTAS)
    k_solve_sep_tri(SharedMoments sh, MomPtrs mp, SolveGeom g, unsigned rows, unsigned nch,
                    double* __restrict__ out, unsigned* __restrict__ pending) {
  pdl_wait();
  constexpr int p = N - 1;
  constexpr int d = p / 2;
  constexpr int nm = 1 + p + p * (p + 1) / 2;
  constexpr int nl = 1 + p;
  for (int it = 0; it < kSepLoop; ++it) {  // kSepLoop tiles of the grid row per CTA
    unsigned lrow, ch;
    if (!sep_cta(g, rows, nch, blockIdx.x * kSepLoop + it, lrow, ch)) return;
    SepNode n;
    bool done = true;
    if (sep_node(g, lrow, ch, threadIdx.x, n)) {
      if (g.mask && !(g.mask[n.row] != 0 && g.mask[n.col] != 0)) {
        out[n.dst] = __longlong_as_double(0x7ff8000000000000ll);
      } else {
        double T[nl];
#pragma unroll
        for (int i = 0; i < nl; ++i) T[i] = ld_stream(mp.T[i] + n.e);  // issue the moment loads first
        double Ps[SepIdx<d>::n], Pt[SepIdx<d>::n];
        sep_load<N>(sh, n.row, Ps);
        sep_load<N>(sh, n.col, Pt);
#pragma unroll
        for (int i = 0; i < SepIdx<d>::n; ++i) Ps[i] *= sh.sw;
        double S[nm];
        sep_assemble<N, false>(sh, Ps, Pt, __ldg(sh.coord + n.row), __ldg(sh.coord + n.col), S);
        double dg[N], b0;
        ridged_diagonal<N>(S, dg);
        done = ldlt_certified<N>(S, T, dg, b0);
        if (done) __stcs(out + n.dst, b0);
      }
    }
    const unsigned miss = __ballot_sync(0xffffffffu, !done);
    if (miss != 0 && (threadIdx.x & 31) == __ffs(miss) - 1) {
      const unsigned wpr = static_cast<unsigned>((g.tc + 31) / 32);
      const unsigned slot = atomicAdd(pending, 1u);
      pending[2 + 2 * slot] = lrow * wpr + (n.c >> 5);
      pending[3 + 2 * slot] = miss;
    }
  }
}

// The windows k_solve_sep_tri flagged: Eigen's pivoted LDLT replayed exactly
// (solve_local_perm), the local-constant fallback and the empty-window list.
// One thread per queued warp word.
template <int N>
__global__ void __launch_bounds__(kSolveTile) k_solve_sep_exact(SharedMoments sh, MomPtrs mp, SolveGeom g,
                                                                const unsigned* __restrict__ pending,
                                                                double* __restrict__ out,
                                                                unsigned long long* __restrict__ empty_count,
                                                                i64* __restrict__ empty_list, i64 list_cap) {
  pdl_wait();
  constexpr int p = N - 1;
  constexpr int d = p / 2;
  constexpr int nm = 1 + p + p * (p + 1) / 2;
  constexpr int nl = 1 + p;
  __shared__ double sm_solve[(nm + nl) * kSolveTile];
  const i64 wpr = (g.tc + 31) / 32;
  const unsigned n_words = pending[0];
  for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < n_words; q += gridDim.x * blockDim.x) {
    const i64 w = pending[2 + 2 * q];
    unsigned bits = pending[3 + 2 * q];
    const int lrow = static_cast<int>(w / wpr);
    const int cw = static_cast<int>(w % wpr) * 32;
    while (bits) {
      const int lane = __ffs(bits) - 1;
      bits &= bits - 1;
      SepNode n;
      if (!sep_node(g, static_cast<unsigned>(lrow), static_cast<unsigned>(cw / kSolveTile),
                    static_cast<unsigned>(cw % kSolveTile + lane), n))
        continue;
      double T[nl], Ps[SepIdx<d>::n], Pt[SepIdx<d>::n], S[nm], b0;
#pragma unroll
      for (int i = 0; i < nl; ++i) T[i] = mp.T[i][n.e];
      sep_load<N>(sh, n.row, Ps);
      sep_load<N>(sh, n.col, Pt);
      sep_assemble<N>(sh, Ps, Pt, __ldg(sh.coord + n.row), __ldg(sh.coord + n.col), S);
      const int st = solve_local_perm<N>(S, T, sm_solve + threadIdx.x, kSolveTile, b0);
      if (st == kFitEmpty) {
        const unsigned long long slot = atomicAdd(empty_count, 1ull);
        if (static_cast<i64>(slot) < list_cap) empty_list[slot] = n.dst;
        out[n.dst] = __longlong_as_double(0x7ff8000000000000ll);
      } else {
        out[n.dst] = b0;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Empty-window fallback ladder (fft_smoother.hpp:471-487): for each listed
// node, up to kWindowRetries direct gathers at 1.5^r h over the binned arrays
// (mean: gather_binned_equations, :236-277; covariance: the pw/pv window
// gather, :668-711), each followed by the ridged solve.
struct LadderGeom {
  int p;                 // dims of the domain (d or 2d)
  i64 shape[kMaxP];
  i64 strides[kMaxP];
  double spacing[kMaxP];
  double h[kMaxP];
};

__global__ void k_ladder(LadderGeom lg, const double* __restrict__ mass, const double* __restrict__ value,
                         const i64* __restrict__ nodes, i64 n_nodes, double* __restrict__ out,
                         unsigned long long* __restrict__ still_empty) {
  pdl_wait();
  __shared__ double red[256];
  __shared__ double acc[kMaxNm + kMaxNl];
  __shared__ int status_sh;
  const int p = lg.p;
  const int nm = 1 + p + p * (p + 1) / 2;
  const int nl = 1 + p;
  for (i64 q = blockIdx.x; q < n_nodes; q += gridDim.x) {
    const i64 flat = nodes[q];
    i64 node[kMaxP];
    {
      i64 rem = flat;
      for (int k = p - 1; k >= 0; --k) {
        node[k] = rem % lg.shape[k];
        rem /= lg.shape[k];
      }
    }
    double scale = 1.0;
    int status = kFitEmpty;
    double b0 = 0.0;
    for (int retry = 0; retry < 3 && status == kFitEmpty; ++retry) {
      scale *= 1.5;
      double hs[kMaxP];
      i64 lo[kMaxP], ext[kMaxP];
      i64 count = 1;
      for (int k = 0; k < p; ++k) {
        hs[k] = lg.h[k] * scale;
        const i64 r = static_cast<i64>(ceil(hs[k] / lg.spacing[k]));
        lo[k] = node[k] - r < 0 ? 0 : node[k] - r;
        const i64 hi = node[k] + r + 1 > lg.shape[k] ? lg.shape[k] : node[k] + r + 1;
        ext[k] = hi - lo[k];
        count *= ext[k];
      }
      double part[kMaxNm + kMaxNl];
      for (int i = 0; i < nm + nl; ++i) part[i] = 0.0;
      for (i64 w = threadIdx.x; w < count; w += blockDim.x) {
        i64 rem = w, off = 0;
        double u[kMaxP];
        for (int k = p - 1; k >= 0; --k) {
          const i64 m = lo[k] + rem % ext[k];
          rem /= ext[k];
          off += m * lg.strides[k];
          u[k] = static_cast<double>(node[k] - m) * lg.spacing[k];
        }
        const double mv = mass[off], vv = value[off];
        if (mv == 0.0 && vv == 0.0) continue;
        double kw = 1.0;
        for (int k = 0; k < p; ++k) {
          const double z = u[k] / hs[k];
          const double t = 1.0 - z * z;
          if (!(t > 0.0)) {
            kw = 0.0;
            break;
          }
          kw *= 0.75 * t / hs[k];
        }
        if (kw == 0.0) continue;
        const double w0 = kw * mv, wy = kw * vv;
        part[0] += w0;
        part[nm] += wy;
        for (int k = 0; k < p; ++k) {
          const double wu = w0 * u[k];
          part[1 + k] += wu;
          part[nm + 1 + k] += wy * u[k];
          for (int l = k; l < p; ++l) part[quad_index(p, k, l)] += wu * u[l];
        }
      }
      for (int i = 0; i < nm + nl; ++i) {
        red[threadIdx.x] = part[i];
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
          if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
          __syncthreads();
        }
        if (threadIdx.x == 0) acc[i] = red[0];
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        int st = kFitEmpty;
        if (acc[0] > 0.0) st = solve_local_any(p, acc, acc + nm, b0);
        status_sh = st;
        if (st != kFitEmpty) out[flat] = b0;
      }
      __syncthreads();
      status = status_sh;
      __syncthreads();
    }
    if (threadIdx.x == 0 && status == kFitEmpty) atomicAdd(still_empty, 1ull);
  }
}

// Covariance centering and symmetrization (fft_smoother.hpp:723-736).  The
// solve filled the upper triangle s <= t; each entry is centered by the mean
// product and written to both (s,t) and (t,s), so the result is exactly
// symmetric.  32x32 tile pairs keep both the row and the mirrored column
// accesses coalesced.
__global__ void k_center_mirror(double* __restrict__ cov, const double* __restrict__ mean,
                                const std::uint8_t* __restrict__ mask, i64 G, i64 I0, i64 I1, i64 out_row0) {
  pdl_wait();
  // Slab form (shard.hpp): row tiles [I0, I1) of 32 rows, cov holds global
  // rows from out_row0 on; mirrors land only inside the slab's own rows (the
  // rest reach their owners through the covariance exchange).
  __shared__ double tile[32][33];
  const i64 tiles = (G + 31) / 32;
  // tile pair (I <= J) of this CTA: row I starts at pair index
  // start(I) = I * tiles - I (I - 1) / 2; invert with a square root, then fix
  // the rounding
  auto start = [tiles](i64 i) { return i * tiles - i * (i - 1) / 2; };
  const i64 t = blockIdx.x + start(I0);
  const double tb = 2.0 * static_cast<double>(tiles) + 1.0;
  i64 I = static_cast<i64>((tb - sqrt(tb * tb - 8.0 * static_cast<double>(t))) * 0.5);
  if (I < 0) I = 0;
  if (I > tiles - 1) I = tiles - 1;
  while (I > 0 && start(I) > t) --I;
  while (I + 1 < tiles && start(I + 1) <= t) ++I;
  const i64 J = I + (t - start(I));
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8 threads
  // the thread's four rows: loads first (independent), then center and store
  const i64 b = J * 32 + tx;
  double v[4];
  bool ok[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const i64 a = I * 32 + ty + 8 * q;
    ok[q] = a < G && b < G && a <= b;
    v[q] = ok[q] ? cov[(a - out_row0) * G + b] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = ty + 8 * q;
    const i64 a = I * 32 + r;
    if (ok[q]) {
      if (!mask || (mask[a] && mask[b])) v[q] -= mean[a] * mean[b];
      cov[(a - out_row0) * G + b] = v[q];
    }
    tile[r][tx] = v[q];
  }
  if (J >= I1) return;  // mirror rows belong to a later slab
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const i64 bm = J * 32 + r, am = I * 32 + tx;  // mirror (bm, am) of the upper entry (am, bm)
    if (am < G && bm < G && am < bm) cov[(bm - out_row0) * G + am] = tile[tx][r];
  }
}

// The centering of k_center_mirror on listed upper entries (flat s G + t,
// s <= t) and their mirrors: the entries the ladder refitted after it.
__global__ void k_center_list(double* __restrict__ cov, const double* __restrict__ mean,
                              const std::uint8_t* __restrict__ mask, i64 G, const i64* __restrict__ list, i64 n) {
  pdl_wait();
  for (i64 q = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 dst = list[q], a = dst / G, b = dst % G;
    double v = cov[dst];
    if (!mask || (mask[a] && mask[b])) v -= mean[a] * mean[b];
    cov[dst] = v;
    if (a < b) cov[b * G + a] = v;
  }
}

__global__ void k_fill_nan(double* p, i64 n) {
  pdl_wait();
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x)
    p[e] = __longlong_as_double(0x7ff8000000000000ll);
}

// ---------------------------------------------------------------------------
namespace {

using SolveLauncher = void (*)(dfpca_context*, const MomPtrs&, const SolveGeom&, double*,
                               unsigned long long*, i64*, i64);
// Tiled upper-triangle launch geometry: (rows x chunks) CTAs, or -1 when the
// chunk does not qualify (not the upper covariance, or too many CTAs; slabs
// always qualify, see run_covariance_impl).
inline i64 tri_ctas(const SolveGeom& g, int& nch) {
  if (!(g.cov && g.upper) || g.tc <= 0 || g.gt > (i64(1) << 30)) return -1;
  nch = static_cast<int>((g.tc + kSolveTile - 1) / kSolveTile);
  const i64 rows = g.npts / g.tc - g.row_lo;
  const i64 n = (rows > 0 ? rows : 0) * nch;
  return n < (i64(1) << 31) ? n : -1;
}
template <int N>
void launch_solve(dfpca_context* ctx, const MomPtrs& mp, const SolveGeom& g, double* out,
                  unsigned long long* cnt, i64* list, i64 cap) {
  int nch = 0;
  if (const i64 n = tri_ctas(g, nch); n >= 0) {
    if (n > 0)
      DFPCA_LAUNCH(ctx, k_solve_tri<N>, static_cast<unsigned>(n), kSolveTile, 0, mp, g, nch, out, cnt, list, cap);
    return;
  }
  DFPCA_LAUNCH(ctx, k_solve<N>, grid_for(g.npts, 128, 148ll * 64), 128, 0, mp, g, out, cnt, list,
               cap);
}
template <int N>
void launch_solve_shared_n(dfpca_context* ctx, const SharedMoments& sh, const MomPtrs& mp, const SolveGeom& g,
                           double* out, unsigned long long* cnt, i64* list, i64 cap) {
  int nch = 0;
  if (const i64 n = tri_ctas(g, nch); n >= 0) {
    if (n > 0) {
      const i64 rows = n / nch;
      if (rows <= 2 * 65535 && rows * g.gt < (i64(1) << 32) && g.npts < (i64(1) << 32) && sh.P) {
        const i64 n_words = rows * ((g.tc + 31) / 32);
        DevBuf<unsigned> pending(static_cast<std::size_t>(2 + 2 * n_words));
        DFPCA_CUDA(cudaMemsetAsync(pending.get(), 0, sizeof(unsigned), ctx->stream));
        unsigned gx = 1;  // widest row pair
        for (i64 y = 0; y < (rows + 1) / 2; ++y) {
          const unsigned c0 = nch - sep_first_chunk(g, static_cast<unsigned>(y), nch);
          const i64 y1 = rows - 1 - y;
          const unsigned c1 = y1 > y ? nch - sep_first_chunk(g, static_cast<unsigned>(y1), nch) : 0u;
          gx = std::max(gx, c0 + c1);
        }
        DFPCA_LAUNCH_PDL(ctx, k_solve_sep_tri<N>, dim3((gx + kSepLoop - 1) / kSepLoop, static_cast<unsigned>((rows + 1) / 2)),
                     kSolveTile, 0, sh, mp,
                     g, static_cast<unsigned>(rows), static_cast<unsigned>(nch), out, pending.get());
        DFPCA_LAUNCH_PDL(ctx, k_solve_sep_exact<N>, 148 * 4, kSolveTile, 0, sh, mp, g, pending.get(), out, cnt, list,
                     cap);
      } else
        DFPCA_LAUNCH(ctx, k_solve_shared_tri<N>, static_cast<unsigned>(n), kSolveTile, 0, sh, mp, g, nch, out, cnt,
                     list, cap);
    }
    return;
  }
  DFPCA_LAUNCH(ctx, k_solve_shared<N>, grid_for(g.npts, 128, 148ll * 64), 128, 0, sh, mp, g, out, cnt, list,
               cap);
}
void launch_solve_shared(int d, dfpca_context* ctx, const SharedMoments& sh, const MomPtrs& mp,
                         const SolveGeom& g, double* out, unsigned long long* cnt, i64* list, i64 cap) {
  switch (d) {
    case 1: launch_solve_shared_n<3>(ctx, sh, mp, g, out, cnt, list, cap); break;
    case 2: launch_solve_shared_n<5>(ctx, sh, mp, g, out, cnt, list, cap); break;
    default: launch_solve_shared_n<7>(ctx, sh, mp, g, out, cnt, list, cap); break;
  }
}

SolveLauncher solve_launcher(int p) {
  switch (p) {
    case 1: return &launch_solve<2>;
    case 2: return &launch_solve<3>;
    case 3: return &launch_solve<4>;
    case 4: return &launch_solve<5>;
    case 5: return &launch_solve<6>;
    default: return &launch_solve<7>;
  }
}

// Runs the passes of a tree over `axes` (indices into cd.shape, processed in
// the given order) starting from `roots`; the final level's arrays are
// returned (keyed by full orders).  Intermediate levels live in `arena`;
// if `final_dst` resolves a pointer for a leaf, the last pass writes there.
struct Leaf {
  Orders ord;
  int budget_max;
  double* ptr;
  View view;  // view of the leaf array over the chunk (for phase S reads)
};

struct TreeAxis {
  int axis_index;  // index into the domain axes (for taps / orders)
  int view_k;      // index into cd.shape
};

std::vector<Leaf> run_tree(dfpca_context* ctx, const std::vector<Leaf>& roots,
                           const std::vector<TreeAxis>& axes, const ChunkDims& cd,
                           const std::vector<AxisTaps>& taps, i64 chunk_elems,
                           double* taps_dev, std::vector<std::unique_ptr<DevBuf<double>>>& keep,
                           const std::function<double*(const Orders&, int)>& final_dst,
                           const std::function<i64(const Orders&, int)>& final_row_stride,
                           bool first_reads_strided, i64 first_row_stride) {
  std::vector<Leaf> cur = roots;
  // axis0_first with a window: levels after the first see planes [lo, hi)
  const bool narrow = cd.axis0_first && cd.win_k == 0 && cd.win_hi >= 0;
  ChunkDims cd_rest = cd;
  i64 off_rest = 0;
  if (narrow) {
    i64 plane = cd.tail;
    for (std::size_t a = 1; a < cd.shape.size(); ++a) plane *= cd.shape[a];
    off_rest = cd.win_lo * plane;
    cd_rest.shape[0] = std::max<i64>(0, cd.win_hi - cd.win_lo);
    cd_rest.tri_params.tri_row0 += cd.win_lo;
    cd_rest.win_k = -1;
  }
  for (std::size_t ai = 0; ai < axes.size(); ++ai) {
    const TreeAxis& ax = axes[ai];
    const bool last = ai + 1 == axes.size();
    const ChunkDims& cdl = (narrow && ai >= 1) ? cd_rest : cd;
    const i64 off = (narrow && ai >= 1) ? off_rest : 0;
    std::vector<Leaf> next;
    std::vector<std::unique_ptr<DevBuf<double>>> level_bufs;
    for (const Leaf& in : cur) {
      const int used = order_sum(in.ord);
      const int n_out = in.budget_max - used + 1;
      PassSpec spec{};
      spec.in = (ai == 0 && first_reads_strided) ? make_view(in.ptr, cdl, ax.view_k, first_row_stride)
                                                 : make_view(in.ptr + off, cdl, ax.view_k);
      if (ai == 0 && first_reads_strided) spec.in = in.view;
      if (ai < cdl.tri.size() && cdl.tri[ai]) {
        spec.in.tri = cdl.tri[ai];
        spec.in.tri_R = cdl.tri_params.tri_R;
        spec.in.tri_G = cdl.tri_params.tri_G;
        spec.in.tri_rn = cdl.tri_params.tri_rn;
        spec.in.tri_n1 = cdl.tri_params.tri_n1;
        spec.in.tri_row0 = cdl.tri_params.tri_row0;
        spec.in.tri_row_hi = cdl.tri_params.tri_row_hi;
        spec.in.tri_t0 = cdl.tri_params.tri_t0;
      }
      if (ax.view_k == cdl.win_k) {
        spec.in.lo = cdl.win_lo;
        spec.in.hi = cdl.win_hi;
      }
      spec.n_out = n_out;
      spec.R = taps[ax.axis_index].R;
      for (int r = 0; r < n_out; ++r) {
        Leaf o;
        o.ord = in.ord;
        o.ord[ax.axis_index] += r;
        o.budget_max = in.budget_max;
        double* dst = last ? final_dst(o.ord, o.budget_max) : nullptr;
        i64 rs = -1;
        if (!dst) {
          level_bufs.push_back(std::make_unique<DevBuf<double>>(static_cast<std::size_t>(chunk_elems)));
          dst = level_bufs.back()->get();
        } else {
          rs = final_row_stride(o.ord, o.budget_max);
        }
        o.ptr = dst;
        if (ai == 0 && cd.axis0_first) {
          // compact [n][outer][inner]: the axis outermost, as the roots
          View v = spec.in;
          v.p = dst;
          v.os = v.inner;
          v.js = v.outer * v.inner;
          v.tri = 0;
          v.lo = 0;
          v.hi = -1;
          spec.out[r] = v;
        } else {
          spec.out[r] = make_view(dst + off, cdl, ax.view_k, rs);
        }
        o.view = spec.out[r];
        spec.taps[r] = taps[ax.axis_index].t[r].data();
        next.push_back(o);
      }
      run_pass(ctx, spec, taps_dev);
    }
    // previous level buffers can be released once this level's passes are
    // queued (stream order protects the reads).
    for (auto& b : keep) {
      (void)b;
    }
    keep.clear();
    for (auto& b : level_bufs) keep.push_back(std::move(b));
    cur = std::move(next);
  }
  return cur;
}

}  // namespace

// ---------------------------------------------------------------------------
// Host orchestration.

struct SmoothTimer {
  dfpca_context* ctx;
  explicit SmoothTimer(dfpca_context* c, const char* name) : ctx(c) { ctx->begin_stage(name); }
  ~SmoothTimer() { ctx->end_stage(); }
};

void validate_bandwidth(const Grid& grid, const double* h);

void run_local_linear(dfpca_context* ctx, const dfpca_binned* b, const Grid& grid, const double* h,
                      int target, double* out_host, dfpca_surface** out_surface) {
  const int d = grid.d;
  const i64 G = grid.G;
  Basis basis(d);
  std::vector<AxisTaps> taps(d);
  for (int k = 0; k < d; ++k) taps[k] = make_taps(h[k], grid.spacing[k]);

  cudaStream_t st = ctx->stream;
  DevBuf<double> taps_dev(3 * (2 * 4096 + 1));
  auto surf = std::make_unique<dfpca_surface>();
  surf->grid = grid;
  surf->kind = target == DFPCA_TARGET_MEAN ? DFPCA_SURFACE_MEAN : DFPCA_SURFACE_DIAG;
  surf->n = G;
  surf->values.alloc(G);

  ctx->begin_stage("moments");
  const double* value = target == DFPCA_TARGET_MEAN ? b->wvalue.get() : b->wsquare.get();
  ChunkDims cd;
  cd.rows = 1;
  for (int k = 0; k < d; ++k) cd.shape.push_back(grid.shape[k]);
  cd.tail = 1;
  std::vector<TreeAxis> axes;
  for (int k = d - 1; k >= 0; --k) axes.push_back({k, k});
  std::vector<Leaf> roots(2);
  roots[0].ord = Orders{};
  roots[0].budget_max = 2;
  roots[0].ptr = const_cast<double*>(b->mass.get());
  roots[1].ord = Orders{};
  roots[1].budget_max = 1;
  roots[1].ptr = const_cast<double*>(value);
  std::vector<std::unique_ptr<DevBuf<double>>> keep;
  std::vector<std::unique_ptr<DevBuf<double>>> finals;
  auto final_dst = [&](const Orders&, int) -> double* {
    finals.push_back(std::make_unique<DevBuf<double>>(static_cast<std::size_t>(G)));
    return finals.back()->get();
  };
  auto final_rs = [&](const Orders&, int) -> i64 { return -1; };
  std::vector<Leaf> leaves = run_tree(ctx, roots, axes, cd, taps, G, taps_dev.get(), keep, final_dst,
                                      final_rs, false, -1);
  ctx->end_stage();

  MomPtrs mp{};
  for (const Leaf& l : leaves) {
    const int idx = basis.find(l.ord);
    if (l.budget_max == 2) mp.S[idx] = l.ptr;
    else mp.T[idx] = l.ptr;
  }

  ctx->begin_stage("solve");
  DevBuf<std::uint8_t> mask_dev;
  if (grid.has_mask) {
    mask_dev.alloc(G);
    DFPCA_CUDA(cudaMemcpyAsync(mask_dev.get(), grid.mask.data(), G, cudaMemcpyHostToDevice, st));
  }
  DevBuf<unsigned long long> cnt(1);
  DevBuf<i64> list(static_cast<std::size_t>(G));
  DFPCA_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), st));
  SolveGeom sg{};
  sg.npts = G;
  sg.tc = G;
  sg.t0 = 0;
  sg.gt = G;
  sg.cov = 0;
  sg.mask = grid.has_mask ? mask_dev.get() : nullptr;
  solve_launcher(d)(ctx, mp, sg, surf->values.get(), cnt.get(), list.get(), G);
  unsigned long long n_empty = 0;
  DFPCA_CUDA(cudaMemcpyAsync(&n_empty, cnt.get(), sizeof(n_empty), cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
  ctx->end_stage();

  if (n_empty > 0) {
    ctx->begin_stage("fallback");
    LadderGeom lg{};
    lg.p = d;
    for (int k = 0; k < d; ++k) {
      lg.shape[k] = grid.shape[k];
      lg.strides[k] = grid.strides[k];
      lg.spacing[k] = grid.spacing[k];
      lg.h[k] = h[k];
    }
    DevBuf<unsigned long long> still(1);
    DFPCA_CUDA(cudaMemsetAsync(still.get(), 0, sizeof(unsigned long long), st));
    DFPCA_LAUNCH(ctx, k_ladder, grid_for(static_cast<i64>(n_empty), 1, 148ll * 8), 256, 0, lg,
                 b->mass.get(), value, list.get(), static_cast<i64>(n_empty), surf->values.get(),
                 still.get());
    unsigned long long n_still = 0;
    DFPCA_CUDA(cudaMemcpyAsync(&n_still, still.get(), sizeof(n_still), cudaMemcpyDeviceToHost, st));
    DFPCA_CUDA(cudaStreamSynchronize(st));
    ctx->end_stage();
    if (n_still > 0)
      fail(kNumeric, "BandwidthTooSmall",
           "binned local linear smoother: " + std::to_string(n_still) +
               " node(s) had no binned mass in the kernel window (AllWeightsZero) after 3 window "
               "enlargements");
  }
  if (out_host)
    DFPCA_CUDA(cudaMemcpyAsync(out_host, surf->values.get(), sizeof(double) * G,
                               cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
  if (out_surface) *out_surface = surf.release();
}

// Pair grids + moments + solve + center + symmetrize for the covariance.
void run_covariance_impl(dfpca_context* ctx, const dfpca_binned* b, const Grid& grid, const double* h,
                         const double* mean_host, const CovShardExec* shard, dfpca_surface** out) {
  host_mark("cov entry");
  const int d = grid.d;
  const int p = 2 * d;
  const i64 G = grid.G;
  const i64 G2 = G * G;
  cudaStream_t st = ctx->stream;
  Basis basis(p);
  std::vector<AxisTaps> taps(p);
  for (int k = 0; k < p; ++k) taps[k] = make_taps(h[k % d], grid.spacing[k % d]);
  DevBuf<double> taps_dev(3 * (2 * 4096 + 1));
  host_mark("taps");

  // Slab of this rank (shard.hpp): pair-grid / t-partial rows are the s1
  // planes [ha, hb), output rows the planes [sa, sb); one device: everything.
  const i64 n1 = grid.shape[0];
  const i64 rn = G / n1;  // s nodes per s1 plane
  const bool sharded = shard != nullptr && shard->plan->world > 1;
  const i64 sa = sharded ? shard->plan->a(shard->rank) : 0, sb = sharded ? shard->plan->b(shard->rank) : n1;
  const i64 ha = sharded ? shard->plan->ha(shard->rank) : 0, hb = sharded ? shard->plan->hb(shard->rank) : n1;
  const i64 L = hb - ha;       // local planes
  const i64 LR = L * rn;       // local pair-grid rows
  const i64 row0 = ha * rn;    // global s of local row 0
  const i64 out_row0 = sa * rn;
  const i64 out_rows = (sb - sa) * rn;
  const i64 col_lo = sa * rn;  // first column any output of this slab needs (t >= s)

  // The call's peak pool use is ~7 pair-grid-sized arrays on the shared
  // design (d = 3 32^3: 55.6 GB measured), ~2x that with pw and the mass
  // orders: map it in one allocation rather than block by block on the
  // first large call (a no-op once the pool holds that much).
  pool_ensure(ctx, static_cast<std::uint64_t>((b->shared_const ? 7.5 : 15.0) * static_cast<double>(LR) *
                                              static_cast<double>(G) * 8.0));

  auto surf = std::make_unique<dfpca_surface>();
  surf->grid = grid;
  surf->kind = DFPCA_SURFACE_COVARIANCE;
  surf->n = out_rows * G;
  surf->row0 = out_row0;
  surf->rows = out_rows;
  surf->values.alloc(static_cast<std::size_t>(surf->n));

  // Shared constant design (dfpca_binned::shared_const): the reference's pw is
  // sw - dm0 [u == v] entry by entry, so the mass moments are closed-form
  // (k_solve_shared) and only pv goes through the pair build and the
  // convolutions.  Used when every kernel window provably holds an
  // off-diagonal pair (a positive off-centre tap on some axis of extent >= 2),
  // i.e. no window can be empty, so the S0 > 0 test can never differ.
  // (DFPCA_GENERAL_PAIRS=1 forces the general path: A/B parity tests)
  bool shared = b->shared_const && std::getenv("DFPCA_GENERAL_PAIRS") == nullptr;
  if (shared) {
    bool some_axis = false;
    for (int k = 0; k < d; ++k) {
      const AxisTaps& a = taps[k];
      some_axis = some_axis || (grid.shape[k] >= 2 && a.R >= 1 && a.t[0][a.R + 1] > 0.0 && a.t[0][a.R - 1] > 0.0);
    }
    shared = some_axis;
  }
  host_mark("surface alloc");
  SharedMoments sh{};
  if (shared) {
    host_mark("shared setup");
    double sw = 0.0;  // the reference's off-band pw entry: ordered sum of (w_i M0) M0
    for (double w : b->pair_weight_h) sw = sw + (w * b->shared_m0) * b->shared_m0;
    sh.sw = sw;
    sh.dm0 = b->shared_dm0;
    // The A / D tables depend only on the axis lengths and taps: built once per
    // context and kept on the device (their host build is O(n^2 R) per axis).
    // (the taps are make_taps(h, spacing) of each axis: those bits key them)
    std::string key = "shared";
    for (int k = 0; k < d; ++k) {
      std::uint64_t hb, sb;
      std::memcpy(&hb, &h[k], sizeof(hb));
      std::memcpy(&sb, &grid.spacing[k], sizeof(sb));
      key += "|" + std::to_string(grid.shape[k]) + ":" + std::to_string(hb) + ":" + std::to_string(sb);
    }
    std::vector<std::size_t> offA(d), offD(d);
    std::size_t total = 0;
    for (int k = 0; k < d; ++k) {
      const i64 n = grid.shape[k];
      offA[k] = total;
      total += 3 * n;
      offD[k] = total;
      total += 9 * n * n;
      sh.n[k] = static_cast<int>(n);
      sh.band[k] = static_cast<int>(taps[k].R + taps[d + k].R);
      sh.inv_n[k] = 1.0f / static_cast<float>(n);
    }
    auto& slot = ctx->table_cache[key];
    if (!slot) {
      std::vector<double> sh_host(total, 0.0);
      for (int k = 0; k < d; ++k) {
        const i64 n = grid.shape[k];
        const AxisTaps& ts = taps[k];
        const AxisTaps& tt = taps[d + k];
        const i64 R = ts.R, Rt = tt.R;
        for (int r = 0; r < 3; ++r)
          for (i64 j = 0; j < n; ++j) {
            double acc = 0.0;
            for (i64 o = -R; o <= R; ++o)
              if (j + o >= 0 && j + o < n) acc += ts.t[r][o + R];
            sh_host[offA[k] + r * n + j] = acc;
          }
        for (int a = 0; a < 3; ++a)
          for (int c = 0; a + c <= 2 && c < 3; ++c)
            for (i64 x = 0; x < n; ++x)
              for (i64 y = 0; y < n; ++y) {
                double acc = 0.0;
                const i64 lo = std::max<i64>({0, x - R, y - Rt}), hi = std::min<i64>({n - 1, x + R, y + Rt});
                for (i64 u = lo; u <= hi; ++u) acc += ts.t[a][u - x + R] * tt.t[c][u - y + Rt];
                sh_host[offD[k] + ((a * 3 + c) * n + x) * n + y] = acc;
              }
      }
      slot = std::make_unique<DevBuf<double>>(total);
      DFPCA_CUDA(cudaMemcpyAsync(slot->get(), sh_host.data(), sizeof(double) * total, cudaMemcpyHostToDevice, st));
      DFPCA_CUDA(cudaStreamSynchronize(st));
    }
    for (int k = 0; k < d; ++k) {
      sh.A[k] = slot->get() + offA[k];
      sh.D[k] = slot->get() + offD[k];
    }
    // per-node products P_a(u) (sep_products' expression order, so the
    // device reads the same bits it would compute) and packed coordinates
    bool fits = d <= 3;
    for (int k = 0; k < d; ++k) fits = fits && grid.shape[k] <= static_cast<i64>(kCoordMask) + 1;
    if (fits) {
      const int ns = sep_stride(d);
      auto& nodes = ctx->table_cache[key + "|nodes"];
      if (!nodes) {
        std::vector<double> host(static_cast<std::size_t>(ns * G + (G + 1) / 2), 0.0);
        unsigned* coord = reinterpret_cast<unsigned*>(host.data() + ns * G);
        std::vector<double> hA(total);
        DFPCA_CUDA(cudaMemcpy(hA.data(), slot->get(), sizeof(double) * total, cudaMemcpyDeviceToHost));
        for (i64 u = 0; u < G; ++u) {
          int j[kMaxDim] = {};
          i64 rest = u;
          for (int k = d - 1; k >= 0; --k) {
            j[k] = static_cast<int>(rest % grid.shape[k]);
            rest /= grid.shape[k];
          }
          unsigned packed = 0;
          for (int k = 0; k < d; ++k) packed |= static_cast<unsigned>(j[k]) << (kCoordBits * k);
          coord[u] = packed;
          auto a = [&](int k, int r) { return hA[offA[k] + r * grid.shape[k] + j[k]]; };
          double z = 1.0;
          for (int k = 0; k < d; ++k) z *= a(k, 0);
          double* row = host.data() + u * ns;
          row[0] = z;
          for (int k = 0; k < d; ++k) {
            double v = 1.0;
            for (int m = 0; m < d; ++m) v *= a(m, m == k ? 1 : 0);
            row[1 + k] = v;
          }
          for (int k = 0; k < d; ++k)
            for (int l = k; l < d; ++l) {
              double v = 1.0;
              for (int m = 0; m < d; ++m) v *= a(m, (m == k) + (m == l));
              row[1 + d + k * d - k * (k - 1) / 2 + (l - k)] = v;
            }
        }
        nodes = std::make_unique<DevBuf<double>>(host.size());
        DFPCA_CUDA(cudaMemcpyAsync(nodes->get(), host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice,
                                   st));
        DFPCA_CUDA(cudaStreamSynchronize(st));
      }
      sh.P = nodes->get();
      sh.coord = reinterpret_cast<const unsigned*>(nodes->get() + ns * G);
      sh.G = G;
    }
  }

  // ---- pair grids (K2) ----
  // one device: the whole G x G grids; a slab: rows [ha, hb) planes, columns
  // from ha (the t window of the slab's outputs), SYRK over its own row tiles
  // and the rest received from the other ranks (shard.hpp, exchange 1)
  DevBuf<double> pw, pv(static_cast<std::size_t>(LR * G));
  if (!shared) pw.alloc(static_cast<std::size_t>(LR * G));
  host_mark("pair buffers");
  ctx->begin_stage("pairs");
  if (sharded) {
    PairWindow win;
    win.row0 = row0;
    win.rows = LR;
    win.col0 = row0;
    win.tm_begin = sa * rn / kShardRowTile;
    win.tm_end = (sb * rn + kShardRowTile - 1) / kShardRowTile;
    double* pwp = shared ? nullptr : pw.get();
    double* pvp = pv.get();
    if (sa < sb)
      build_pair_grids(ctx, b, pwp, pvp, &win,
                       [&](bool pw_syrk) { shard->exchange_pairs(pw_syrk ? pwp : nullptr, pvp, pw_syrk); });
    else if (!pair_grids_sparse(ctx, b))  // idle rank: still takes part in the exchange
      shard->exchange_pairs(nullptr, nullptr, !shared && !b->identical_mass);
  } else {
    build_pair_grids(ctx, b, shared ? nullptr : pw.get(), pv.get());
  }
  ctx->end_stage();

  // for the centering (K5): uploaded while the pair build runs
  DevBuf<double> mean_dev(static_cast<std::size_t>(G));
  DFPCA_CUDA(cudaMemcpyAsync(mean_dev.get(), mean_host, sizeof(double) * G, cudaMemcpyHostToDevice, st));

  // ---- phase T: t-axis passes over row chunks of the pair grids ----
  ctx->begin_stage("moments");
  std::vector<std::unique_ptr<DevBuf<double>>> tpart_store;
  std::map<std::pair<Orders, int>, double*> tpart;
  // t-partials: all t-multi-indices with |a| <= 2 (mass) / <= 1 (value)
  {
    // enumerate leaves of the t-tree
    std::vector<Orders> mass_idx, val_idx;
    std::function<void(int, Orders, int, int, std::vector<Orders>&)> rec =
        [&](int k, Orders o, int used, int mx, std::vector<Orders>& outv) {
          if (k == p) {
            outv.push_back(o);
            return;
          }
          for (int r = 0; r + used <= mx; ++r) {
            Orders q = o;
            q[k] = r;
            rec(k + 1, q, used + r, mx, outv);
          }
        };
    rec(d, Orders{}, 0, 2, mass_idx);
    rec(d, Orders{}, 0, 1, val_idx);
    if (shared) mass_idx.clear();
    for (auto& o : mass_idx) {
      tpart_store.push_back(std::make_unique<DevBuf<double>>(static_cast<std::size_t>(LR * G)));
      tpart[{o, 2}] = tpart_store.back()->get();
    }
    for (auto& o : val_idx) {
      tpart_store.push_back(std::make_unique<DevBuf<double>>(static_cast<std::size_t>(LR * G)));
      tpart[{o, 1}] = tpart_store.back()->get();
    }
    // test aid: NaN-fill the t-partials so an entry read without being
    // written (the upper-triangle trims) poisons the result
    if (std::getenv("DFPCA_POISON"))
      for (auto& buf : tpart_store) DFPCA_CUDA(cudaMemsetAsync(buf->get(), 0xff, buf->bytes(), st));
  }
  // chunk rows (s nodes) so intermediates stay bounded
  // ~2 GiB per level array set (DFPCA_CHUNK_GIB overrides: larger chunks mean
  // fewer, longer pass launches at d = 3)
  i64 budget_bytes = i64(1) << 31;
  if (const char* e = std::getenv("DFPCA_CHUNK_GIB")) budget_bytes = std::max<i64>(1, std::atoll(e)) << 30;
  const i64 budget_elems = std::max<i64>(G, budget_bytes / 8);
  i64 sc = std::max<i64>(1, std::min<i64>(G, budget_elems / std::max<i64>(G, 1) / 4));
  std::vector<TreeAxis> taxes;
  for (int k = p - 1; k >= d; --k) taxes.push_back({k, k - d});
  for (i64 s0 = 0; s0 < (sa < sb ? LR : 0); s0 += sc) {
    const i64 rows = std::min(sc, LR - s0);
    ChunkDims cd;
    cd.rows = rows;
    for (int k = d; k < p; ++k) cd.shape.push_back(grid.shape[k - d]);
    cd.tail = 1;
    std::vector<Leaf> roots;
    if (!shared) {
      Leaf r{};
      r.budget_max = 2;
      r.ptr = pw.get() + s0 * G;
      roots.push_back(r);
    }
    {
      Leaf r{};
      r.budget_max = 1;
      r.ptr = pv.get() + s0 * G;
      roots.push_back(r);
    }
    if (d == 2) {
      // fused two-axis t-phase: the 64x64 t-plane of a row never leaves smem
      TPhase2Spec ts{};
      ts.value_only = shared;
      ts.pw = shared ? nullptr : pw.get() + s0 * G;
      ts.pv = pv.get() + s0 * G;
      ts.rows = rows;
      ts.n1 = grid.shape[0];
      ts.n2 = grid.shape[1];
      const int mo[6][2] = {{0, 0}, {1, 0}, {2, 0}, {0, 1}, {1, 1}, {0, 2}};
      const int vo[3][2] = {{0, 0}, {1, 0}, {0, 1}};
      for (int i = 0; i < 6 && !shared; ++i) {
        Orders o{};
        o[2] = mo[i][0];
        o[3] = mo[i][1];
        ts.mass_out[i] = tpart.at({o, 2}) + s0 * G;
      }
      for (int i = 0; i < 3; ++i) {
        Orders o{};
        o[2] = vo[i][0];
        o[3] = vo[i][1];
        ts.value_out[i] = tpart.at({o, 1}) + s0 * G;
      }
      for (int ax = 0; ax < 2; ++ax) {
        ts.R[ax] = taps[2 + ax].R;
        for (int r = 0; r < 3; ++r) ts.taps[ax][r] = taps[2 + ax].t[r].data();
      }
      // the s-phase below runs in one column chunk with per-tile row trimming
      // (View::tri): a t-partial entry (s, t) is read only if plane(s) <=
      // plane(t) + R_s1 + the planes one 64-column tile spans
      const i64 s_chunk = std::max<i64>(1, std::min<i64>(G, budget_elems / std::max<i64>(G, 1) / 4));
      if (s_chunk >= G - col_lo) {
        ts.s_base = ha * rn + s0;
        ts.rn = rn;
        ts.t1_margin = static_cast<int>(taps[0].R + (64 + rn - 1) / rn);
      }
      if (run_tphase2(ctx, ts)) continue;
    }
    std::vector<std::unique_ptr<DevBuf<double>>> keep;
    auto final_dst = [&](const Orders& o, int bm) -> double* { return tpart.at({o, bm}) + s0 * G; };
    auto final_rs = [&](const Orders&, int) -> i64 { return -1; };
    if (d == 3) {
      // d = 3: the fused two-axis kernel on the contiguous (t2, t3) planes --
      // one plane per (s row, t1), the same passes in the same order as the
      // tree (t3, then t2) -- then one t1 pass; the t3 / t2 partials never
      // reach HBM
      TPhase2Spec ts{};
      ts.value_only = shared;
      ts.pw = shared ? nullptr : pw.get() + s0 * G;
      ts.pv = pv.get() + s0 * G;
      ts.rows = rows * grid.shape[0];
      ts.n1 = grid.shape[1];
      ts.n2 = grid.shape[2];
      const int mo[6][2] = {{0, 0}, {1, 0}, {2, 0}, {0, 1}, {1, 1}, {0, 2}};
      const int vo[3][2] = {{0, 0}, {1, 0}, {0, 1}};
      std::vector<Leaf> planes;
      std::vector<std::unique_ptr<DevBuf<double>>> plane_bufs;
      auto add = [&](int budget, int a2, int a3) -> double* {
        plane_bufs.push_back(std::make_unique<DevBuf<double>>(static_cast<std::size_t>(rows * G)));
        Leaf l{};
        l.ord = Orders{};
        l.ord[4] = a2;
        l.ord[5] = a3;
        l.budget_max = budget;
        l.ptr = plane_bufs.back()->get();
        planes.push_back(l);
        return l.ptr;
      };
      for (int i = 0; i < 6 && !shared; ++i) ts.mass_out[i] = add(2, mo[i][0], mo[i][1]);
      for (int i = 0; i < 3; ++i) ts.value_out[i] = add(1, vo[i][0], vo[i][1]);
      for (int ax = 0; ax < 2; ++ax) {
        ts.R[ax] = taps[4 + ax].R;
        for (int r = 0; r < 3; ++r) ts.taps[ax][r] = taps[4 + ax].t[r].data();
      }
      if (run_tphase2(ctx, ts)) {
        const std::vector<TreeAxis> t1ax = {TreeAxis{3, 0}};
        run_tree(ctx, planes, t1ax, cd, taps, rows * G, taps_dev.get(), keep, final_dst, final_rs, false, -1);
        continue;
      }
    }
    run_tree(ctx, roots, taxes, cd, taps, rows * G, taps_dev.get(), keep, final_dst, final_rs, false,
             -1);
  }

  // ---- phase S: s-axis passes over column chunks, then solve ----
  DevBuf<std::uint8_t> mask_dev;
  if (grid.has_mask) {
    mask_dev.alloc(G);
    DFPCA_CUDA(cudaMemcpyAsync(mask_dev.get(), grid.mask.data(), G, cudaMemcpyHostToDevice, st));
  }
  DevBuf<unsigned long long> cnt(1);
  const i64 list_cap = std::min<i64>(G2, i64(1) << 26);
  DevBuf<i64> list(static_cast<std::size_t>(list_cap));
  DFPCA_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), st));
  // Column chunks of the t-partials.  Only the upper triangle s <= t (flat
  // node order) is smoothed: the covariance is symmetric by construction
  // (the reference averages the (s,t) and (t,s) fits of mirror-image windows,
  // fft_smoother.hpp:730-736), so the lower triangle is the mirror copy
  // written by the symmetrization pass.  A chunk of columns [t0, t0+cols)
  // needs output planes s1 < s1_out and, for the last (s1) pass, input planes
  // s1 < s1_out + R.  A slab (shard.hpp) starts its columns at its first
  // output row, reads its local planes [ha, hb) and writes planes [sa, sb).
  const i64 R0 = taps[0].R;
  i64 tc = std::max<i64>(1, std::min<i64>(G, budget_elems / std::max<i64>(G, 1) / 4));
  // s1 first, then the in-plane axes: the in-plane passes then cover only
  // the output planes (the s1 pass reads the R extra planes once)
  std::vector<TreeAxis> saxes;
  for (int k = 0; k < d; ++k) saxes.push_back({k, k});
  for (i64 t0 = col_lo; t0 < G && sa < sb; t0 += tc) {
    const i64 cols = std::min(tc, G - t0);
    const i64 s1_out = std::min<i64>(sb, (t0 + cols - 1) / rn + 1) - ha;  // local end of output planes
    const i64 s1_in = std::min<i64>(L, s1_out + R0);
    // d = 2 with all columns in one chunk: the per-tile restriction of the
    // pass kernels (View::tri) trims the s rows column tile by column tile
    const bool tri_tiles = d == 2 && t0 == col_lo && cols == G - col_lo;
    ChunkDims cd;
    cd.rows = 1;
    for (int k = 0; k < d; ++k) cd.shape.push_back(grid.shape[k]);
    cd.shape[0] = s1_in;
    cd.tail = cols;
    if (tri_tiles) {
      cd.tri = {2, 3};  // s1 pass, then the s2 pass over the output planes
      cd.tri_params.tri_R = static_cast<int>(R0);
      cd.tri_params.tri_G = cols;
      cd.tri_params.tri_rn = rn;
      cd.tri_params.tri_n1 = L;
      cd.tri_params.tri_row0 = ha;
      cd.tri_params.tri_row_hi = sb;
      cd.tri_params.tri_t0 = t0;
    }
    // the s1 pass writes the output planes [sa, s1_out) only (a slab's own)
    cd.win_k = 0;
    cd.win_lo = sa - ha;
    cd.win_hi = s1_out;
    cd.axis0_first = true;
    const i64 chunk_elems = s1_in * rn * cols;
    // roots: the t-partials viewed along s1 (planes s1 < s1_in, stride rn * G),
    // outer = the in-plane s nodes (stride G), inner = the chunk's columns
    std::vector<Leaf> roots;
    for (auto& kv : tpart) {
      Leaf r;
      r.ord = kv.first.first;
      r.budget_max = kv.first.second;
      r.ptr = kv.second + t0;
      View v;
      v.p = r.ptr;
      v.n = s1_in;
      v.js = rn * G;
      v.outer = rn;
      v.os = G;
      v.inner = cols;
      r.view = v;
      roots.push_back(r);
    }
    std::vector<std::unique_ptr<DevBuf<double>>> keep;
    std::vector<std::unique_ptr<DevBuf<double>>> finals;
    auto final_dst = [&](const Orders&, int) -> double* {
      finals.push_back(std::make_unique<DevBuf<double>>(static_cast<std::size_t>(chunk_elems)));
      return finals.back()->get();
    };
    auto final_rs = [&](const Orders&, int) -> i64 { return -1; };
    SolveGeom sg{};
    sg.npts = s1_out * rn * cols;
    sg.tc = cols;
    sg.t0 = t0;
    sg.gt = G;
    sg.cov = 1;
    sg.upper = 1;
    sg.mask = grid.has_mask ? mask_dev.get() : nullptr;
    sg.row_lo = (sa - ha) * rn;
    sg.row0 = row0;
    sg.out_row0 = out_row0;
    if (sharded) {
      int nch = 0;
      if (tri_ctas(sg, nch) < 0) fail(kConfig, "InvalidArgument", "covariance slab too large for the tiled solve");
    }
    std::vector<Leaf> leaves =
        run_tree(ctx, roots, saxes, cd, taps, chunk_elems, taps_dev.get(), keep, final_dst, final_rs, true, -1);
    MomPtrs mp{};
    for (const Leaf& l : leaves) {
      const int idx = basis.find(l.ord);
      if (l.budget_max == 2) mp.S[idx] = l.ptr;
      else mp.T[idx] = l.ptr;
    }
    ctx->end_stage();
    ctx->begin_stage("solve");
    if (shared) launch_solve_shared(d, ctx, sh, mp, sg, surf->values.get(), cnt.get(), list.get(), list_cap);
    else solve_launcher(p)(ctx, mp, sg, surf->values.get(), cnt.get(), list.get(), list_cap);
    ctx->end_stage();
    ctx->begin_stage("moments");
  }
  unsigned long long n_empty = 0;
  const i64 tiles = (G + 31) / 32;
  const i64 I0 = out_row0 / 32, I1 = (out_row0 + out_rows + 31) / 32;
  auto pstart = [tiles](i64 i) { return i * tiles - i * (i - 1) / 2; };
  const i64 pairs = out_rows > 0 ? pstart(I1) - pstart(I0) : 0;  // (slab rows start on 64-row tiles)
  if (!sharded) {
    // One device: center and mirror without waiting for the empty-window
    // count (read back with the final sync); empty windows, if any, are then
    // refitted by the ladder and re-centered entry by entry (same formula).
    unsigned long long* slot = ctx->pinned_u64(1);
    DFPCA_CUDA(cudaMemcpyAsync(slot, cnt.get(), sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    ctx->end_stage();
    ctx->begin_stage("center");
    if (pairs > 0)
      DFPCA_LAUNCH_PDL(ctx, k_center_mirror, static_cast<unsigned>(pairs), 256, 0, surf->values.get(), mean_dev.get(),
                   grid.has_mask ? mask_dev.get() : nullptr, G, I0, I1, out_row0);
    ctx->end_stage();
    DFPCA_CUDA(cudaStreamSynchronize(st));
    n_empty = *slot;
    tpart_store.clear();
    if (n_empty == 0) {
      *out = surf.release();
      return;
    }
  } else {
    DFPCA_CUDA(cudaMemcpyAsync(&n_empty, cnt.get(), sizeof(n_empty), cudaMemcpyDeviceToHost, st));
    DFPCA_CUDA(cudaStreamSynchronize(st));
    ctx->end_stage();
    tpart_store.clear();
  }
  if (sharded) {
    // every rank must take the same branch before the covariance exchange
    const unsigned long long any_empty = shard->max_over_ranks(n_empty);
    if (any_empty > 0) {
      // Empty kernel windows somewhere: the fallback ladder
      // (fft_smoother.hpp:471-487) gathers windows enlarged up to 1.5^3 h,
      // past the slab halo.  Every rank (all take this branch) runs the
      // whole covariance on its own device -- the one-GPU path, so the
      // ladder and the bits are exactly the one-GPU ones -- and keeps its
      // rows; the rows are complete, so no exchange follows.
      dfpca_surface* full_raw = nullptr;
      run_covariance_impl(ctx, b, grid, h, mean_host, nullptr, &full_raw);
      std::unique_ptr<dfpca_surface> full(full_raw);
      if (out_rows > 0)
        DFPCA_CUDA(cudaMemcpyAsync(surf->values.get(), full->values.get() + out_row0 * G,
                                   sizeof(double) * out_rows * G, cudaMemcpyDeviceToDevice, st));
      DFPCA_CUDA(cudaStreamSynchronize(st));
      *out = surf.release();
      return;
    }
  }

  if (n_empty > 0) {
    if (static_cast<i64>(n_empty) > list_cap)
      fail(kNumeric, "BandwidthTooSmall",
           "binned covariance smoother: too many empty kernel windows");
    ctx->begin_stage("fallback");
    if (shared) {  // not reachable by construction; rebuild both grids for the gathers
      pw.alloc(static_cast<std::size_t>(G2));
      build_pair_grids(ctx, b, pw.get(), pv.get());
    }
    LadderGeom lg{};
    lg.p = p;
    for (int k = 0; k < p; ++k) {
      lg.shape[k] = grid.shape[k % d];
      lg.spacing[k] = grid.spacing[k % d];
      lg.h[k] = h[k % d];
    }
    for (int k = p - 1, s = 1; k >= 0; --k) {
      lg.strides[k] = s;
      s *= static_cast<int>(lg.shape[k]);
    }
    DevBuf<unsigned long long> still(1);
    DFPCA_CUDA(cudaMemsetAsync(still.get(), 0, sizeof(unsigned long long), st));
    DFPCA_LAUNCH(ctx, k_ladder, grid_for(static_cast<i64>(n_empty), 1, 148ll * 8), 256, 0, lg,
                 pw.get(), pv.get(), list.get(), static_cast<i64>(n_empty), surf->values.get(),
                 still.get());
    unsigned long long n_still = 0;
    DFPCA_CUDA(cudaMemcpyAsync(&n_still, still.get(), sizeof(n_still), cudaMemcpyDeviceToHost, st));
    DFPCA_CUDA(cudaStreamSynchronize(st));
    ctx->end_stage();
    if (n_still > 0)
      fail(kNumeric, "BandwidthTooSmall",
           "binned covariance smoother: " + std::to_string(n_still) +
               " node(s) had no binned mass in the kernel window (AllWeightsZero) after 3 window "
               "enlargements");
    if (!sharded) {  // the refitted entries, centered and mirrored like the rest
      DFPCA_LAUNCH(ctx, k_center_list, grid_for(static_cast<i64>(n_empty), 256), 256, 0, surf->values.get(),
                   mean_dev.get(), grid.has_mask ? mask_dev.get() : nullptr, G, list.get(),
                   static_cast<i64>(n_empty));
      DFPCA_CUDA(cudaStreamSynchronize(st));
      *out = surf.release();
      return;
    }
  }

  // ---- center + symmetrize (K5) ----
  ctx->begin_stage("center");
  if (pairs > 0)
    DFPCA_LAUNCH_PDL(ctx, k_center_mirror, static_cast<unsigned>(pairs), 256, 0, surf->values.get(), mean_dev.get(),
                 grid.has_mask ? mask_dev.get() : nullptr, G, I0, I1, out_row0);
  ctx->end_stage();
  if (sharded) {  // exchange 2: the lower-triangle blocks of this slab's rows
    ctx->begin_stage("exchange");
    shard->exchange_cov(surf->values.get());
    ctx->end_stage();
  }
  DFPCA_CUDA(cudaStreamSynchronize(st));
  *out = surf.release();
}

void run_covariance(dfpca_context* ctx, const dfpca_binned* b, const Grid& grid, const double* h,
                    const double* mean_host, dfpca_surface** out) {
  run_covariance_impl(ctx, b, grid, h, mean_host, nullptr, out);
}

}  // namespace dfpca_gpu
