// K3+K4 fused for the 2-d covariance (p = 4 covariates): the last separable
// pass (axis s1) produces all 20 kernel moments of a tile of grid points in
// registers and feeds them straight into the per-node 5x5 local-linear solve,
// so the 15 S-moment and 5 T-moment arrays (320 B/pt written and re-read)
// never reach HBM.  Replaces, for d = 2, the final SeparableConv axis stage
// (conv.hpp:280-331) of every engine plus solve_binned_box
// (fft_smoother.hpp:450-488).
//
// Inputs: the 14 s2-level partials (10 mass-like, 4 value-like) in canonical
// order -- multi-indices (a, b, c) over axes (s2, t1, t2), lexicographic,
// |.| <= 2 for mass and <= 1 for value -- each compact [n(s1)][inner].
// CTA tile: the full s1 extent x 8 contiguous inner columns (64 B rows),
// staged once in shared memory (57 KB).  Each thread owns one column and two
// consecutive s1 outputs: 40 moment accumulators, then two register solves.
#include <algorithm>
#include <utility>

#include "conv.cuh"
#include "fused.cuh"
#include "solve.cuh"

namespace dfpca_gpu {
namespace {

constexpr int kCols = 8;
constexpr int kJB2 = 2;
constexpr int kIn = 14;

struct P4Table {
  int sum[kIn];
  int isval[kIn];
  int eng[kIn][3];
};

__host__ __device__ constexpr int p4_engine(int o0, int o1, int o2, int o3) {
  const int o[4] = {o0, o1, o2, o3};
  const int s = o0 + o1 + o2 + o3;
  if (s == 0) return 0;
  if (s == 1) {
    for (int k = 0; k < 4; ++k)
      if (o[k] == 1) return 1 + k;
  }
  int k = -1, l = -1;
  for (int i = 0; i < 4; ++i) {
    if (o[i] == 2) {
      k = i;
      l = i;
    } else if (o[i] == 1) {
      if (k < 0) k = i;
      else l = i;
    }
  }
  return 1 + 4 + k * 4 - k * (k - 1) / 2 + (l - k);
}

constexpr P4Table make_p4() {
  P4Table t{};
  int idx = 0;
  for (int mx = 2; mx >= 1; --mx)  // mass inputs first (budget 2), then value (budget 1)
    for (int a = 0; a <= mx; ++a)
      for (int b = 0; a + b <= mx; ++b)
        for (int c = 0; a + b + c <= mx; ++c) {
          t.sum[idx] = a + b + c;
          t.isval[idx] = mx == 1;
          for (int r = 0; r < 3; ++r) t.eng[idx][r] = (r + a + b + c <= mx) ? p4_engine(r, a, b, c) : -1;
          ++idx;
        }
  return t;
}

constexpr P4Table kTab = make_p4();

struct Taps1P {
  double t[3][2 * kMaxTemplR + 1];
};

struct Ptrs14 {
  const double* in[kIn];
};

// Accumulates input K's contribution (all its s1 orders) to the moments of
// two consecutive outputs j0, j0+1; every table lookup is a constant
// expression, so the moment slots are registers.
template <int K, int R>
__device__ __forceinline__ void accum_input(const double* sm, int n, int c, int j0, double (&mom)[20][kJB2],
                                            const Taps1P& tp) {
  constexpr int base = kTab.isval[K] ? 15 : 0;
  constexpr int e0 = kTab.eng[K][0], e1 = kTab.eng[K][1], e2 = kTab.eng[K][2];
  const double* colp = sm + K * n * kCols + c;
#pragma unroll
  for (int m = -R; m < kJB2 + R; ++m) {
    const int jm = j0 + m;
    const double x = (jm >= 0 && jm < n) ? colp[jm * kCols] : 0.0;
#pragma unroll
    for (int jj = 0; jj < kJB2; ++jj) {
      const int o = m - jj;
      if (o >= -R && o <= R) {
        if constexpr (e0 >= 0) mom[base + e0][jj] = fma(tp.t[0][o + R], x, mom[base + e0][jj]);
        if constexpr (e1 >= 0) mom[base + e1][jj] = fma(tp.t[1][o + R], x, mom[base + e1][jj]);
        if constexpr (e2 >= 0) mom[base + e2][jj] = fma(tp.t[2][o + R], x, mom[base + e2][jj]);
      }
    }
  }
}

template <int R, int... K>
__device__ __forceinline__ void accum_all(std::integer_sequence<int, K...>, const double* sm, int n, int c,
                                          int j0, double (&mom)[20][kJB2], const Taps1P& tp) {
  (accum_input<K, R>(sm, n, c, j0, mom, tp), ...);
}

// Solve of output JJ of the thread's pair (compile-time JJ keeps mom in registers).
template <int JJ>
__device__ __forceinline__ void solve_point(const double (&mom)[20][kJB2], int j0, int n, i64 col, i64 cols,
                                            i64 s2n, i64 t0, i64 G, const std::uint8_t* __restrict__ mask,
                                            double* __restrict__ out, unsigned long long* __restrict__ cnt,
                                            i64* __restrict__ list, i64 cap) {
  const int s1 = j0 + JJ;
  if (s1 >= n) return;
  const i64 s2 = col / cols, tc = col % cols;
  const i64 s = static_cast<i64>(s1) * s2n + s2, t = t0 + tc;
  const i64 dst = s * G + t;
  if (mask && !(mask[s] && mask[t])) {
    out[dst] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  double S[15], T[5];
#pragma unroll
  for (int i = 0; i < 15; ++i) S[i] = mom[i][JJ];
#pragma unroll
  for (int i = 0; i < 5; ++i) T[i] = mom[15 + i][JJ];
  double b0;
  const int st = solve_local_dev<5>(S, T, b0);
  if (st == kFitEmpty) {
    const unsigned long long q = atomicAdd(cnt, 1ull);
    if (static_cast<i64>(q) < cap) list[q] = dst;
    out[dst] = __longlong_as_double(0x7ff8000000000000ll);
  } else {
    out[dst] = b0;
  }
}

template <int R>
__global__ void __launch_bounds__(256) k_s1_solve_p4(Ptrs14 ip, int n, i64 inner, i64 cols, i64 t0, i64 G,
                                                     i64 s2n, Taps1P tp, const std::uint8_t* __restrict__ mask,
                                                     double* __restrict__ out,
                                                     unsigned long long* __restrict__ cnt,
                                                     i64* __restrict__ list, i64 cap) {
  extern __shared__ double sm[];  // [kIn][n][kCols]
  const i64 c0 = static_cast<i64>(blockIdx.x) * kCols;
#pragma unroll
  for (int k = 0; k < kIn; ++k) {
    const double* src = ip.in[k];
    for (int e = threadIdx.x; e < n * kCols; e += blockDim.x) {
      const int j = e / kCols, c = e % kCols;
      sm[k * n * kCols + e] = (c0 + c < inner) ? src[static_cast<i64>(j) * inner + c0 + c] : 0.0;
    }
  }
  __syncthreads();
  const int c = threadIdx.x % kCols;
  const i64 col = c0 + c;
  for (int j0 = (threadIdx.x / kCols) * kJB2; j0 < n; j0 += (blockDim.x / kCols) * kJB2) {
    double mom[20][kJB2];
#pragma unroll
    for (int i = 0; i < 20; ++i)
#pragma unroll
      for (int jj = 0; jj < kJB2; ++jj) mom[i][jj] = 0.0;
    accum_all<R>(std::make_integer_sequence<int, kIn>{}, sm, n, c, j0, mom, tp);
    if (col >= inner) continue;
    solve_point<0>(mom, j0, n, col, cols, s2n, t0, G, mask, out, cnt, list, cap);
    solve_point<1>(mom, j0, n, col, cols, s2n, t0, G, mask, out, cnt, list, cap);
  }
}

template <int R>
void launch_s1(dfpca_context* ctx, const S1SolveSpec& s, const Taps1P& tp) {
  Ptrs14 ip;
  for (int k = 0; k < kIn; ++k) ip.in[k] = s.in[k];
  const std::size_t smem = sizeof(double) * kIn * s.n * kCols;
  DFPCA_CUDA(cudaFuncSetAttribute(k_s1_solve_p4<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  const i64 blocks = (s.inner + kCols - 1) / kCols;
  DFPCA_LAUNCH(ctx, k_s1_solve_p4<R>, static_cast<unsigned>(blocks), 256, smem, ip, static_cast<int>(s.n),
               s.inner, s.cols, s.t0, s.G, s.s2n, tp, s.mask, s.out, s.cnt, s.list, s.cap);
}

}  // namespace

bool run_s1_solve_p4(dfpca_context* ctx, const S1SolveSpec& s) {
  if (s.R < 1 || s.R > 12 || s.n > 128) return false;
  if (sizeof(double) * kIn * s.n * kCols > 200 * 1024) return false;
  Taps1P tp{};
  for (int r = 0; r < 3; ++r)
    for (int o = 0; o <= 2 * s.R; ++o) tp.t[r][o] = s.taps[r][o];
  switch (s.R) {
#define DFPCA_S1_CASE(r) \
  case r:                \
    launch_s1<r>(ctx, s, tp); \
    return true;
    DFPCA_S1_CASE(1) DFPCA_S1_CASE(2) DFPCA_S1_CASE(3) DFPCA_S1_CASE(4) DFPCA_S1_CASE(5) DFPCA_S1_CASE(6)
    DFPCA_S1_CASE(7) DFPCA_S1_CASE(8) DFPCA_S1_CASE(9) DFPCA_S1_CASE(10) DFPCA_S1_CASE(11) DFPCA_S1_CASE(12)
#undef DFPCA_S1_CASE
    default:
      return false;
  }
}

// Canonical input order of run_s1_solve_p4 (host side mirror of make_p4).
std::vector<std::array<int, 4>> s1_p4_input_order() {
  std::vector<std::array<int, 4>> out;  // {budget, a, b, c}
  for (int mx = 2; mx >= 1; --mx)
    for (int a = 0; a <= mx; ++a)
      for (int b = 0; a + b <= mx; ++b)
        for (int c = 0; a + b + c <= mx; ++c) out.push_back({mx, a, b, c});
  return out;
}

}  // namespace dfpca_gpu
