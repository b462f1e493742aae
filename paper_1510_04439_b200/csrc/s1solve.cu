// K3+K4 fused for the 2-d covariance (p = 4 covariates): the last separable
// pass (axis s1) of all 20 kernel moments and the per-node 5x5 local-linear
// solve, per tile of 4 covariance columns, without the 20 moment arrays ever
// reaching HBM (they are 2 x 20 x 8 B = 320 B/pt of write + re-read when the
// pass and the solve are separate kernels).  Replaces, for d = 2, the final
// SeparableConv axis stage of every engine (conv.hpp:280-331) and
// solve_binned_box (fft_smoother.hpp:450-488).
//
// Per tile (all s1 rows x 4 inner columns, inner = s2 * cols + t):
//   stage   the 14 s2-level partials (10 mass-like, 4 value-like, canonical
//           order, see s1_p4_input_order) into shared memory with cp.async,
//           double-buffered across the persistent loop;
//   phase 1 each (input, column, 8-row block) work item convolves along s1
//           and writes its 1-3 moment orders into a shared-memory moment tile
//           (each moment comes from exactly one input, so no accumulation);
//   phase 2 one thread per node with s <= t reads its 20 moments and runs the
//           register LDLT solve (solve.cuh).
// Only the rows the upper triangle needs are staged (s1 < s1_out + R) and
// solved (s1 < s1_out), as in the trimmed axis passes.
#include <algorithm>
#include <array>
#include <vector>

#include "conv.cuh"
#include "s1solve.cuh"
#include "solve.cuh"

namespace dfpca_gpu {
namespace {

constexpr int kIn = 14;
constexpr int kTC = 4;    // inner columns per tile
constexpr int kJ = 8;     // rows per work item
constexpr int kMaxRows = 64;

struct P4Tab {
  int nord[kIn];      // orders the input contributes (1..3)
  int slot[kIn][3];   // moment slot per order: 0..14 S, 15..19 T
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
  return 1 + 4 + k * 4 - k * (k - 1) / 2 + (l - k);  // MomentBasis::quadratic
}

P4Tab make_tab() {
  P4Tab t{};
  int idx = 0;
  for (int mx = 2; mx >= 1; --mx)
    for (int a = 0; a <= mx; ++a)
      for (int b = 0; a + b <= mx; ++b)
        for (int c = 0; a + b + c <= mx; ++c) {
          t.nord[idx] = mx - (a + b + c) + 1;
          for (int r = 0; r < 3; ++r)
            t.slot[idx][r] = (r + a + b + c <= mx) ? (mx == 1 ? 15 : 0) + p4_engine(r, a, b, c) : -1;
          ++idx;
        }
  return t;
}

struct Taps1 {
  double t[3][2 * kMaxTemplR + 1];
};

struct In14 {
  const double* p[kIn];
};

__device__ inline void cpa16(void* smem, const void* gmem, int bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ inline void cpa8(void* smem, const void* gmem, int bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}

// One work item: input column `col` convolved along s1 for rows j0..j0+7,
// its NO orders written to their moment slots.
template <int R, int NO>
__device__ __forceinline__ void item_moments(const double* __restrict__ col, int j0, int rows, int nout,
                                             const int* slot, const Taps1& tp, double* __restrict__ mom, int c) {
  double acc[NO][kJ];
#pragma unroll
  for (int r = 0; r < NO; ++r)
#pragma unroll
    for (int jj = 0; jj < kJ; ++jj) acc[r][jj] = 0.0;
#pragma unroll
  for (int m = -R; m < kJ + R; ++m) {
    const int jm = j0 + m;
    const double x = (jm >= 0 && jm < rows) ? col[jm * kTC] : 0.0;
#pragma unroll
    for (int jj = 0; jj < kJ; ++jj) {
      const int o = m - jj;
      if (o >= -R && o <= R) {
#pragma unroll
        for (int r = 0; r < NO; ++r) acc[r][jj] = fma(tp.t[r][o + R], x, acc[r][jj]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < NO; ++r) {
    double* m0 = mom + (slot[r] * kMaxRows) * kTC + c;
#pragma unroll
    for (int jj = 0; jj < kJ; ++jj)
      if (j0 + jj < nout) m0[(j0 + jj) * kTC] = acc[r][jj];
  }
}

template <int R, int VEC>
__global__ void __launch_bounds__(256) k_s1_solve(In14 ip, P4Tab tab, Taps1 tp, int n1, int inner, int cols,
                                                  int t0, int s2n, i64 G, int triR,
                                                  const std::uint8_t* __restrict__ mask, double* __restrict__ out,
                                                  unsigned long long* __restrict__ cnt, i64* __restrict__ list,
                                                  i64 cap) {
  extern __shared__ __align__(16) double sm[];
  const int in_elems = kIn * kMaxRows * kTC;
  double* mom = sm + 2 * in_elems;  // [20][kMaxRows][kTC]
  const int n_tiles = (inner + kTC - 1) / kTC;
  // rows of a tile: s1_out from the largest t of its columns (upper triangle)
  auto extent = [&](int c0, int& rows, int& nout) {
    const int c1 = min(c0 + kTC, inner) - 1;
    const int tmax = (c0 / cols == c1 / cols) ? t0 + c1 % cols : t0 + cols - 1;
    nout = min(n1, tmax / s2n + 1);
    rows = min(n1, nout + triR);
  };
  auto issue = [&](int tile, int buf) {
    const int c0 = tile * kTC;
    int rows, nout;
    extent(c0, rows, nout);
    double* dst = sm + buf * in_elems;
    const int avail_cols = inner - c0;
#pragma unroll
    for (int k = 0; k < kIn; ++k) {  // compile-time k keeps the pointer table in registers
      const double* src = ip.p[k];
      for (int e = threadIdx.x * VEC; e < rows * kTC; e += blockDim.x * VEC) {
        const int j = e / kTC, c = e % kTC;
        const int avail = avail_cols - c;
        const int bytes = avail >= VEC ? 8 * VEC : (avail > 0 ? 8 * avail : 0);
        const double* g = bytes ? src + static_cast<i64>(j) * inner + c0 + c : src;
        double* d = dst + (k * kMaxRows + j) * kTC + c;
        if (VEC == 2) cpa16(d, g, bytes);
        else cpa8(d, g, bytes);
      }
    }
  };
  int buf = 0;
  int tile = blockIdx.x;
  if (tile < n_tiles) issue(tile, 0);
  asm volatile("cp.async.commit_group;\n" ::);
  for (; tile < n_tiles; tile += gridDim.x) {
    const int next = tile + gridDim.x;
    if (next < n_tiles) issue(next, buf ^ 1);
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();
    const int c0 = tile * kTC;
    int rows, nout;
    extent(c0, rows, nout);
    const double* in = sm + buf * in_elems;
    // phase 1: moments into shared memory
    const int jblocks = (nout + kJ - 1) / kJ;
    for (int item = threadIdx.x; item < kIn * kTC * jblocks; item += blockDim.x) {
      const int k = item / (kTC * jblocks);
      const int rem = item - k * kTC * jblocks;
      const int c = rem % kTC, j0 = (rem / kTC) * kJ;
      const double* col = in + k * kMaxRows * kTC + c;
      const int no = tab.nord[k];
      const int slot[3] = {tab.slot[k][0], tab.slot[k][1], tab.slot[k][2]};
      if (no == 3) item_moments<R, 3>(col, j0, rows, nout, slot, tp, mom, c);
      else if (no == 2) item_moments<R, 2>(col, j0, rows, nout, slot, tp, mom, c);
      else item_moments<R, 1>(col, j0, rows, nout, slot, tp, mom, c);
    }
    __syncthreads();
    // phase 2: one solve per node with s <= t
    for (int pt = threadIdx.x; pt < nout * kTC; pt += blockDim.x) {
      const int j = pt / kTC, c = pt % kTC;
      const int col = c0 + c;
      if (col >= inner) continue;
      const int s2 = col / cols, tc = col - s2 * cols;
      const i64 s = static_cast<i64>(j) * s2n + s2, t = t0 + tc;
      if (s > t) continue;
      const i64 dst = s * G + t;
      if (mask && !(mask[s] && mask[t])) {
        out[dst] = __longlong_as_double(0x7ff8000000000000ll);
        continue;
      }
      double S[15], T[5];
#pragma unroll
      for (int i = 0; i < 15; ++i) S[i] = mom[(i * kMaxRows + j) * kTC + c];
#pragma unroll
      for (int i = 0; i < 5; ++i) T[i] = mom[((15 + i) * kMaxRows + j) * kTC + c];
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
    __syncthreads();  // buffers are reused by the next iteration's prefetch
    buf ^= 1;
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
}

template <int R>
void launch(dfpca_context* ctx, const S1SolveSpec& s, const P4Tab& tab, const Taps1& tp) {
  In14 ip;
  for (int k = 0; k < kIn; ++k) ip.p[k] = s.in[k];
  const std::size_t smem = sizeof(double) * (2 * kIn * kMaxRows * kTC + 20 * kMaxRows * kTC);
  bool vec2 = (s.inner % 2 == 0);
  for (int k = 0; k < kIn; ++k) vec2 = vec2 && reinterpret_cast<std::uintptr_t>(s.in[k]) % 16 == 0;
  auto kern = vec2 ? k_s1_solve<R, 2> : k_s1_solve<R, 1>;
  DFPCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
  const i64 tiles = (s.inner + kTC - 1) / kTC;
  const unsigned grid = static_cast<unsigned>(std::min<i64>(tiles, static_cast<i64>(std::max(per_sm, 1)) * ctx->sm_count));
  if (vec2)
    DFPCA_LAUNCH(ctx, (k_s1_solve<R, 2>), grid, 256, smem, ip, tab, tp, static_cast<int>(s.n),
                 static_cast<int>(s.inner), static_cast<int>(s.cols), static_cast<int>(s.t0), static_cast<int>(s.s2n),
                 s.G, s.R, s.mask, s.out, s.cnt, s.list, s.cap);
  else
    DFPCA_LAUNCH(ctx, (k_s1_solve<R, 1>), grid, 256, smem, ip, tab, tp, static_cast<int>(s.n),
                 static_cast<int>(s.inner), static_cast<int>(s.cols), static_cast<int>(s.t0), static_cast<int>(s.s2n),
                 s.G, s.R, s.mask, s.out, s.cnt, s.list, s.cap);
}

}  // namespace

bool run_s1_solve_p4(dfpca_context* ctx, const S1SolveSpec& s) {
  if (s.R < 1 || s.R > 12 || s.n > kMaxRows || s.inner >= (1ll << 31) || s.t0 + s.cols >= (1ll << 31)) return false;
  static const P4Tab tab = make_tab();
  Taps1 tp{};
  for (int r = 0; r < 3; ++r)
    for (int o = 0; o <= 2 * s.R; ++o) tp.t[r][o] = s.taps[r][o];
  switch (s.R) {
#define DFPCA_S1_CASE(r) \
  case r:                \
    launch<r>(ctx, s, tab, tp); \
    return true;
    DFPCA_S1_CASE(1) DFPCA_S1_CASE(2) DFPCA_S1_CASE(3) DFPCA_S1_CASE(4) DFPCA_S1_CASE(5) DFPCA_S1_CASE(6)
    DFPCA_S1_CASE(7) DFPCA_S1_CASE(8) DFPCA_S1_CASE(9) DFPCA_S1_CASE(10) DFPCA_S1_CASE(11) DFPCA_S1_CASE(12)
#undef DFPCA_S1_CASE
    default:
      return false;
  }
}

std::vector<std::array<int, 4>> s1_p4_input_order() {
  std::vector<std::array<int, 4>> out;  // {budget, a, b, c}
  for (int mx = 2; mx >= 1; --mx)
    for (int a = 0; a <= mx; ++a)
      for (int b = 0; a + b <= mx; ++b)
        for (int c = 0; a + b + c <= mx; ++c) out.push_back({mx, a, b, c});
  return out;
}

}  // namespace dfpca_gpu
