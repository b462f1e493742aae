// K3: one separable convolution pass along one axis, producing up to three
// moment orders from a single read of the input (tree-factored moments).
//
// Replaces AxisConv::run_line / SeparableConv::convolve_axis
// (conv.hpp:161-201, 280-331).  out[j] = sum_{o=-R..R} taps[o+R] * in[j+o]
// with zero extension beyond the axis, accumulated in ascending o exactly as
// the reference's direct path (conv.hpp:165-173).  The reference switches to
// overlap-add FFT for >= 33 taps (conv.hpp:73); the device path stays direct
// (the FP64 pass is FMA-bound, not transform-bound, at these axis lengths),
// which is the exact-arithmetic twin of the FFT result.
//
// Layout: the full axis extent of a tile of 32 columns (or 32 lines when the
// axis is the contiguous one) is staged once in shared memory, so every input
// element is read from HBM exactly once per pass; each thread then produces a
// block of JB consecutive outputs whose taps are kernel parameters (constant
// bank operands of DFMA, no registers), with the loop over stencil offsets
// fully unrolled for the radius R.
#include <algorithm>
#include <cstdint>

#include "conv.cuh"

namespace dfpca_gpu {
namespace {

constexpr int kTile = 32;  // columns (or lines) per CTA
constexpr int kJB = 8;     // outputs per thread along the axis
constexpr int kMaxN = 128; // longest axis staged whole in shared memory

struct TapsP {
  double t[3][2 * kMaxTemplR + 1];
};

__device__ inline void cp_async_c16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ inline void cp_async_c8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ inline void cp_async_commit_c() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ inline void cp_async_wait_c() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Columns variant: the axis is not the contiguous one (inner >= 16).
// Persistent CTAs walk the tiles (outer index, 32-column chunk); the next
// tile's full-axis column block is copied into the other half of a
// double-buffered shared-memory ring with cp.async while the current one is
// convolved, so the HBM reads overlap the FMA work.
// One thread's kJB outputs along the axis from a staged column; CHECK
// selects bounds-checked loads (tile edges) or the plain interior path.
template <int R, int NO, bool CHECK>
__device__ __forceinline__ void conv_block(const double* __restrict__ col, int j0, int rows, const TapsP& tp,
                                           double (&acc)[NO][kJB]) {
#pragma unroll
  for (int r = 0; r < NO; ++r)
#pragma unroll
    for (int jj = 0; jj < kJB; ++jj) acc[r][jj] = 0.0;
#pragma unroll
  for (int m = -R; m < kJB + R; ++m) {
    const int jm = j0 + m;
    const double x = CHECK ? ((jm >= 0 && jm < rows) ? col[jm * kTile] : 0.0) : col[jm * kTile];
#pragma unroll
    for (int jj = 0; jj < kJB; ++jj) {
      const int o = m - jj;
      if (o >= -R && o <= R) {
#pragma unroll
        for (int r = 0; r < NO; ++r) acc[r][jj] = fma(tp.t[r][o + R], x, acc[r][jj]);
      }
    }
  }
}

template <int R, int NO, int VEC>
__global__ void __launch_bounds__(256) k_pass_cols(View in, View o0, View o1, View o2, TapsP tp) {
  extern __shared__ __align__(16) double sm[];  // [2][n][kTile]
  const int n = static_cast<int>(in.n);
  const int inner = static_cast<int>(in.inner);
  const int chunks = (inner + kTile - 1) / kTile;
  const int n_tiles = static_cast<int>(in.outer) * chunks;
  const int tile_elems = n * kTile;
  const int tri = in.tri, triR = in.tri_R, triG = static_cast<int>(in.tri_G), tri_rn = static_cast<int>(in.tri_rn),
            tri_n1 = static_cast<int>(in.tri_n1);
  // rows to stage and outputs to produce for a tile (all of them unless the
  // upper-triangle restriction applies, see View::tri); 32-bit integer math
  auto extent = [&](int ob, int c0, int& rows, int& nout) {
    rows = n;
    nout = n;
    if (tri == 0) return;
    const int c1 = (c0 + kTile < inner ? c0 + kTile : inner) - 1;
    const int tmax = (c0 / triG == c1 / triG) ? c1 % triG : triG - 1;
    const int s1_out = tmax / tri_rn + 1;
    if (tri == 1) {
      const int s1_in = s1_out + triR < tri_n1 ? s1_out + triR : tri_n1;
      if (ob >= s1_in) rows = nout = 0;
    } else {
      nout = s1_out < n ? s1_out : n;
      rows = nout + triR < n ? nout + triR : n;
    }
  };
  auto issue = [&](int tile, int buf) {
    const int ob = tile / chunks;
    const int c0 = (tile - ob * chunks) * kTile;
    int rows, nout;
    extent(ob, c0, rows, nout);
    const double* src = in.p + ob * in.os + c0;
    double* dst = sm + buf * tile_elems;
    const int avail_cols = inner - c0;
    for (int e = threadIdx.x * VEC; e < rows * kTile; e += blockDim.x * VEC) {
      const int j = e / kTile, c = e % kTile;
      const int avail = avail_cols - c;
      const int bytes = avail >= VEC ? 8 * VEC : (avail > 0 ? 8 * avail : 0);
      const double* g = bytes ? src + j * in.js + c : in.p;
      if (VEC == 2) cp_async_c16(dst + e, g, bytes);
      else cp_async_c8(dst + e, g, bytes);
    }
  };
  int buf = 0;
  int tile = blockIdx.x;
  if (tile < n_tiles) issue(tile, 0);
  cp_async_commit_c();
  const int c = threadIdx.x % kTile;
  for (; tile < n_tiles; tile += gridDim.x) {
    const int next = tile + gridDim.x;
    if (next < n_tiles) issue(next, buf ^ 1);
    cp_async_commit_c();
    cp_async_wait_c<1>();
    __syncthreads();
    const int ob = tile / chunks;
    const int c0 = (tile - ob * chunks) * kTile;
    int rows, nout;
    extent(ob, c0, rows, nout);
    const double* col = sm + buf * tile_elems + c;
    const bool col_ok = c0 + c < inner;
    double* b0 = o0.p + ob * o0.os + c0 + c;
    double* b1 = o1.p + ob * o1.os + c0 + c;
    double* b2 = o2.p + ob * o2.os + c0 + c;
    for (int j0 = (threadIdx.x / kTile) * kJB; j0 < nout; j0 += (blockDim.x / kTile) * kJB) {
      double acc[NO][kJB];
      if (j0 >= R && j0 + kJB + R <= rows)
        conv_block<R, NO, false>(col, j0, rows, tp, acc);
      else
        conv_block<R, NO, true>(col, j0, rows, tp, acc);
      if (col_ok) {
#pragma unroll
        for (int jj = 0; jj < kJB; ++jj) {
          const int j = j0 + jj;
          if (j < nout) {
            b0[j * o0.js] = acc[0][jj];
            if (NO > 1) b1[j * o1.js] = acc[NO > 1 ? 1 : 0][jj];
            if (NO > 2) b2[j * o2.js] = acc[NO > 2 ? 2 : 0][jj];
          }
        }
      }
    }
    __syncthreads();  // everyone is done with this buffer before it is refilled
    buf ^= 1;
  }
  cp_async_wait_c<0>();
}

// Lines variant: the axis is the contiguous one (inner == 1); a CTA stages
// kTile consecutive lines, row-padded to avoid bank conflicts.
template <int R, int NO>
__global__ void __launch_bounds__(256) k_pass_rows(View in, View o0, View o1, View o2, TapsP tp) {
  extern __shared__ double sm[];  // [kTile][n + 1] input, then NO output tiles of the same shape
  const i64 n = in.n;
  const i64 ld = n + 1;
  double* so = sm + kTile * ld;
  const i64 l0 = static_cast<i64>(blockIdx.x) * kTile;
  for (int e = threadIdx.x; e < n * kTile; e += blockDim.x) {
    const int l = e / n, j = e % n;
    sm[l * ld + j] = (l0 + l < in.outer) ? in.p[(l0 + l) * in.os + j * in.js] : 0.0;
  }
  __syncthreads();
  const int l = threadIdx.x % kTile;
  const bool line_ok = l0 + l < in.outer;
  for (int j0 = (threadIdx.x / kTile) * kJB; j0 < n; j0 += (blockDim.x / kTile) * kJB) {
    double acc[NO][kJB];
#pragma unroll
    for (int r = 0; r < NO; ++r)
#pragma unroll
      for (int jj = 0; jj < kJB; ++jj) acc[r][jj] = 0.0;
#pragma unroll
    for (int m = -R; m < kJB + R; ++m) {
      const int jm = j0 + m;
      const double x = (jm >= 0 && jm < n) ? sm[l * ld + jm] : 0.0;
#pragma unroll
      for (int jj = 0; jj < kJB; ++jj) {
        const int o = m - jj;
        if (o >= -R && o <= R) {
#pragma unroll
          for (int r = 0; r < NO; ++r) acc[r][jj] = fma(tp.t[r][o + R], x, acc[r][jj]);
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < kJB; ++jj) {
      const i64 j = j0 + jj;
      if (j < n) {
#pragma unroll
        for (int r = 0; r < NO; ++r) so[(r * kTile + l) * ld + j] = acc[r][jj];
      }
    }
  }
  __syncthreads();
  (void)line_ok;
  // coalesced write-back: consecutive threads -> consecutive j of one line
  for (int e = threadIdx.x; e < n * kTile; e += blockDim.x) {
    const int ll = e / n, j = e % n;
    if (l0 + ll >= in.outer) continue;
    o0.p[(l0 + ll) * o0.os + j * o0.js] = so[(0 * kTile + ll) * ld + j];
    if (NO > 1) o1.p[(l0 + ll) * o1.os + j * o1.js] = so[(1 * kTile + ll) * ld + j];
    if (NO > 2) o2.p[(l0 + ll) * o2.os + j * o2.js] = so[(2 * kTile + ll) * ld + j];
  }
}

// ---------------------------------------------------------------------------
// Fused 2-axis t-phase.  One CTA per pair-grid row s: the t-plane [n1][n2]
// is staged once (row pitch n2+1 against bank conflicts); for each t2-order
// the t2 pass writes a shared-memory plane, and the t1 pass over it writes
// the final t-partials straight to HBM, coalesced along t2.  Both axes use the
// same template radius R (the narrower axis is zero-padded).
struct Taps2P {
  double t[2][3][2 * kMaxTemplR + 1];
};

template <int R, int ORD>
__device__ inline void tp_conv_rows(const double* X, double* Y, int n1, int n2, int ld,
                                    const Taps2P& tp) {
  // Y[l][j] = sum_o taps[t2][order][o] X[l][j+o]  (lines l = t1, axis t2)
  const int nb = (n2 + kJB - 1) / kJB;
  for (int item = threadIdx.x; item < n1 * nb; item += blockDim.x) {
    const int l = item % n1, j0 = (item / n1) * kJB;
    double acc[kJB];
#pragma unroll
    for (int jj = 0; jj < kJB; ++jj) acc[jj] = 0.0;
#pragma unroll
    for (int m = -R; m < kJB + R; ++m) {
      const int jm = j0 + m;
      const double x = (jm >= 0 && jm < n2) ? X[l * ld + jm] : 0.0;
#pragma unroll
      for (int jj = 0; jj < kJB; ++jj) {
        const int o = m - jj;
        if (o >= -R && o <= R) acc[jj] = fma(tp.t[1][ORD][o + R], x, acc[jj]);
      }
    }
#pragma unroll
    for (int jj = 0; jj < kJB; ++jj)
      if (j0 + jj < n2) Y[l * ld + j0 + jj] = acc[jj];
  }
}

template <int R, int NO>
__device__ inline void tp_conv_cols(const double* Y, int n1, int n2, int ld, double* const* outs,
                                    i64 row_off, const Taps2P& tp) {
  // out_r[j][c] = sum_o taps[t1][r][o] Y[j+o][c]   (axis t1, columns c = t2)
  const int nb = (n1 + kJB - 1) / kJB;
  for (int item = threadIdx.x; item < n2 * nb; item += blockDim.x) {
    const int c = item % n2, j0 = (item / n2) * kJB;
    double acc[NO][kJB];
#pragma unroll
    for (int r = 0; r < NO; ++r)
#pragma unroll
      for (int jj = 0; jj < kJB; ++jj) acc[r][jj] = 0.0;
#pragma unroll
    for (int m = -R; m < kJB + R; ++m) {
      const int jm = j0 + m;
      const double x = (jm >= 0 && jm < n1) ? Y[jm * ld + c] : 0.0;
#pragma unroll
      for (int jj = 0; jj < kJB; ++jj) {
        const int o = m - jj;
        if (o >= -R && o <= R) {
#pragma unroll
          for (int r = 0; r < NO; ++r) acc[r][jj] = fma(tp.t[0][r][o + R], x, acc[r][jj]);
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < kJB; ++jj) {
      const int j = j0 + jj;
      if (j < n1) {
#pragma unroll
        for (int r = 0; r < NO; ++r) outs[r][row_off + static_cast<i64>(j) * n2 + c] = acc[r][jj];
      }
    }
  }
}

struct TPhaseOut {
  double* m[6];
  double* v[3];
};

template <int R>
__global__ void __launch_bounds__(256) k_tphase2(const double* __restrict__ pw, const double* __restrict__ pv,
                                                 i64 rows, int n1, int n2, TPhaseOut out, Taps2P tp) {
  extern __shared__ double sm[];
  const int ld = n2 + 1;
  const int pe = n1 * ld;  // padded plane
  double* Y = sm + 2 * pe;
  const i64 plane = static_cast<i64>(n1) * n2;
  // Planes of this CTA in order: (s, pw), (s, pv), (s + grid, pw), ...; the
  // next plane is copied into the other X buffer (cp.async, 8-byte granules
  // because of the bank-conflict padding) while the current one is convolved.
  auto issue = [&](i64 q, int buf) {
    const i64 s = q >> 1;
    const double* src = ((q & 1) ? pv : pw) + s * plane;
    double* X = sm + buf * pe;
    for (int e = threadIdx.x; e < plane; e += blockDim.x) cp_async_c8(X + (e / n2) * ld + e % n2, src + e, 8);
  };
  const i64 q_end = 2 * rows;
  const i64 q_step = 2 * static_cast<i64>(gridDim.x);
  i64 q = 2 * static_cast<i64>(blockIdx.x);
  int buf = 0;
  if (q < q_end) issue(q, 0);
  cp_async_commit_c();
  while (q < q_end) {
    const i64 next = (q & 1) ? q - 1 + q_step : q + 1;
    if (next < q_end) issue(next, buf ^ 1);
    cp_async_commit_c();
    cp_async_wait_c<1>();
    __syncthreads();
    const double* X = sm + buf * pe;
    const i64 off = (q >> 1) * plane;
    const int pass = static_cast<int>(q & 1);
    const int max_order = pass == 0 ? 2 : 1;
    for (int r2 = 0; r2 <= max_order; ++r2) {
      if (r2 == 0) tp_conv_rows<R, 0>(X, Y, n1, n2, ld, tp);
      else if (r2 == 1) tp_conv_rows<R, 1>(X, Y, n1, n2, ld, tp);
      else tp_conv_rows<R, 2>(X, Y, n1, n2, ld, tp);
      __syncthreads();
      if (pass == 0) {
        if (r2 == 0) {
          double* o[3] = {out.m[0], out.m[1], out.m[2]};
          tp_conv_cols<R, 3>(Y, n1, n2, ld, o, off, tp);
        } else if (r2 == 1) {
          double* o[2] = {out.m[3], out.m[4]};
          tp_conv_cols<R, 2>(Y, n1, n2, ld, o, off, tp);
        } else {
          double* o[1] = {out.m[5]};
          tp_conv_cols<R, 1>(Y, n1, n2, ld, o, off, tp);
        }
      } else {
        if (r2 == 0) {
          double* o[2] = {out.v[0], out.v[1]};
          tp_conv_cols<R, 2>(Y, n1, n2, ld, o, off, tp);
        } else {
          double* o[1] = {out.v[2]};
          tp_conv_cols<R, 1>(Y, n1, n2, ld, o, off, tp);
        }
      }
      __syncthreads();
    }
    buf ^= 1;
    q = next;
  }
  cp_async_wait_c<0>();
}

// Generic pass: any radius, any axis length; one thread per output element.
__global__ void k_pass_generic(View in, View o0, View o1, View o2, int n_out,
                               const double* __restrict__ taps, int R) {
  const i64 total = in.outer * in.n * in.inner;
  const int W = 2 * R + 1;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 i = e % in.inner;
    const i64 j = (e / in.inner) % in.n;
    const i64 ob = e / (in.inner * in.n);
    const double* src = in.p + ob * in.os + i;
    const i64 olo = j - R < 0 ? -j : -R;
    const i64 ohi = j + R > in.n - 1 ? in.n - 1 - j : R;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (i64 o = olo; o <= ohi; ++o) {
      const double x = src[(j + o) * in.js];
      a0 = fma(taps[o + R], x, a0);
      if (n_out > 1) a1 = fma(taps[W + o + R], x, a1);
      if (n_out > 2) a2 = fma(taps[2 * W + o + R], x, a2);
    }
    o0.p[ob * o0.os + j * o0.js + i] = a0;
    if (n_out > 1) o1.p[ob * o1.os + j * o1.js + i] = a1;
    if (n_out > 2) o2.p[ob * o2.os + j * o2.js + i] = a2;
  }
}

template <int R, int NO>
void launch_tiled(dfpca_context* ctx, const PassSpec& s, const TapsP& tp) {
  const View& in = s.in;
  const View o1 = s.n_out > 1 ? s.out[1] : s.out[0];
  const View o2 = s.n_out > 2 ? s.out[2] : s.out[0];
  if (in.inner == 1) {
    const i64 blocks = (in.outer + kTile - 1) / kTile;
    const std::size_t smem = sizeof(double) * kTile * (in.n + 1) * (1 + NO);
    if (smem > 48 * 1024)
      DFPCA_CUDA(cudaFuncSetAttribute(k_pass_rows<R, NO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    DFPCA_LAUNCH(ctx, (k_pass_rows<R, NO>), static_cast<unsigned>(blocks), 256, smem, in,
                 s.out[0], o1, o2, tp);
  } else {
    const i64 tiles = in.outer * ((in.inner + kTile - 1) / kTile);
    const std::size_t smem = sizeof(double) * 2 * kTile * in.n;
    const bool vec2 = (in.os % 2 == 0) && (in.js % 2 == 0) &&
                      (reinterpret_cast<std::uintptr_t>(in.p) % 16 == 0);
    auto kern = vec2 ? k_pass_cols<R, NO, 2> : k_pass_cols<R, NO, 1>;
    if (smem > 48 * 1024)
      DFPCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
    const i64 blocks = std::min<i64>(tiles, static_cast<i64>(std::max(per_sm, 1)) * ctx->sm_count);
    if (vec2)
      DFPCA_LAUNCH(ctx, (k_pass_cols<R, NO, 2>), static_cast<unsigned>(blocks), 256, smem, in, s.out[0], o1,
                   o2, tp);
    else
      DFPCA_LAUNCH(ctx, (k_pass_cols<R, NO, 1>), static_cast<unsigned>(blocks), 256, smem, in, s.out[0], o1,
                   o2, tp);
  }
}

template <int R>
void launch_r(dfpca_context* ctx, const PassSpec& s, const TapsP& tp) {
  switch (s.n_out) {
    case 1: launch_tiled<R, 1>(ctx, s, tp); break;
    case 2: launch_tiled<R, 2>(ctx, s, tp); break;
    default: launch_tiled<R, 3>(ctx, s, tp); break;
  }
}

void launch_by_radius(dfpca_context* ctx, const PassSpec& s, const TapsP& tp) {
  switch (s.R) {
#define DFPCA_R_CASE(r) \
  case r:               \
    launch_r<r>(ctx, s, tp); \
    break;
    DFPCA_R_CASE(0) DFPCA_R_CASE(1) DFPCA_R_CASE(2) DFPCA_R_CASE(3) DFPCA_R_CASE(4)
    DFPCA_R_CASE(5) DFPCA_R_CASE(6) DFPCA_R_CASE(7) DFPCA_R_CASE(8) DFPCA_R_CASE(9)
    DFPCA_R_CASE(10) DFPCA_R_CASE(11) DFPCA_R_CASE(12) DFPCA_R_CASE(13) DFPCA_R_CASE(14)
    DFPCA_R_CASE(15) DFPCA_R_CASE(16) DFPCA_R_CASE(17) DFPCA_R_CASE(18) DFPCA_R_CASE(19)
    DFPCA_R_CASE(20) DFPCA_R_CASE(21) DFPCA_R_CASE(22) DFPCA_R_CASE(23) DFPCA_R_CASE(24)
#undef DFPCA_R_CASE
    default:
      break;
  }
}

template <int R>
void launch_tphase2(dfpca_context* ctx, const TPhase2Spec& s, const Taps2P& tp) {
  TPhaseOut out;
  for (int i = 0; i < 6; ++i) out.m[i] = s.mass_out[i];
  for (int i = 0; i < 3; ++i) out.v[i] = s.value_out[i];
  const int n1 = static_cast<int>(s.n1), n2 = static_cast<int>(s.n2);
  const std::size_t smem = sizeof(double) * 3 * n1 * (n2 + 1);
  DFPCA_CUDA(cudaFuncSetAttribute(k_tphase2<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tphase2<R>, 256, smem);
  const unsigned grid =
      static_cast<unsigned>(std::min<i64>(s.rows, static_cast<i64>(std::max(per_sm, 1)) * ctx->sm_count));
  DFPCA_LAUNCH(ctx, k_tphase2<R>, grid, 256, smem, s.pw, s.pv, s.rows, n1, n2, out, tp);
}

void launch_tphase2_r(dfpca_context* ctx, const TPhase2Spec& s, const Taps2P& tp, int R) {
  switch (R) {
#define DFPCA_T_CASE(r) \
  case r:               \
    launch_tphase2<r>(ctx, s, tp); \
    break;
    DFPCA_T_CASE(1) DFPCA_T_CASE(2) DFPCA_T_CASE(3) DFPCA_T_CASE(4) DFPCA_T_CASE(5) DFPCA_T_CASE(6)
    DFPCA_T_CASE(7) DFPCA_T_CASE(8) DFPCA_T_CASE(9) DFPCA_T_CASE(10) DFPCA_T_CASE(11) DFPCA_T_CASE(12)
    DFPCA_T_CASE(13) DFPCA_T_CASE(14) DFPCA_T_CASE(15) DFPCA_T_CASE(16) DFPCA_T_CASE(17) DFPCA_T_CASE(18)
    DFPCA_T_CASE(19) DFPCA_T_CASE(20) DFPCA_T_CASE(21) DFPCA_T_CASE(22) DFPCA_T_CASE(23) DFPCA_T_CASE(24)
#undef DFPCA_T_CASE
    default:
      break;
  }
}

}  // namespace

bool run_tphase2(dfpca_context* ctx, const TPhase2Spec& s) {
  const int R = std::max(s.R[0], s.R[1]);
  if (R < 1 || R > kMaxTemplR) return false;
  if (sizeof(double) * 3 * s.n1 * (s.n2 + 1) > 200 * 1024) return false;
  Taps2P tp{};
  for (int ax = 0; ax < 2; ++ax)
    for (int r = 0; r < 3; ++r)
      for (int o = -s.R[ax]; o <= s.R[ax]; ++o) tp.t[ax][r][o + R] = s.taps[ax][r][o + s.R[ax]];
  launch_tphase2_r(ctx, s, tp, R);
  return true;
}

void run_pass(dfpca_context* ctx, const PassSpec& s, double* taps_dev) {
  const int R = s.R;
  const bool tiled_ok = R <= kMaxTemplR && s.in.n <= kMaxN && s.in.n >= 1 &&
                        (s.in.inner == 1 || s.in.inner >= 16) &&
                        s.in.outer * ((s.in.inner + kTile - 1) / kTile) < (1ll << 31) &&
                        s.in.inner < (1ll << 31);
  if (tiled_ok) {
    TapsP tp{};
    for (int r = 0; r < s.n_out; ++r)
      for (int o = 0; o <= 2 * R; ++o) tp.t[r][o] = s.taps[r][o];
    launch_by_radius(ctx, s, tp);
    return;
  }
  const int W = 2 * R + 1;
  std::vector<double> host(static_cast<std::size_t>(3 * W), 0.0);
  for (int r = 0; r < s.n_out; ++r)
    std::copy(s.taps[r], s.taps[r] + W, host.begin() + r * W);
  DFPCA_CUDA(cudaMemcpyAsync(taps_dev, host.data(), sizeof(double) * host.size(),
                             cudaMemcpyHostToDevice, ctx->stream));
  const View o1 = s.n_out > 1 ? s.out[1] : s.out[0];
  const View o2 = s.n_out > 2 ? s.out[2] : s.out[0];
  const i64 total = s.in.outer * s.in.n * s.in.inner;
  DFPCA_LAUNCH(ctx, k_pass_generic, grid_for(total, 256, 148ll * 64), 256, 0, s.in, s.out[0], o1,
               o2, s.n_out, taps_dev, R);
}

}  // namespace dfpca_gpu
