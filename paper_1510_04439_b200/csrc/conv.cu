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

#include "conv.cuh"

namespace dfpca_gpu {
namespace {

constexpr int kTile = 32;  // columns (or lines) per CTA
constexpr int kJB = 8;     // outputs per thread along the axis
constexpr int kMaxN = 128; // longest axis staged whole in shared memory

struct TapsP {
  double t[3][2 * kMaxTemplR + 1];
};

// Columns variant: the axis is not the contiguous one (inner >= 16).
template <int R, int NO>
__global__ void __launch_bounds__(256) k_pass_cols(View in, View o0, View o1, View o2, TapsP tp) {
  extern __shared__ double sm[];  // [n][kTile]
  const i64 n = in.n;
  const i64 chunks = (in.inner + kTile - 1) / kTile;
  const i64 ob = blockIdx.x / chunks;
  const i64 c0 = (blockIdx.x % chunks) * kTile;
  const double* src = in.p + ob * in.os + c0;
  for (int e = threadIdx.x; e < n * kTile; e += blockDim.x) {
    const int j = e / kTile, c = e % kTile;
    sm[e] = (c0 + c < in.inner) ? src[j * in.js + c] : 0.0;
  }
  __syncthreads();
  const int c = threadIdx.x % kTile;
  const bool col_ok = c0 + c < in.inner;
  for (int j0 = (threadIdx.x / kTile) * kJB; j0 < n; j0 += (blockDim.x / kTile) * kJB) {
    double acc[NO][kJB];
#pragma unroll
    for (int r = 0; r < NO; ++r)
#pragma unroll
      for (int jj = 0; jj < kJB; ++jj) acc[r][jj] = 0.0;
#pragma unroll
    for (int m = -R; m < kJB + R; ++m) {
      const int jm = j0 + m;
      const double x = (jm >= 0 && jm < n) ? sm[jm * kTile + c] : 0.0;
#pragma unroll
      for (int jj = 0; jj < kJB; ++jj) {
        const int o = m - jj;
        if (o >= -R && o <= R) {
#pragma unroll
          for (int r = 0; r < NO; ++r) acc[r][jj] = fma(tp.t[r][o + R], x, acc[r][jj]);
        }
      }
    }
    if (col_ok) {
#pragma unroll
      for (int jj = 0; jj < kJB; ++jj) {
        const i64 j = j0 + jj;
        if (j < n) {
          o0.p[ob * o0.os + j * o0.js + c0 + c] = acc[0][jj];
          if (NO > 1) o1.p[ob * o1.os + j * o1.js + c0 + c] = acc[NO > 1 ? 1 : 0][jj];
          if (NO > 2) o2.p[ob * o2.os + j * o2.js + c0 + c] = acc[NO > 2 ? 2 : 0][jj];
        }
      }
    }
  }
}

// Lines variant: the axis is the contiguous one (inner == 1); a CTA stages
// kTile consecutive lines, row-padded to avoid bank conflicts.
template <int R, int NO>
__global__ void __launch_bounds__(256) k_pass_rows(View in, View o0, View o1, View o2, TapsP tp) {
  extern __shared__ double sm[];  // [kTile][n + 1]
  const i64 n = in.n;
  const i64 ld = n + 1;
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
    __syncwarp();
    if (line_ok) {
#pragma unroll
      for (int jj = 0; jj < kJB; ++jj) {
        const i64 j = j0 + jj;
        if (j < n) {
          o0.p[(l0 + l) * o0.os + j * o0.js] = acc[0][jj];
          if (NO > 1) o1.p[(l0 + l) * o1.os + j * o1.js] = acc[NO > 1 ? 1 : 0][jj];
          if (NO > 2) o2.p[(l0 + l) * o2.os + j * o2.js] = acc[NO > 2 ? 2 : 0][jj];
        }
      }
    }
  }
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
    const std::size_t smem = sizeof(double) * kTile * (in.n + 1);
    DFPCA_LAUNCH(ctx, (k_pass_rows<R, NO>), static_cast<unsigned>(blocks), 256, smem, in,
                 s.out[0], o1, o2, tp);
  } else {
    const i64 blocks = in.outer * ((in.inner + kTile - 1) / kTile);
    const std::size_t smem = sizeof(double) * kTile * in.n;
    DFPCA_LAUNCH(ctx, (k_pass_cols<R, NO>), static_cast<unsigned>(blocks), 256, smem, in,
                 s.out[0], o1, o2, tp);
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

}  // namespace

void run_pass(dfpca_context* ctx, const PassSpec& s, double* taps_dev) {
  const int R = s.R;
  const bool tiled_ok = R <= kMaxTemplR && s.in.n <= kMaxN && s.in.n >= 1 &&
                        (s.in.inner == 1 || s.in.inner >= 16) &&
                        s.in.outer * ((s.in.inner + kTile - 1) / kTile) < (1ll << 31);
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
