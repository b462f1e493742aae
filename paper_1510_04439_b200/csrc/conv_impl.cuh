// K3 kernels: one separable convolution pass along one axis, producing up to
// three moment orders from a single read of the input (tree-factored moments),
// and the fused two-axis t-phase of the 2-d covariance.
//
// Replaces AxisConv::run_line / SeparableConv::convolve_axis
// (conv.hpp:161-201, 280-331).  out[j] = sum_{o=-R..R} taps[o+R] * in[j+o]
// with zero extension beyond the axis, accumulated in ascending o exactly as
// the reference's direct path (conv.hpp:165-173).  The reference switches to
// overlap-add FFT for >= 33 taps (conv.hpp:73); the device path stays direct
// (the FP64 pass is FMA-bound, not transform-bound, at these axis lengths),
// which is the exact-arithmetic twin of the FFT result.
//
// Included only by the conv_r*.cu instantiation units.
#pragma once

#include <algorithm>
#include <cstdint>

#include "conv_detail.cuh"

namespace dfpca_gpu {
namespace conv_detail {

// ------------------------------------------------------------ primitives --
__device__ inline unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ inline void cp_async_c8(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_addr(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ inline void cp_async_commit_c() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ inline void cp_async_wait_c() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ inline void mbar_init(std::uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ inline void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
// arrive (release) + expect `bytes` more transaction bytes for this phase
__device__ inline void mbar_arrive_tx(std::uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ inline void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}
__device__ inline void mbar_wait(std::uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// bulk (TMA-engine) copy of `bytes` (multiple of 16, 16-byte aligned ends)
__device__ inline void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// --------------------------------------------------------- columns kernel --
// The axis is not the contiguous one (inner >= 16).  Persistent CTAs walk the
// tiles (outer index, kTC-column chunk).  Each tile's full-axis column block
// [rows][kTC] is staged in shared memory, double-buffered: while tile i is
// convolved, tile i + grid is in flight.  BULK: warp 0 moves each staged row
// with one cp.async.bulk (TMA engine, completion on an mbarrier), so loading
// costs ~one instruction per 512-byte row; otherwise every thread issues
// 8-byte cp.async (unaligned views).  Thread (c, g) owns column c and output
// blocks j0 = g*JB, g*JB + 4*JB, ... (4 row groups of 64 threads, JB = 8); its JB
// consecutive outputs per order sit in registers, and the taps are kernel
// parameters (uniform-register operands of DFMA).
struct TileMeta {
  int ob, c0, rows, nout, lo;
};

template <int R, int NO, int JB, bool CHECK>
__device__ __forceinline__ void conv_block(const double* __restrict__ col, int j0, int rows, const TapsP& tp,
                                           double (&acc)[NO][JB]) {
#pragma unroll
  for (int r = 0; r < NO; ++r)
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) acc[r][jj] = 0.0;
#pragma unroll
  for (int m = -R; m < JB + R; ++m) {
    const int jm = j0 + m;
    const double x = CHECK ? ((jm >= 0 && jm < rows) ? col[jm * kTC] : 0.0) : col[jm * kTC];
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) {
      const int o = m - jj;
      if (o >= -R && o <= R) {
#pragma unroll
        for (int r = 0; r < NO; ++r) acc[r][jj] = fma(tp.t[r][o + R], x, acc[r][jj]);
      }
    }
  }
}

// BULK runs warp-specialized: kThreads compute threads plus one producer warp
// that issues the row copies of tile k + 2 as soon as the compute warps have
// released its buffer (an "empty" mbarrier per buffer, one arrival per compute
// warp), so no CTA-wide barrier separates the tiles.
constexpr int kProducerThreads = 32;

template <int R, int NO, int JB, bool BULK>
__global__ void __launch_bounds__(kThreads + kProducerThreads) k_pass_cols(View in, View o0, View o1, View o2,
                                                                           TapsP tp) {
  pdl_wait();
  extern __shared__ __align__(128) double sm[];  // [2][n][kTC]
  __shared__ __align__(8) std::uint64_t bar[2];
  __shared__ __align__(8) std::uint64_t empty_bar[2];
  __shared__ TileMeta meta[2];
  constexpr int kGroups = kThreads / kTC;
  const int n = static_cast<int>(in.n);
  const int inner = static_cast<int>(in.inner);
  const int chunks = (inner + kTC - 1) / kTC;
  const int n_tiles = static_cast<int>(in.outer) * chunks;
  const int tile_elems = n * kTC;
  const int tri = in.tri, triR = in.tri_R, triG = static_cast<int>(in.tri_G), tri_rn = static_cast<int>(in.tri_rn),
            tri_n1 = static_cast<int>(in.tri_n1);
  const int tri_t0 = static_cast<int>(in.tri_t0), tri_row0 = static_cast<int>(in.tri_row0),
            tri_row_hi = static_cast<int>(in.tri_row_hi);
  const int win_lo = static_cast<int>(in.lo), win_hi = static_cast<int>(in.hi);
  // rows to stage and outputs to produce (all unless the upper-triangle
  // restriction applies, see View::tri)
  auto make_meta = [&](int tile) {
    TileMeta mt;
    mt.ob = tile / chunks;
    mt.c0 = (tile - mt.ob * chunks) * kTC;
    mt.rows = n;
    mt.nout = n;
    mt.lo = win_lo;
    if (win_hi >= 0) {
      mt.nout = win_hi < n ? win_hi : n;
      mt.rows = mt.nout + R < n ? mt.nout + R : n;
    }
    if (tri != 0) {
      const int c1 = (mt.c0 + kTC < inner ? mt.c0 + kTC : inner) - 1;
      const int tmax = (mt.c0 / triG == c1 / triG) ? c1 % triG : triG - 1;
      int s1_out = (tmax + tri_t0) / tri_rn + 1;  // global planes
      if (tri_row_hi >= 0 && s1_out > tri_row_hi) s1_out = tri_row_hi;
      s1_out -= tri_row0;  // local
      if (s1_out < 0) s1_out = 0;
      if (tri == 1) {
        const int s1_in = s1_out + triR < tri_n1 ? s1_out + triR : tri_n1;
        if (mt.ob >= s1_in) mt.rows = mt.nout = 0;
      } else if (tri == 3) {  // in-plane pass after the s1 pass: output planes only
        if (mt.ob >= s1_out) mt.rows = mt.nout = 0;
      } else {
        mt.nout = s1_out < n ? s1_out : n;
        mt.rows = mt.nout + triR < n ? mt.nout + triR : n;
      }
    }
    return mt;
  };
  const int lane = threadIdx.x & 31;
  // stage `tile` into buffer b (warp 0 when BULK, every thread otherwise)
  auto issue = [&](int tile, int b) {
    const TileMeta mt = make_meta(tile);
    const double* src = in.p + mt.ob * in.os + mt.c0;
    double* dst = sm + b * tile_elems;
    const int cols = inner - mt.c0 < kTC ? inner - mt.c0 : kTC;
    if constexpr (BULK) {
      const unsigned row_bytes = 8u * static_cast<unsigned>(cols);
      if (lane == 0) {
        meta[b] = mt;
        mbar_arrive_tx(&bar[b], row_bytes * static_cast<unsigned>(mt.rows));
      }
      __syncwarp();
      for (int j = lane; j < mt.rows; j += 32) bulk_g2s(dst + j * kTC, src + j * in.js, row_bytes, &bar[b]);
    } else {
      if (threadIdx.x == 0) meta[b] = mt;
      for (int e = threadIdx.x; e < mt.rows * kTC; e += kThreads) {
        const int j = e / kTC, c = e % kTC;
        const bool ok = c < cols;
        cp_async_c8(dst + e, ok ? src + j * in.js + c : in.p, ok ? 8 : 0);
      }
    }
  };
  const int c = threadIdx.x % kTC;
  const int g = threadIdx.x / kTC;
  // convolve the staged tile in buffer b (compute threads)
  auto compute = [&](int b) {
    const TileMeta mt = meta[b];
    const double* col = sm + b * tile_elems + c;
    if (mt.c0 + c < inner) {
      const i64 cb = mt.c0 + c;
      double* b0 = o0.p + mt.ob * o0.os + cb;
      double* b1 = o1.p + mt.ob * o1.os + cb;
      double* b2 = o2.p + mt.ob * o2.os + cb;
      for (int j0 = mt.lo + g * JB; j0 < mt.nout; j0 += kGroups * JB) {
        double acc[NO][JB];
        if (j0 >= R && j0 + JB + R <= mt.rows)
          conv_block<R, NO, JB, false>(col, j0, mt.rows, tp, acc);
        else
          conv_block<R, NO, JB, true>(col, j0, mt.rows, tp, acc);
        double* p0 = b0 + j0 * o0.js;
        double* p1 = b1 + j0 * o1.js;
        double* p2 = b2 + j0 * o2.js;
        if (j0 + JB <= mt.nout) {
#pragma unroll
          for (int jj = 0; jj < JB; ++jj) {
            p0[jj * o0.js] = acc[0][jj];
            if (NO > 1) p1[jj * o1.js] = acc[NO > 1 ? 1 : 0][jj];
            if (NO > 2) p2[jj * o2.js] = acc[NO > 2 ? 2 : 0][jj];
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < JB; ++jj) {
            if (j0 + jj < mt.nout) {
              p0[jj * o0.js] = acc[0][jj];
              if (NO > 1) p1[jj * o1.js] = acc[NO > 1 ? 1 : 0][jj];
              if (NO > 2) p2[jj * o2.js] = acc[NO > 2 ? 2 : 0][jj];
            }
          }
        }
      }
    }
  };
  if constexpr (BULK) {
    constexpr unsigned kComputeWarps = kThreads / 32;
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      mbar_init(&empty_bar[0], kComputeWarps);
      mbar_init(&empty_bar[1], kComputeWarps);
      mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x >= kThreads) {  // producer warp
      int k = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
        const int b = k & 1;
        if (k >= 2) mbar_wait(&empty_bar[b], static_cast<unsigned>((k >> 1) - 1) & 1u);
        issue(tile, b);
      }
      return;
    }
    int k = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
      const int b = k & 1;
      mbar_wait(&bar[b], static_cast<unsigned>(k >> 1) & 1u);
      compute(b);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[b]);
    }
  } else {
    int buf = 0;
    int tile = blockIdx.x;
    if (tile < n_tiles) issue(tile, 0);
    cp_async_commit_c();
    for (; tile < n_tiles; tile += gridDim.x) {
      const int next = tile + gridDim.x;
      if (next < n_tiles) issue(next, buf ^ 1);
      cp_async_commit_c();
      cp_async_wait_c<1>();
      __syncthreads();
      compute(buf);
      __syncthreads();  // everyone is done with this buffer before it is refilled
      buf ^= 1;
    }
    cp_async_wait_c<0>();
  }
}

// ----------------------------------------------------------- lines kernel --
// The axis is the contiguous one (inner == 1); a CTA stages kLines
// consecutive lines, row-padded against bank conflicts, and writes back
// through a shared-memory output tile so the global stores stay coalesced.
template <int R, int NO>
__global__ void __launch_bounds__(kThreads) k_pass_rows(View in, View o0, View o1, View o2, TapsP tp) {
  pdl_wait();
  extern __shared__ double sm[];  // [kLines][n + 1] input, then NO output tiles of the same shape
  const i64 n = in.n;
  const i64 ld = n + 1;
  double* so = sm + kLines * ld;
  const i64 l0 = static_cast<i64>(blockIdx.x) * kLines;
  for (int e = threadIdx.x; e < n * kLines; e += blockDim.x) {
    const int l = e / n, j = e % n;
    sm[l * ld + j] = (l0 + l < in.outer) ? in.p[(l0 + l) * in.os + j * in.js] : 0.0;
  }
  __syncthreads();
  const int l = threadIdx.x % kLines;
  for (int j0 = (threadIdx.x / kLines) * kJBr; j0 < n; j0 += (blockDim.x / kLines) * kJBr) {
    double acc[NO][kJBr];
#pragma unroll
    for (int r = 0; r < NO; ++r)
#pragma unroll
      for (int jj = 0; jj < kJBr; ++jj) acc[r][jj] = 0.0;
#pragma unroll
    for (int m = -R; m < kJBr + R; ++m) {
      const int jm = j0 + m;
      const double x = (jm >= 0 && jm < n) ? sm[l * ld + jm] : 0.0;
#pragma unroll
      for (int jj = 0; jj < kJBr; ++jj) {
        const int o = m - jj;
        if (o >= -R && o <= R) {
#pragma unroll
          for (int r = 0; r < NO; ++r) acc[r][jj] = fma(tp.t[r][o + R], x, acc[r][jj]);
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < kJBr; ++jj) {
      const i64 j = j0 + jj;
      if (j < n) {
#pragma unroll
        for (int r = 0; r < NO; ++r) so[(r * kLines + l) * ld + j] = acc[r][jj];
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * kLines; e += blockDim.x) {
    const int ll = e / n, j = e % n;
    if (l0 + ll >= in.outer) continue;
    o0.p[(l0 + ll) * o0.os + j * o0.js] = so[(0 * kLines + ll) * ld + j];
    if (NO > 1) o1.p[(l0 + ll) * o1.os + j * o1.js] = so[(1 * kLines + ll) * ld + j];
    if (NO > 2) o2.p[(l0 + ll) * o2.os + j * o2.js] = so[(2 * kLines + ll) * ld + j];
  }
}

// ---------------------------------------------------- fused 2-axis t-phase --
// One CTA per pair-grid row s: the t-plane [n1][n2] is staged once (row pitch
// n2+1 against bank conflicts); for each t2-order the t2 pass writes a
// shared-memory plane, and the t1 pass over it writes the final t-partials
// straight to HBM, coalesced along t2.  Both axes use the same template
// radius R (the narrower axis is zero-padded).
template <int R, int ORD>
__device__ inline void tp_conv_rows(const double* X, double* Y, int n1, int n2, int ld, const Taps2P& tp, int l0) {
  // Y[l][j] = sum_o taps[t2][order][o] X[l][j+o]  (lines l = t1 >= l0, axis t2)
  const int nb = (n2 + kJBr - 1) / kJBr;
  const int nl = n1 - l0;
  for (int item = threadIdx.x; item < nl * nb; item += blockDim.x) {
    const int l = l0 + item % nl, j0 = (item / nl) * kJBr;
    double acc[kJBr];
#pragma unroll
    for (int jj = 0; jj < kJBr; ++jj) acc[jj] = 0.0;
#pragma unroll
    for (int m = -R; m < kJBr + R; ++m) {
      const int jm = j0 + m;
      const double x = (jm >= 0 && jm < n2) ? X[l * ld + jm] : 0.0;
#pragma unroll
      for (int jj = 0; jj < kJBr; ++jj) {
        const int o = m - jj;
        if (o >= -R && o <= R) acc[jj] = fma(tp.t[1][ORD][o + R], x, acc[jj]);
      }
    }
#pragma unroll
    for (int jj = 0; jj < kJBr; ++jj)
      if (j0 + jj < n2) Y[l * ld + j0 + jj] = acc[jj];
  }
}

template <int R, int NO>
__device__ inline void tp_conv_cols(const double* Y, int n1, int n2, int ld, double* const* outs, i64 row_off,
                                    const Taps2P& tp, int j_lo) {
  // out_r[j][c] = sum_o taps[t1][r][o] Y[j+o][c]   (axis t1 rows j >= j_lo, columns c = t2)
  const int nb = (n1 - j_lo + kJBr - 1) / kJBr;
  for (int item = threadIdx.x; item < n2 * nb; item += blockDim.x) {
    const int c = item % n2, j0 = j_lo + (item / n2) * kJBr;
    double acc[NO][kJBr];
#pragma unroll
    for (int r = 0; r < NO; ++r)
#pragma unroll
      for (int jj = 0; jj < kJBr; ++jj) acc[r][jj] = 0.0;
#pragma unroll
    for (int m = -R; m < kJBr + R; ++m) {
      const int jm = j0 + m;
      const double x = (jm >= 0 && jm < n1) ? Y[jm * ld + c] : 0.0;
#pragma unroll
      for (int jj = 0; jj < kJBr; ++jj) {
        const int o = m - jj;
        if (o >= -R && o <= R) {
#pragma unroll
          for (int r = 0; r < NO; ++r) acc[r][jj] = fma(tp.t[0][r][o + R], x, acc[r][jj]);
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < kJBr; ++jj) {
      const int j = j0 + jj;
      if (j < n1) {
#pragma unroll
        for (int r = 0; r < NO; ++r) outs[r][row_off + static_cast<i64>(j) * n2 + c] = acc[r][jj];
      }
    }
  }
}

template <int R>
__global__ void __launch_bounds__(kThreads) k_tphase2(const double* __restrict__ pw, const double* __restrict__ pv,
                                                      i64 rows, int n1, int n2, int value_only, TPhaseOut out,
                                                      Taps2P tp) {
  pdl_wait();
  extern __shared__ double sm[];
  const int ld = n2 + 1;
  const int pe = n1 * ld;  // padded plane
  double* Y = sm + 2 * pe;
  const i64 plane = static_cast<i64>(n1) * n2;
  // Planes of this CTA in order: (s, pw), (s, pv), (s + grid, pw), ... (only
  // the pv planes when value_only); the next plane is copied into the other X
  // buffer (cp.async, 8-byte granules because of the bank-conflict padding)
  // while the current one is convolved.  With the upper-triangle trim, row s
  // outputs t1 >= j_lo(s) and needs input lines t1 >= j_lo(s) - R.
  auto j_lo_of = [&](i64 s) -> int {
    if (out.t1_margin < 0) return 0;
    const long long lo = (out.s_base + s) / out.rn - out.t1_margin;
    return lo <= 0 ? 0 : (lo >= n1 ? n1 : static_cast<int>(lo));
  };
  auto issue = [&](i64 s, int pass, int buf) {
    const double* src = (pass ? pv : pw) + s * plane;
    double* X = sm + buf * pe;
    const int l0 = j_lo_of(s) - R > 0 ? j_lo_of(s) - R : 0;
    for (int e = l0 * n2 + threadIdx.x; e < plane; e += blockDim.x) cp_async_c8(X + (e / n2) * ld + e % n2, src + e, 8);
  };
  const int first_pass = value_only ? 1 : 0;
  i64 s = blockIdx.x;
  int pass = first_pass;
  int buf = 0;
  if (s < rows) issue(s, pass, 0);
  cp_async_commit_c();
  while (s < rows) {
    const bool same_row = pass == 0;
    const i64 ns = same_row ? s : s + gridDim.x;
    const int npass = same_row ? 1 : first_pass;
    if (ns < rows) issue(ns, npass, buf ^ 1);
    cp_async_commit_c();
    cp_async_wait_c<1>();
    __syncthreads();
    const double* X = sm + buf * pe;
    const i64 off = s * plane;
    const int max_order = pass == 0 ? 2 : 1;
    const int j_lo = j_lo_of(s);
    const int l0 = j_lo - R > 0 ? j_lo - R : 0;
    for (int r2 = 0; r2 <= max_order; ++r2) {
      if (r2 == 0) tp_conv_rows<R, 0>(X, Y, n1, n2, ld, tp, l0);
      else if (r2 == 1) tp_conv_rows<R, 1>(X, Y, n1, n2, ld, tp, l0);
      else tp_conv_rows<R, 2>(X, Y, n1, n2, ld, tp, l0);
      __syncthreads();
      if (pass == 0) {
        if (r2 == 0) {
          double* o[3] = {out.m[0], out.m[1], out.m[2]};
          tp_conv_cols<R, 3>(Y, n1, n2, ld, o, off, tp, j_lo);
        } else if (r2 == 1) {
          double* o[2] = {out.m[3], out.m[4]};
          tp_conv_cols<R, 2>(Y, n1, n2, ld, o, off, tp, j_lo);
        } else {
          double* o[1] = {out.m[5]};
          tp_conv_cols<R, 1>(Y, n1, n2, ld, o, off, tp, j_lo);
        }
      } else {
        if (r2 == 0) {
          double* o[2] = {out.v[0], out.v[1]};
          tp_conv_cols<R, 2>(Y, n1, n2, ld, o, off, tp, j_lo);
        } else {
          double* o[1] = {out.v[2]};
          tp_conv_cols<R, 1>(Y, n1, n2, ld, o, off, tp, j_lo);
        }
      }
      __syncthreads();
    }
    buf ^= 1;
    s = ns;
    pass = npass;
  }
  cp_async_wait_c<0>();
}

// The fused t-phase on zero-padded shared planes, so the inner loops carry
// no bounds tests: X lines hold R
// zeros on each side (pitch ldx, odd), Y holds R zero rows above and R + kJBv
// below (a t1 block may start at any row; pitch ldy, odd); the pads
// are zeroed once and never written.  One X buffer: the next plane's copy is
// issued after the last t2 pass of the current one has read X, so it
// overlaps the t1 pass.  Same products, same order as k_tphase2
// (bit-identical), which remains as DFPCA_TPHASE_2BUF=1 and for planes too
// large for the padded buffers.
#ifndef DFPCA_TPV_JB
#define DFPCA_TPV_JB 8
#endif
constexpr int kJBv = DFPCA_TPV_JB;  // outputs per thread of the padded t-phase
__host__ __device__ constexpr int tpv_ldx(int n2, int R) { return ((n2 + kJBv - 1) / kJBv * kJBv + 2 * R) | 1; }
__host__ __device__ constexpr int tpv_ldy(int n2) { return n2 | 1; }
__host__ __device__ constexpr int tpv_yrows(int n1, int R) { return n1 + kJBv + 2 * R; }  // t1 blocks start at any j_lo

template <int R, int ORD>
__device__ inline void tpv_conv_rows(const double* X, double* Y, int n1, int n2, int ldx, int ldy, const Taps2P& tp,
                                     int l0) {
  const int nb = (n2 + kJBv - 1) / kJBv;
  const int nl = n1 - l0;
  for (int item = threadIdx.x; item < nl * nb; item += blockDim.x) {
    const int l = l0 + item % nl, j0 = (item / nl) * kJBv;
    const double* xr = X + l * ldx + j0;  // xr[m + R] = X[l][j0 + m]
    double acc[kJBv];
#pragma unroll
    for (int jj = 0; jj < kJBv; ++jj) acc[jj] = 0.0;
#pragma unroll
    for (int m = -R; m < kJBv + R; ++m) {
      const double x = xr[m + R];
#pragma unroll
      for (int jj = 0; jj < kJBv; ++jj) {
        const int o = m - jj;
        if (o >= -R && o <= R) acc[jj] = fma(tp.t[1][ORD][o + R], x, acc[jj]);
      }
    }
    double* yr = Y + (l + R) * ldy + j0;
#pragma unroll
    for (int jj = 0; jj < kJBv; ++jj)
      if (j0 + jj < n2) yr[jj] = acc[jj];
  }
}

template <int R, int NO>
__device__ inline void tpv_conv_cols(const double* Y, int n1, int n2, int ldy, double* const* outs, i64 row_off,
                                     const Taps2P& tp, int j_lo) {
  const int nb = (n1 - j_lo + kJBv - 1) / kJBv;
  for (int item = threadIdx.x; item < n2 * nb; item += blockDim.x) {
    const int c = item % n2, j0 = j_lo + (item / n2) * kJBv;
    const double* yc = Y + j0 * ldy + c;  // yc[(m + R) ldy] = Y[j0 + m][c]
    double acc[NO][kJBv];
#pragma unroll
    for (int r = 0; r < NO; ++r)
#pragma unroll
      for (int jj = 0; jj < kJBv; ++jj) acc[r][jj] = 0.0;
#pragma unroll
    for (int m = -R; m < kJBv + R; ++m) {
      const double x = yc[(m + R) * ldy];
#pragma unroll
      for (int jj = 0; jj < kJBv; ++jj) {
        const int o = m - jj;
        if (o >= -R && o <= R) {
#pragma unroll
          for (int r = 0; r < NO; ++r) acc[r][jj] = fma(tp.t[0][r][o + R], x, acc[r][jj]);
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < kJBv; ++jj) {
      const int j = j0 + jj;
      if (j < n1) {
#pragma unroll
        for (int r = 0; r < NO; ++r) outs[r][row_off + static_cast<i64>(j) * n2 + c] = acc[r][jj];
      }
    }
  }
}

template <int R, bool VO>  // VO: value planes only (the shared design), no mass-order code
__global__ void __launch_bounds__(kThreads, 2) k_tphase2v(const double* __restrict__ pw, const double* __restrict__ pv,
                                                          i64 rows, int n1, int n2, TPhaseOut out, Taps2P tp) {
  pdl_wait();
  extern __shared__ double sm[];
  const int ldx = tpv_ldx(n2, R), ldy = tpv_ldy(n2);
  double* X = sm;
  double* Y = sm + n1 * ldx;
  const int ny = tpv_yrows(n1, R);
  for (int e = threadIdx.x; e < n1 * ldx + ny * ldy; e += blockDim.x) sm[e] = 0.0;  // the pads
  __syncthreads();
  const i64 plane = static_cast<i64>(n1) * n2;
  auto j_lo_of = [&](i64 s) -> int {
    if (out.t1_margin < 0) return 0;
    const long long lo = (out.s_base + s) / out.rn - out.t1_margin;
    return lo <= 0 ? 0 : (lo >= n1 ? n1 : static_cast<int>(lo));
  };
  auto issue = [&](i64 s, int pass) {
    const double* src = (pass ? pv : pw) + s * plane;
    const int l0 = j_lo_of(s) - R > 0 ? j_lo_of(s) - R : 0;
    for (int e = l0 * n2 + threadIdx.x; e < plane; e += blockDim.x)
      cp_async_c8(X + (e / n2) * ldx + R + e % n2, src + e, 8);
  };
  // planes in order: (s, pw), (s, pv), (s + grid, pw), ... (pv only when value_only)
  const int first_pass = VO ? 1 : 0;
  i64 s = blockIdx.x;
  int pass = first_pass;
  if (s < rows) issue(s, pass);
  cp_async_commit_c();
  while (s < rows) {
    const bool same_row = pass == 0;
    const i64 ns = same_row ? s : s + gridDim.x;
    const int npass = same_row ? 1 : first_pass;
    cp_async_wait_c<0>();
    __syncthreads();
    const i64 off = s * plane;
    const int j_lo = j_lo_of(s);
    const int l0 = j_lo - R > 0 ? j_lo - R : 0;
    const int max_order = !VO && pass == 0 ? 2 : 1;
    for (int r2 = 0; r2 <= max_order; ++r2) {
      if (r2 == 0) tpv_conv_rows<R, 0>(X, Y, n1, n2, ldx, ldy, tp, l0);
      else if (r2 == 1) tpv_conv_rows<R, 1>(X, Y, n1, n2, ldx, ldy, tp, l0);
      else tpv_conv_rows<R, 2>(X, Y, n1, n2, ldx, ldy, tp, l0);
      __syncthreads();
      if (r2 == max_order) {  // X is free: the next plane streams in under the t1 pass
        if (ns < rows) issue(ns, npass);
        cp_async_commit_c();
      }
      if (!VO && pass == 0) {
        if (r2 == 0) {
          double* o[3] = {out.m[0], out.m[1], out.m[2]};
          tpv_conv_cols<R, 3>(Y, n1, n2, ldy, o, off, tp, j_lo);
        } else if (r2 == 1) {
          double* o[2] = {out.m[3], out.m[4]};
          tpv_conv_cols<R, 2>(Y, n1, n2, ldy, o, off, tp, j_lo);
        } else {
          double* o[1] = {out.m[5]};
          tpv_conv_cols<R, 1>(Y, n1, n2, ldy, o, off, tp, j_lo);
        }
      } else if (r2 == 0) {
        double* o[2] = {out.v[0], out.v[1]};
        tpv_conv_cols<R, 2>(Y, n1, n2, ldy, o, off, tp, j_lo);
      } else {
        double* o[1] = {out.v[2]};
        tpv_conv_cols<R, 1>(Y, n1, n2, ldy, o, off, tp, j_lo);
      }
      __syncthreads();
    }
    s = ns;
    pass = npass;
  }
  cp_async_wait_c<0>();
}

// ------------------------------------------------------------- launchers --
template <typename K>
inline unsigned persistent_grid(dfpca_context* ctx, K kern, std::size_t smem, i64 work, int threads = kThreads) {
  allow_smem(kern, smem);  // dynamic + static shared memory may cross 48 KB even when smem alone does not
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  return static_cast<unsigned>(
      std::max<i64>(1, std::min<i64>(work, static_cast<i64>(std::max(per_sm, 1)) * ctx->sm_count)));
}

template <int R, int NO, int JB, bool BULK>
void launch_cols(dfpca_context* ctx, const PassSpec& s, const View& o1, const View& o2, const TapsP& tp) {
  const View& in = s.in;
  const i64 tiles = in.outer * ((in.inner + kTC - 1) / kTC);
  const std::size_t smem = sizeof(double) * 2 * kTC * in.n;
  const int threads = BULK ? kThreads + kProducerThreads : kThreads;
  const unsigned grid = persistent_grid(ctx, k_pass_cols<R, NO, JB, BULK>, smem, tiles, threads);
  DFPCA_LAUNCH_PDL(ctx, (k_pass_cols<R, NO, JB, BULK>), grid, threads, smem, in, s.out[0], o1, o2, tp);
}

template <int R, int NO>
void launch_tiled(dfpca_context* ctx, const PassSpec& s, const TapsP& tp) {
  const View& in = s.in;
  const View o1 = s.n_out > 1 ? s.out[1] : s.out[0];
  const View o2 = s.n_out > 2 ? s.out[2] : s.out[0];
  if (in.inner == 1) {
    const i64 blocks = (in.outer + kLines - 1) / kLines;
    const std::size_t smem = sizeof(double) * kLines * (in.n + 1) * (1 + NO);
    allow_smem(k_pass_rows<R, NO>, smem);
    DFPCA_LAUNCH(ctx, (k_pass_rows<R, NO>), static_cast<unsigned>(blocks), kThreads, smem, in, s.out[0], o1, o2,
                 tp);
    return;
  }
  // bulk row copies need 16-byte aligned, 16-byte multiple rows
  const bool bulk = (in.os % 2 == 0) && (in.js % 2 == 0) && (in.inner % 2 == 0) &&
                    (reinterpret_cast<std::uintptr_t>(in.p) % 16 == 0);
  // JB = 8: measured faster than 16 for every order count at n = 64 (the
  // 16-output blocks cost occupancy: 156 registers at NO = 3)
  if (bulk) launch_cols<R, NO, 8, true>(ctx, s, o1, o2, tp);
  else launch_cols<R, NO, 8, false>(ctx, s, o1, o2, tp);
}

template <int R>
void launch_pass(dfpca_context* ctx, const PassSpec& s, const TapsP& tp) {
  switch (s.n_out) {
    case 1: launch_tiled<R, 1>(ctx, s, tp); break;
    case 2: launch_tiled<R, 2>(ctx, s, tp); break;
    default: launch_tiled<R, 3>(ctx, s, tp); break;
  }
}

template <int R>
void launch_tphase2(dfpca_context* ctx, const TPhase2Spec& s, const Taps2P& tp) {
  TPhaseOut out;
  for (int i = 0; i < 6; ++i) out.m[i] = s.mass_out[i];
  for (int i = 0; i < 3; ++i) out.v[i] = s.value_out[i];
  out.s_base = s.s_base;
  out.rn = s.rn;
  out.t1_margin = s.t1_margin;
  const int n1 = static_cast<int>(s.n1), n2 = static_cast<int>(s.n2);
  const std::size_t smem1 = sizeof(double) * (static_cast<std::size_t>(n1) * tpv_ldx(n2, R) +
                                              static_cast<std::size_t>(tpv_yrows(n1, R)) * tpv_ldy(n2));
  if (smem1 <= 200 * 1024 && std::getenv("DFPCA_TPHASE_2BUF") == nullptr) {
    if (s.value_only) {
      const unsigned grid1 = persistent_grid(ctx, k_tphase2v<R, true>, smem1, s.rows);
      DFPCA_LAUNCH_PDL(ctx, (k_tphase2v<R, true>), grid1, kThreads, smem1, s.pw, s.pv, s.rows, n1, n2, out, tp);
    } else {
      const unsigned grid1 = persistent_grid(ctx, k_tphase2v<R, false>, smem1, s.rows);
      DFPCA_LAUNCH_PDL(ctx, (k_tphase2v<R, false>), grid1, kThreads, smem1, s.pw, s.pv, s.rows, n1, n2, out, tp);
    }
    return;
  }
  const std::size_t smem = sizeof(double) * 3 * n1 * (n2 + 1);
  const unsigned grid = persistent_grid(ctx, k_tphase2<R>, smem, s.rows);
  DFPCA_LAUNCH(ctx, k_tphase2<R>, grid, kThreads, smem, s.pw, s.pv, s.rows, n1, n2, s.value_only ? 1 : 0, out,
               tp);
}

}  // namespace conv_detail
}  // namespace dfpca_gpu

// Explicit instantiation of the launchers for one radius (conv_r*.cu).
#define DFPCA_CONV_INSTANTIATE(r)                                                                             \
  template void dfpca_gpu::conv_detail::launch_pass<r>(dfpca_context*, const dfpca_gpu::PassSpec&,            \
                                                       const dfpca_gpu::conv_detail::TapsP&);                 \
  template void dfpca_gpu::conv_detail::launch_tphase2<r>(dfpca_context*, const dfpca_gpu::TPhase2Spec&,      \
                                                          const dfpca_gpu::conv_detail::Taps2P&);
