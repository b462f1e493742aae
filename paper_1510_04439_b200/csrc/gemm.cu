// FP64 GEMM on the DMMA tensor pipe (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).
//
// tcgen05 has no f64 kind, so FP64 tensor math on sm_100a is the warp-level
// DMMA path; measured on this pool's B200 it peaks at ~37 TFLOP/s (the DFMA
// rate as well, tools/fp64_peak.cu), and it moves 4x fewer operand bytes per
// FMA through registers than DFMA, which is what lets a tile reach that peak.
//
// CTA tile 64 x 64, 4 warps each owning a 32 x 32 block (4 x 4 DMMA tiles),
// 4 CTAs per SM so 4 warps per scheduler hide the fragment-load latency; the
// small tile keeps the last wave short (G = 4096: 2080 upper tiles, 94% of the
// final wave busy vs 89% with 128 x 128) and gives a thin slab of a sharded
// pair grid enough tiles to fill the SMs.  K is staged 16 at
// a time through a 3-deep cp.async (LDGSTS) ring in shared memory, rows padded
// by 4 doubles so one warp's k-strided fragment loads spread over all banks.
// Per-row weights (the pair weights of the SYRK) are applied by a separate
// scaling pass so the operand copies stay asynchronous.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "gemm.cuh"

namespace dfpca_gpu {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int LDS = BM + 4;
#ifndef DFPCA_GEMM_WM
#define DFPCA_GEMM_WM 32
#endif
constexpr int WM = DFPCA_GEMM_WM, WN = 32;
constexpr int MT = WM / 8, NT = WN / 8;
constexpr int WARPS_N = BN / WN;
constexpr int NTHREADS = 32 * (BM / WM) * WARPS_N;
constexpr int CTAS_PER_SM = 4;
constexpr int STAGES = 3;
constexpr int STAGE_DOUBLES = 2 * BK * LDS;  // A and B tiles

__device__ inline void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ inline void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ inline void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ inline void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ inline void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// VEC: doubles per cp.async (2 when every row start is 16-byte aligned).
template <int VEC>
__global__ void __launch_bounds__(NTHREADS, CTAS_PER_SM)
    k_gemm_tn(i64 M, i64 N, i64 K, const double* __restrict__ A, i64 lda, const double* __restrict__ B,
              i64 ldb, double* __restrict__ C, i64 ldc, int symmetric, i64 tiles_n, i64 k_chunk,
              i64 split_stride, i64 tm_begin, i64 tm_end, const int4* __restrict__ items,
              double* __restrict__ ws, i64 k_mid, i64 a_col0) {
  pdl_wait();
  extern __shared__ __align__(16) double smem[];

  // symmetric: one work item per CTA (items, sym_items()): a tile pair
  // (tm <= tn) of row tiles [tm_begin, tm_end) (a slab of a sharded pair grid,
  // shard.hpp; C's row 0 is global row tm_begin * BM and mirrored tiles are
  // written only inside the slab), either whole or one K half of a split tile
  // whose two partial sums go to ws and are added by k_sym_split_reduce
  i64 tm, tn;
  int kpart = -1, slot = 0;
  if (symmetric) {
    const int4 it = items[blockIdx.x];
    tm = it.x;
    tn = it.y;
    kpart = it.z;
    slot = it.w;
  } else {
    tm = blockIdx.x / tiles_n;
    tn = blockIdx.x % tiles_n;
  }
  const i64 m0 = tm * BM, n0 = tn * BN;
  i64 k_begin = blockIdx.y * k_chunk;
  i64 k_end = (k_begin + k_chunk < K) ? k_begin + k_chunk : K;
  if (kpart == 0) k_end = k_mid;
  if (kpart == 1) k_begin = k_mid;
  C += blockIdx.y * split_stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / WARPS_N) * WM, wn0 = (warp % WARPS_N) * WN;

  // Stage loader: BK rows x BM doubles of A and of B, VEC doubles per copy;
  // out-of-range elements are zero-filled by the copy's src-size operand.
  auto load_stage = [&](int slot, i64 k0) {
    double* As = smem + slot * STAGE_DOUBLES;
    double* Bs = As + BK * LDS;
    constexpr int per_row = BM / VEC;
    for (int e = tid; e < BK * per_row; e += NTHREADS) {
      const int kr = e / per_row, c = (e % per_row) * VEC;
      const i64 k = k0 + kr;
      const bool krow = k < k_end;
      {
        const i64 col = m0 + c;
        const i64 avail = krow ? (M - col) : 0;
        const int bytes = avail >= VEC ? 8 * VEC : (avail > 0 ? 8 * static_cast<int>(avail) : 0);
        const double* src = bytes ? A + k * lda + (col - a_col0) : A;  // A holds columns from a_col0
        if (VEC == 2) cp_async16(As + kr * LDS + c, src, bytes);
        else cp_async8(As + kr * LDS + c, src, bytes);
      }
      {
        const i64 col = n0 + c;
        const i64 avail = krow ? (N - col) : 0;
        const int bytes = avail >= VEC ? 8 * VEC : (avail > 0 ? 8 * static_cast<int>(avail) : 0);
        const double* src = bytes ? B + k * ldb + col : B;
        if (VEC == 2) cp_async16(Bs + kr * LDS + c, src, bytes);
        else cp_async8(Bs + kr * LDS + c, src, bytes);
      }
    }
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const i64 nk = (k_end - k_begin + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, k_begin + s * BK);
    cp_async_commit();
  }
  for (i64 kb = 0; kb < nk; ++kb) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    // prefetch stage kb + STAGES - 1 into the slot freed at kb - 1
    const i64 pf = kb + STAGES - 1;
    if (pf < nk) load_stage(static_cast<int>(pf % STAGES), k_begin + pf * BK);
    cp_async_commit();
    const double* as = smem + (kb % STAGES) * STAGE_DOUBLES;
    const double* bs = as + BK * LDS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int kr = kk + (lane & 3);
      double af[MT], bf[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) af[i] = as[kr * LDS + wm0 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = bs[kr * LDS + wn0 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  if (kpart >= 0) {  // half of a split tile: the whole 64 x 64 partial to ws
    double* wt = ws + (static_cast<i64>(slot) * 2 + kpart) * (BM * BN);
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int r = wm0 + i * 8 + (lane >> 2), c = wn0 + j * 8 + 2 * (lane & 3);
        *reinterpret_cast<double2*>(wt + r * BN + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    return;
  }
  // Epilogue: fragment (i, j) holds C[row][col], C[row][col + 1].
  const i64 crow0 = symmetric ? tm_begin * BM : 0;
  const bool mirror = symmetric && tm != tn && tn < tm_end;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const i64 row = m0 + wm0 + i * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const i64 col = n0 + wn0 + j * 8 + 2 * (lane & 3);
      if (row < M) {
        double* crow = C + (row - crow0) * ldc;
        if (col + 1 < N && (ldc % 2) == 0) {
          *reinterpret_cast<double2*>(crow + col) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else {
          if (col < N) crow[col] = acc[i][j][0];
          if (col + 1 < N) crow[col + 1] = acc[i][j][1];
        }
      }
      if (mirror && row < M) {
        if (col < N) C[(col - crow0) * ldc + row] = acc[i][j][0];
        if (col + 1 < N) C[(col + 1 - crow0) * ldc + row] = acc[i][j][1];
      }
    }
  }
}

// Split tiles of the symmetric product: C = first K half + second K half (in
// that order), written like a whole tile (direct, and mirrored inside the slab).
__global__ void k_sym_split_reduce(const int4* __restrict__ split_items, const double* __restrict__ ws, i64 M,
                                   i64 N, double* __restrict__ C, i64 ldc, i64 tm_begin, i64 tm_end) {
  pdl_wait();
  const int4 it = split_items[blockIdx.x];
  const i64 tm = it.x, tn = it.y;
  const double* w0 = ws + static_cast<i64>(it.w) * 2 * (BM * BN);
  const double* w1 = w0 + BM * BN;
  const i64 crow0 = tm_begin * BM;
  const bool mirror = tm != tn && tn < tm_end;
  for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
    const i64 row = tm * BM + e / BN, col = tn * BN + e % BN;
    if (row >= M || col >= N) continue;
    const double v = w0[e] + w1[e];
    C[(row - crow0) * ldc + col] = v;
    if (mirror) C[(col - crow0) * ldc + row] = v;
  }
}

// Deterministic split-K reduction: slabs summed in ascending split order.
__global__ void k_splitk_reduce(const double* __restrict__ ws, i64 splits, i64 M, i64 N,
                                double* __restrict__ C, i64 ldc) {
  pdl_wait();
  const i64 total = M * N;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / N, c = e % N;
    double s = 0.0;
    for (i64 q = 0; q < splits; ++q) s += ws[q * total + e];
    C[r * ldc + c] = s;
  }
}

// out[k][m] = w[k] * in[k][col0 + m], m < M  (rounded product, as the
// reference's pw * m); a slab scales only the columns of its own row tiles.
__global__ void k_scale_rows(const double* __restrict__ in, const double* __restrict__ w, i64 K, i64 M,
                             i64 ld, i64 col0, double* __restrict__ out) {
  pdl_wait();
  const i64 total = K * M;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 k = e / M, m = e % M;
    out[k * M + m] = __dmul_rn(w[k], in[k * ld + col0 + m]);
  }
}

template <int VEC>
void launch(dfpca_context* ctx, dim3 grid, std::size_t smem, i64 M, i64 N, i64 K, const double* A, i64 lda,
            const double* B, i64 ldb, double* C, i64 ldc, int symmetric, i64 tiles_n, i64 k_chunk,
            i64 split_stride, i64 tm_begin, i64 tm_end, const int4* items, double* ws, i64 k_mid, i64 a_col0) {
  allow_smem(k_gemm_tn<VEC>, smem);
  DFPCA_LAUNCH(ctx, k_gemm_tn<VEC>, grid, NTHREADS, smem, M, N, K, A, lda, B, ldb, C, ldc, symmetric,
               tiles_n, k_chunk, split_stride, tm_begin, tm_end, items, ws, k_mid, a_col0);
}

}  // namespace

// Skinny products: as many K splits as keep the launch inside one wave of
// CTAS_PER_SM CTAs per SM (a second, partial wave would double the time).
i64 gemm_splits(const dfpca_context* ctx, i64 M, i64 N, i64 K) {
  const i64 blocks = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const i64 slots = static_cast<i64>(CTAS_PER_SM) * ctx->sm_count;
  i64 splits = 1;
  if (blocks < slots / 2 && K >= 1024) {
    splits = std::min<i64>(slots / blocks, K / 256);
    splits = std::max<i64>(splits, 1);
  }
  return splits;
}

void gemm_tn(dfpca_context* ctx, i64 M, i64 N, i64 K, const double* A, i64 lda, const double* w,
             const double* B, i64 ldb, double* C, i64 ldc, bool symmetric, i64 tm_begin, i64 tm_end,
             i64 force_splits) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    for (i64 r = 0; r < M; ++r)
      DFPCA_CUDA(cudaMemsetAsync(C + r * ldc, 0, sizeof(double) * N, ctx->stream));
    return;
  }
  const i64 tiles_m = (M + BM - 1) / BM;
  if (symmetric && M == N && A == B && lda == ldb && ozaki_enabled() &&
      ozaki_syrk(ctx, M, K, A, lda, w, C, ldc, std::max<i64>(0, tm_begin) * BM,
                 (tm_end < 0 || tm_end > tiles_m ? tiles_m : tm_end) * BM))
    return;
  DevBuf<double> scaled;
  i64 a_col0 = 0;
  if (w) {
    // weighted operand: the columns the launch reads (a slab's own row tiles)
    i64 c0 = 0, c1 = M;
    if (symmetric) {
      const i64 te = (tm_end < 0 || tm_end > tiles_m) ? tiles_m : tm_end;
      c0 = std::max<i64>(0, tm_begin) * BM;
      c1 = std::min<i64>(M, te * BM);
    }
    const i64 Mw = std::max<i64>(1, c1 - c0);
    scaled.alloc(static_cast<std::size_t>(K * Mw));
    DFPCA_LAUNCH(ctx, k_scale_rows, grid_for(K * Mw, 256), 256, 0, A, w, K, Mw, lda, c0, scaled.get());
    A = scaled.get();
    lda = Mw;
    a_col0 = c0;
  }
  const i64 tiles_n = (N + BN - 1) / BN;
  const std::size_t smem = sizeof(double) * STAGES * STAGE_DOUBLES;  // 52 KB
  const bool vec2 = (lda % 2 == 0) && (ldb % 2 == 0) && (reinterpret_cast<std::uintptr_t>(A) % 16 == 0) &&
                    (reinterpret_cast<std::uintptr_t>(B) % 16 == 0);
  if (tm_end < 0 || tm_end > tiles_m) tm_end = tiles_m;
  if (tm_begin < 0) tm_begin = 0;
  if (symmetric && tm_begin >= tm_end) return;
  // upper tile pairs of row tiles [tm_begin, tm_end)
  const i64 blocks = symmetric ? (tm_end - tm_begin) * tiles_m - (tm_end * (tm_end - 1) - tm_begin * (tm_begin - 1)) / 2
                               : tiles_m * tiles_n;
  // Skinny products (the projection GEMMs) get a deterministic split-K so the
  // grid covers the SMs.
  i64 splits = symmetric ? 1 : gemm_splits(ctx, M, N, K);
  if (!symmetric && force_splits > 0) splits = force_splits;  // row-sharded products: same sums as unsharded
  i64 k_chunk = K;
  double* out = C;
  i64 ldo = ldc, stride = 0;
  if (splits > 1) {
    k_chunk = (K + splits - 1) / splits;
    k_chunk = (k_chunk + BK - 1) / BK * BK;
    splits = (K + k_chunk - 1) / k_chunk;
    out = reinterpret_cast<double*>(ctx->scratch_bytes(sizeof(double) * splits * M * N));
    ldo = N;
    stride = M * N;
  }
  // symmetric: the work list (whole tiles first, then the halves of the split
  // tiles, so the halves fill the last wave)
  std::vector<int4> items, split_items;
  i64 k_mid = 0;
  DevBuf<int4> d_items, d_split;
  DevBuf<double> ws;
  i64 n_blocks = blocks;
  if (symmetric) {
    // Split rule, a function of the whole grid and the device only (never of
    // the slab), so a tile's sums are the same for any rank count: the
    // far-off-diagonal tiles tn - tm >= k0, just enough of them to cover the
    // partial last wave of the one-device launch.
    const i64 T = tiles_m, total = T * (T + 1) / 2, W = static_cast<i64>(CTAS_PER_SM) * ctx->sm_count;
    const i64 rem = total % W;
    i64 k0 = T;  // no split
    if (rem > 0 && K >= 4 * BK)
      for (i64 cand = T - 1; cand >= 1; --cand)
        if ((T - cand) * (T - cand + 1) / 2 >= rem) {
          k0 = cand;
          break;
        }
    k_mid = ((K / 2 + BK - 1) / BK) * BK;
    for (i64 tm = tm_begin; tm < tm_end; ++tm)
      for (i64 tn = tm; tn < tiles_m; ++tn) {
        if (tn - tm >= k0) split_items.push_back(make_int4(static_cast<int>(tm), static_cast<int>(tn), 0,
                                                           static_cast<int>(split_items.size())));
        else items.push_back(make_int4(static_cast<int>(tm), static_cast<int>(tn), -1, 0));
      }
    for (const int4& it : split_items) items.push_back(make_int4(it.x, it.y, 0, it.w));
    for (const int4& it : split_items) items.push_back(make_int4(it.x, it.y, 1, it.w));
    n_blocks = static_cast<i64>(items.size());
    d_items.alloc(items.size());
    DFPCA_CUDA(cudaMemcpyAsync(d_items.get(), items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice,
                               ctx->stream));
    if (!split_items.empty()) {
      ws.alloc(static_cast<std::size_t>(split_items.size() * 2 * BM * BN));
      d_split.alloc(split_items.size());
      DFPCA_CUDA(cudaMemcpyAsync(d_split.get(), split_items.data(), sizeof(int4) * split_items.size(),
                                 cudaMemcpyHostToDevice, ctx->stream));
    }
  }
  const dim3 grid(static_cast<unsigned>(n_blocks), static_cast<unsigned>(splits));
  if (vec2)
    launch<2>(ctx, grid, smem, M, N, K, A, lda, B, ldb, out, ldo, symmetric ? 1 : 0, tiles_n, k_chunk, stride,
              tm_begin, tm_end, d_items.get(), ws.get(), k_mid, a_col0);
  else
    launch<1>(ctx, grid, smem, M, N, K, A, lda, B, ldb, out, ldo, symmetric ? 1 : 0, tiles_n, k_chunk, stride,
              tm_begin, tm_end, d_items.get(), ws.get(), k_mid, a_col0);
  if (!split_items.empty())
    DFPCA_LAUNCH(ctx, k_sym_split_reduce, static_cast<unsigned>(split_items.size()), 256, 0, d_split.get(), ws.get(),
                 M, N, C, ldc, tm_begin, tm_end);
  if (splits > 1)
    DFPCA_LAUNCH(ctx, k_splitk_reduce, grid_for(M * N, 256), 256, 0, out, splits, M, N, C, ldc);
}

}  // namespace dfpca_gpu
