// FP64 GEMM on the DMMA tensor pipe (mma.sync.m8n8k4.f64 -> SASS DMMA.8).
//
// tcgen05 has no f64 kind, so FP64 tensor math on sm_100a is the warp-level
// DMMA path; measured on this pool's B200 it peaks at ~37 TFLOP/s, the same
// as DFMA, but it moves 4x fewer operand bytes per FMA through registers and
// shared memory, which is what lets a tile reach that peak.
//
// CTA tile 128 x 128, K staged 16 at a time through double-buffered shared
// memory; 8 warps, each owning a 64 x 32 block = 8 x 4 DMMA tiles of 8 x 8.
// Operand rows are padded to 132 doubles so the k-strided fragment loads of
// one warp spread over all 32 banks.
#include <algorithm>

#include "gemm.cuh"

namespace dfpca_gpu {
namespace {

constexpr int BM = 128, BN = 128, BK = 16;
constexpr int LDS = 132;
constexpr int WM = 64, WN = 32;
constexpr int MT = WM / 8, NT = WN / 8;

__device__ inline void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256, 1)
    k_gemm_tn(i64 M, i64 N, i64 K, const double* __restrict__ A, i64 lda,
              const double* __restrict__ w, const double* __restrict__ B, i64 ldb,
              double* __restrict__ C, i64 ldc, int symmetric, i64 tiles_n, i64 k_chunk,
              i64 split_stride) {
  extern __shared__ double smem[];
  double* As = smem;                  // [2][BK][LDS]
  double* Bs = smem + 2 * BK * LDS;   // [2][BK][LDS]

  i64 tm, tn;
  if (symmetric) {
    // enumerate upper-triangular tile pairs (tm <= tn)
    i64 t = blockIdx.x;
    tm = 0;
    while (t >= tiles_n - tm) {
      t -= tiles_n - tm;
      ++tm;
    }
    tn = tm + t;
  } else {
    tm = blockIdx.x / tiles_n;
    tn = blockIdx.x % tiles_n;
  }
  const i64 m0 = tm * BM, n0 = tn * BN;
  // split-K: blockIdx.y owns K range [k_begin, k_end) and its own C slab
  const i64 k_begin = blockIdx.y * k_chunk;
  const i64 k_end = (k_begin + k_chunk < K) ? k_begin + k_chunk : K;
  C += blockIdx.y * split_stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / 4) * WM, wn0 = (warp % 4) * WN;

  // Global -> register staging: each thread moves 8 doubles of A and of B per
  // stage (BK * BM / 256), as rows of 128 consecutive doubles.
  double ra[8], rb[8];
  auto load_stage = [&](i64 k0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + q * 256;
      const int kr = e / BM, c = e % BM;
      const i64 k = k0 + kr;
      double av = 0.0, bv = 0.0;
      if (k < k_end) {
        if (m0 + c < M) {
          av = A[k * lda + m0 + c];
          if (w) av = __dmul_rn(w[k], av);
        }
        if (n0 + c < N) bv = B[k * ldb + n0 + c];
      }
      ra[q] = av;
      rb[q] = bv;
    }
  };
  auto store_stage = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + q * 256;
      const int kr = e / BM, c = e % BM;
      As[(buf * BK + kr) * LDS + c] = ra[q];
      Bs[(buf * BK + kr) * LDS + c] = rb[q];
    }
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const i64 nk = (k_end - k_begin + BK - 1) / BK;
  load_stage(k_begin);
  store_stage(0);
  __syncthreads();
  for (i64 kb = 0; kb < nk; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nk) load_stage(k_begin + (kb + 1) * BK);
    const double* as = As + buf * BK * LDS;
    const double* bs = Bs + buf * BK * LDS;
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
    if (kb + 1 < nk) store_stage(buf ^ 1);
    __syncthreads();
  }

  // Epilogue: fragment (i, j) holds C[row][col], C[row][col + 1].
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const i64 row = m0 + wm0 + i * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const i64 col = n0 + wn0 + j * 8 + 2 * (lane & 3);
      if (row < M) {
        if (col + 1 < N && (ldc % 2) == 0) {
          *reinterpret_cast<double2*>(C + row * ldc + col) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else if (col + 1 < N) {
          C[row * ldc + col] = acc[i][j][0];
          C[row * ldc + col + 1] = acc[i][j][1];
        } else if (col < N) {
          C[row * ldc + col] = acc[i][j][0];
        }
      }
      if (symmetric && tm != tn && row < M) {
        if (col < N) C[col * ldc + row] = acc[i][j][0];
        if (col + 1 < N) C[(col + 1) * ldc + row] = acc[i][j][1];
      }
    }
  }
}

// Deterministic split-K reduction: slabs summed in ascending split order.
__global__ void k_splitk_reduce(const double* __restrict__ ws, i64 splits, i64 M, i64 N,
                                double* __restrict__ C, i64 ldc) {
  const i64 total = M * N;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / N, c = e % N;
    double s = 0.0;
    for (i64 q = 0; q < splits; ++q) s += ws[q * total + e];
    C[r * ldc + c] = s;
  }
}

}  // namespace

void gemm_tn(dfpca_context* ctx, i64 M, i64 N, i64 K, const double* A, i64 lda, const double* w,
             const double* B, i64 ldb, double* C, i64 ldc, bool symmetric) {
  if (M <= 0 || N <= 0) return;
  const i64 tiles_m = (M + BM - 1) / BM;
  const i64 tiles_n = (N + BN - 1) / BN;
  const std::size_t smem = sizeof(double) * 4 * BK * LDS;  // 67.6 KB
  static bool attr_set = false;
  if (!attr_set) {
    DFPCA_CUDA(cudaFuncSetAttribute(k_gemm_tn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    attr_set = true;
  }
  const i64 blocks = symmetric ? tiles_m * (tiles_m + 1) / 2 : tiles_m * tiles_n;
  if (K <= 0) {
    for (i64 r = 0; r < M; ++r)
      DFPCA_CUDA(cudaMemsetAsync(C + r * ldc, 0, sizeof(double) * N, ctx->stream));
    return;
  }
  // Skinny products (the projection GEMMs) get a deterministic split-K so the
  // grid covers the 148 SMs.
  i64 splits = 1;
  if (!symmetric && blocks < 2 * ctx->sm_count && K >= 1024) {
    splits = std::min<i64>((2 * ctx->sm_count + blocks - 1) / blocks, K / 256);
    splits = std::max<i64>(splits, 1);
  }
  if (splits == 1) {
    DFPCA_LAUNCH(ctx, k_gemm_tn, dim3(static_cast<unsigned>(blocks), 1), 256, smem, M, N, K, A, lda,
                 w, B, ldb, C, ldc, symmetric ? 1 : 0, tiles_n, K, (i64)0);
    return;
  }
  i64 k_chunk = (K + splits - 1) / splits;
  k_chunk = (k_chunk + BK - 1) / BK * BK;
  splits = (K + k_chunk - 1) / k_chunk;
  double* ws = reinterpret_cast<double*>(ctx->scratch_bytes(sizeof(double) * splits * M * N));
  DFPCA_LAUNCH(ctx, k_gemm_tn, dim3(static_cast<unsigned>(blocks), static_cast<unsigned>(splits)), 256,
               smem, M, N, K, A, lda, w, B, ldb, ws, N, 0, tiles_n, k_chunk, M * N);
  DFPCA_LAUNCH(ctx, k_splitk_reduce, grid_for(M * N, 256), 256, 0, ws, splits, M, N, C, ldc);
}

}  // namespace dfpca_gpu
