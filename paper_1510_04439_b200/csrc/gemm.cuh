// FP64 tensor-core (DMMA) GEMM used by the pair-grid build (K2) and the
// random-projection eigensolver (K6).
#pragma once

#include "common.cuh"

namespace dfpca_gpu {

// C[m][n] = sum_k (w ? w[k] * A[k][m] : A[k][m]) * B[k][n]
//   A: K x M row-major (lda >= M), B: K x N row-major (ldb >= N),
//   C: M x N row-major (ldc >= N).
// symmetric: A and B describe the same operand pair of a SYRK (M == N, and the
// result is symmetric); only tiles with tile_n >= tile_m are computed and the
// transposed tile is written as well.
// beta_one: accumulate into C instead of overwriting it.
void gemm_tn(dfpca_context* ctx, i64 M, i64 N, i64 K, const double* A, i64 lda, const double* w,
             const double* B, i64 ldb, double* C, i64 ldc, bool symmetric);

}  // namespace dfpca_gpu
