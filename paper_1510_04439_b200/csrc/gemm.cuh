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
// tm_begin / tm_end (symmetric only): compute the row tiles [tm_begin, tm_end)
// of the upper tile triangle; C's row 0 is then global row tm_begin * 128 and
// mirrored tiles are written only when they fall inside those rows (slab of a
// sharded pair grid, shard.hpp).
// force_splits (> 0, non-symmetric): the split-K count, so that a row block of
// a product is summed exactly like the unsharded product (gemm_splits).
void gemm_tn(dfpca_context* ctx, i64 M, i64 N, i64 K, const double* A, i64 lda, const double* w,
             const double* B, i64 ldb, double* C, i64 ldc, bool symmetric, i64 tm_begin = 0,
             i64 tm_end = -1, i64 force_splits = 0);

// The pair-grid SYRK by the Ozaki scheme on the int8 tensor cores (ozaki.cu):
// rows [row0, row1) of C = (w * A)^T A (A: K x G row-major; C's row 0 is
// global row row0): every t >= s of those rows, and the mirror entries whose
// row is in the range too (gemm_tn's slab contract; the whole matrix for
// [0, G)).  Bit-identical for any row range (exact integer slice products).
// False when not applicable (no weights, K > 16384).  ozaki_enabled():
// DFPCA_SYRK is not "dmma".
bool ozaki_enabled();
bool ozaki_syrk(dfpca_context* ctx, i64 G, i64 K, const double* A, i64 lda, const double* w, double* C, i64 ldc,
                i64 row0, i64 row1);

// Split-K count gemm_tn picks for a non-symmetric M x N x K product.
i64 gemm_splits(const dfpca_context* ctx, i64 M, i64 N, i64 K);

}  // namespace dfpca_gpu
