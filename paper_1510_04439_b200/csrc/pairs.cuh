// K2 entry point (pairs.cu): pair-product grids pw / pv, whole or one slab
// window of a sharded covariance (shard.hpp).
#pragma once

#include <functional>

#include "common.cuh"

namespace dfpca_gpu {

// Rows [row0, row0 + rows) x columns [col0, G) of the pair grids, stored with
// leading dimension G from row row0 on.  The SYRK computes the upper tile
// pairs of row tiles [tm_begin, tm_end) (tm_end < 0: all); the rest of the
// window must be supplied by `exchange` (called after the SYRK and before the
// band fix-up, with whether pw came from the SYRK as well).  Default: the
// whole G x G grid on one device.
struct PairWindow {
  i64 row0 = 0;
  i64 rows = -1;
  i64 col0 = 0;
  i64 tm_begin = 0;
  i64 tm_end = -1;
};

// Whether the pair grids of b take the sparse route (sum_i nnz_i^2 records,
// bit-identical to the reference) rather than the SYRK; the same answer on
// every rank.  The sparse route computes whole windows: no exchange.
bool pair_grids_sparse(dfpca_context* ctx, const dfpca_binned* b);

void build_pair_grids(dfpca_context* ctx, const dfpca_binned* b, double* pw, double* pv,
                      const PairWindow* win = nullptr,
                      const std::function<void(bool pw_from_syrk)>& exchange = {});

}  // namespace dfpca_gpu
