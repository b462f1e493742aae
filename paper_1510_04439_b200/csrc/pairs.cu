// K2: pair-product grids (reference PairGridSource, fft_smoother.hpp:291-443).
//
//   pw(s,t) = sum_i w_i M_i(s) M_i(t) - diag_mass band
//   pv(s,t) = sum_i w_i V_i(s) V_i(t) - diag_value band
//
// The sum over samples is a SYRK with K = n_pair: computed on the FP64 tensor
// pipe (gemm.cu) for the upper tile triangle and mirrored.  When every sample
// has the same mass grid (the GridNodes / shared-design case, detected at
// binning time) pw is the rank-one product W M(s) M(t) and costs one pass.
//
// Exactness where it matters.  Near the diagonal the reference's pw is
// "sample sum minus band", and for pairs that only share one observation the
// two sums are identical sequences, so the reference gets an exact 0 there
// (which later decides whether a kernel window is empty).  A reordered SYRK
// would leave +-1 ulp there.  k_band_fix therefore recomputes every pw entry
// with a nonzero band in the reference order -- samples ascending, separate
// multiply and add, (w_i M_i(s)) M_i(t) (fft_smoother.hpp:397-402) -- and
// subtracts the band once (:433-434), making those entries bit-identical.
#include <functional>
#include <vector>

#include "gemm.cuh"
#include "pairs.cuh"
#include "shard.hpp"

namespace dfpca_gpu {
namespace {

// pw over rows [row0, row0 + rows), columns [col0, G) of the window
// (pw points at row row0, leading dimension G).
__global__ void k_rank_one(double* __restrict__ pw, const double* __restrict__ m, double W, i64 G, i64 row0,
                           i64 rows, i64 col0) {
  const i64 w = G - col0;
  const i64 total = rows * w;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / w, t = col0 + e % w;
    pw[r * G + t] = __dmul_rn(__dmul_rn(W, m[row0 + r]), m[t]);
  }
}

// Band fix-up, one warp per band entry (u, code) with a nonzero band.
//  * pw: recomputed exactly in the reference order and minus the band, so the
//    near-diagonal cancellations that decide empty windows are bit-identical.
//    The lanes form the per-sample products (w_i M_i(s)) M_i(t) of 32
//    consecutive samples in parallel (one rounded multiply pair each, as in
//    the reference) and lane 0 adds them in ascending sample order.  With a
//    shared mass grid (identical_mass) M_i(s) = M(s) for every i.
//  * pv: only the band subtraction (pv never decides emptiness; the SYRK sum
//    differs from the reference's by reassociation only).
//  * pw == nullptr: the pv subtraction alone (shared-design covariance, whose
//    mass moments come in closed form, smooth.cu).
__global__ void k_band_fix(const double* __restrict__ diag_mass, const double* __restrict__ diag_value,
                           i64 G, int d, i64 codes, DevGrid g, const double* __restrict__ ps_mass,
                           int identical, const double* __restrict__ w, i64 n_pair, double w_seq,
                           double* __restrict__ pw, double* __restrict__ pv, i64 row0, i64 rows, i64 col0) {
  // window: band entries of rows u in [row0, row0 + rows) and columns t >= col0;
  // pw / pv point at row row0 (leading dimension G)
  const int lane = threadIdx.x & 31;
  const i64 warps = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  const i64 total = rows * codes;
  for (i64 e0 = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5; e0 < total; e0 += warps) {
    const i64 e = e0 + row0 * codes;
    const double dm = diag_mass[e], dv = diag_value[e];
    if (dm == 0.0 && dv == 0.0) continue;
    const i64 u = e / codes;
    i64 code = e % codes;
    int off[kMaxDim];
    for (int k = d - 1; k >= 0; --k) {
      off[k] = static_cast<int>(code % 3) - 1;
      code /= 3;
    }
    i64 rem = u, t = 0;
    bool inside = true;
    for (int k = d - 1; k >= 0; --k) {
      const i64 a = rem % g.shape[k];
      rem /= g.shape[k];
      const i64 bk = a + off[k];
      if (bk < 0 || bk >= g.shape[k]) inside = false;
      t += bk * g.strides[k];
    }
    if (!inside || t < col0) continue;
    const i64 at = (u - row0) * G + t;
    if (pw == nullptr) {  // value grid only (shared-design covariance)
      if (lane == 0) pv[at] = __dsub_rn(pv[at], dv);
      continue;
    }
    double sw = 0.0;
    const double ms0 = identical ? ps_mass[u] : 0.0, mt0 = identical ? ps_mass[t] : 0.0;
    // shared unit masses (every subject observed once at both nodes):
    // (w_i * 1) * 1 == w_i, so the ordered sum is the ordered sum of the
    // weights, W_seq, computed once on the host in the same order
    const bool unit = identical && ms0 == 1.0 && mt0 == 1.0;
    if (unit) sw = w_seq;
    for (i64 i0 = 0; i0 < (unit ? 0 : n_pair); i0 += 32) {
      const i64 i = i0 + lane;
      double pm = 0.0;
      if (i < n_pair) {
        const double ms = identical ? ms0 : ps_mass[i * G + u];
        const double mt = identical ? mt0 : ps_mass[i * G + t];
        pm = __dmul_rn(__dmul_rn(w[i], ms), mt);
      }
      const int cnt = n_pair - i0 < 32 ? static_cast<int>(n_pair - i0) : 32;
      for (int q = 0; q < cnt; ++q) sw = __dadd_rn(sw, __shfl_sync(0xffffffffu, pm, q));
    }
    if (lane == 0) {
      pw[at] = __dsub_rn(sw, dm);
      pv[at] = __dsub_rn(pv[at], dv);
    }
  }
}


}  // namespace

DevGrid upload_grid_axes(dfpca_context* ctx, const Grid& g, DevBuf<double>& storage);

void build_pair_grids(dfpca_context* ctx, const dfpca_binned* b, double* pw, double* pv, const PairWindow* win,
                      const std::function<void(bool pw_from_syrk)>& exchange) {
  const i64 G = b->grid.G;
  const i64 n = b->n_pair;
  PairWindow full;
  full.rows = G;
  const PairWindow& w = win ? *win : full;
  const i64 tiles = (G + kShardRowTile - 1) / kShardRowTile;
  const i64 tm_end = w.tm_end < 0 ? tiles : w.tm_end;
  // own SYRK rows inside the window buffer
  const i64 own = w.tm_begin * kShardRowTile - w.row0;
  double W = 0.0;
  for (double x : b->pair_weight_h) W += x;  // sequential, as the reference's sample loop
  DevBuf<double> axes;
  const DevGrid dg = upload_grid_axes(ctx, b->grid, axes);  // (synchronizes: before the SYRK is queued)
  if (pw) {
    if (b->identical_mass) {
      DFPCA_LAUNCH(ctx, k_rank_one, grid_for(w.rows * (G - w.col0), 256, 148ll * 16), 256, 0, pw,
                   b->ps_mass.get(), W, G, w.row0, w.rows, w.col0);
    } else {
      gemm_tn(ctx, G, G, n, b->ps_mass.get(), G, b->pair_weight.get(), b->ps_mass.get(), G, pw + own * G, G, true,
              w.tm_begin, tm_end);
    }
  }
  if (pv)
    gemm_tn(ctx, G, G, n, b->ps_value.get(), G, b->pair_weight.get(), b->ps_value.get(), G, pv + own * G, G, true,
            w.tm_begin, tm_end);
  if (exchange) exchange(pw != nullptr && !b->identical_mass);
  if (pv)
    DFPCA_LAUNCH(ctx, k_band_fix, grid_for(w.rows * b->codes * 32, 256, 148ll * 32), 256, 0,
                 b->diag_mass.get(), b->diag_value.get(), G, b->grid.d, b->codes, dg,
                 b->ps_mass.get(), b->identical_mass ? 1 : 0, b->pair_weight.get(), n, W, pw, pv, w.row0, w.rows,
                 w.col0);
}

}  // namespace dfpca_gpu
