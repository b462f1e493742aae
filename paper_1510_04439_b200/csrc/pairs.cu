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
// would leave +-1 ulp there.  k_band_exact therefore recomputes every entry
// with a nonzero band in the reference order -- samples ascending, separate
// multiply and add, (w_i M_i(s)) M_i(t) (fft_smoother.hpp:397-402) -- and
// subtracts the band once (:433-434), making those entries bit-identical.
#include <vector>

#include "gemm.cuh"

namespace dfpca_gpu {
namespace {

__global__ void k_rank_one(double* __restrict__ pw, const double* __restrict__ m, double W, i64 G) {
  const i64 total = G * G;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 s = e / G, t = e % G;
    pw[e] = __dmul_rn(__dmul_rn(W, m[s]), m[t]);
  }
}

// One thread per band entry (u, code) whose band value is nonzero.
__global__ void k_band_exact(const double* __restrict__ diag_mass, const double* __restrict__ diag_value,
                             i64 G, int d, i64 codes, DevGrid g, const double* __restrict__ ps_mass,
                             const double* __restrict__ ps_value, const double* __restrict__ w,
                             i64 n_pair, double* __restrict__ pw, double* __restrict__ pv) {
  const i64 total = G * codes;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const double dm = diag_mass[e], dv = diag_value[e];
    if (dm == 0.0 && dv == 0.0) continue;
    const i64 u = e / codes;
    i64 code = e % codes;
    // decode offsets (last axis fastest) and the partner node
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
    if (!inside) continue;
    double sw = 0.0, sv = 0.0;
    for (i64 i = 0; i < n_pair; ++i) {
      const double ma = ps_mass[i * G + u], mb = ps_mass[i * G + t];
      const double va = ps_value[i * G + u], vb = ps_value[i * G + t];
      sw = __dadd_rn(sw, __dmul_rn(__dmul_rn(w[i], ma), mb));
      sv = __dadd_rn(sv, __dmul_rn(__dmul_rn(w[i], va), vb));
    }
    pw[u * G + t] = __dsub_rn(sw, dm);
    pv[u * G + t] = __dsub_rn(sv, dv);
  }
}

// Band subtraction for the rank-one / SYRK result at entries where the band
// is nonzero is done by k_band_exact; nothing else carries a band.

}  // namespace

DevGrid upload_grid_axes(dfpca_context* ctx, const Grid& g, DevBuf<double>& storage);

void build_pair_grids(dfpca_context* ctx, const dfpca_binned* b, double* pw, double* pv) {
  const i64 G = b->grid.G;
  const i64 n = b->n_pair;
  if (pw) {
    if (b->identical_mass) {
      double W = 0.0;
      for (double x : b->pair_weight_h) W += x;  // sequential, as the reference's sample loop
      DFPCA_LAUNCH(ctx, k_rank_one, grid_for(G * G, 256, 148ll * 16), 256, 0, pw, b->ps_mass.get(), W, G);
    } else {
      gemm_tn(ctx, G, G, n, b->ps_mass.get(), G, b->pair_weight.get(), b->ps_mass.get(), G, pw, G, true);
    }
  }
  if (pv) gemm_tn(ctx, G, G, n, b->ps_value.get(), G, b->pair_weight.get(), b->ps_value.get(), G, pv, G, true);
  if (pw && pv) {
    DevBuf<double> axes;
    DevGrid dg = upload_grid_axes(ctx, b->grid, axes);
    DFPCA_LAUNCH(ctx, k_band_exact, grid_for(G * b->codes, 128, 148ll * 32), 128, 0,
                 b->diag_mass.get(), b->diag_value.get(), G, b->grid.d, b->codes, dg,
                 b->ps_mass.get(), b->ps_value.get(), b->pair_weight.get(), n, pw, pv);
    DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
}

}  // namespace dfpca_gpu
