// K3 dispatch: picks the register-tiled kernels of conv_impl.cuh (one
// instantiation per stencil radius, compiled in conv_r*.cu) or the generic
// any-radius pass.  See conv_impl.cuh for the algorithm and the reference
// citations (conv.hpp:161-201, 280-331).
#include <cstdlib>
#include <algorithm>
#include <cstdint>
#include <vector>

#include "conv_detail.cuh"

namespace dfpca_gpu {
namespace {

using conv_detail::Taps2P;
using conv_detail::TapsP;

// Generic pass: any radius, any axis length; one thread per output element.
__global__ void k_pass_generic(View in, View o0, View o1, View o2, int n_out,
                               const double* __restrict__ taps, int R) {
  pdl_wait();
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

// Radius bucket of the register-tiled kernels: exact up to 24, then 32 / 48.
int tiled_radius(int R) { return R <= 24 ? R : (R <= 32 ? 32 : 48); }

void launch_by_radius(dfpca_context* ctx, const PassSpec& s, const TapsP& tp) {
  switch (tiled_radius(s.R)) {
#define DFPCA_R_CASE(r)                                \
  case r:                                              \
    conv_detail::launch_pass<r>(ctx, s, tp);           \
    break;
    DFPCA_R_CASE(0) DFPCA_R_CASE(1) DFPCA_R_CASE(2) DFPCA_R_CASE(3) DFPCA_R_CASE(4)
    DFPCA_R_CASE(5) DFPCA_R_CASE(6) DFPCA_R_CASE(7) DFPCA_R_CASE(8) DFPCA_R_CASE(9)
    DFPCA_R_CASE(10) DFPCA_R_CASE(11) DFPCA_R_CASE(12) DFPCA_R_CASE(13) DFPCA_R_CASE(14)
    DFPCA_R_CASE(15) DFPCA_R_CASE(16) DFPCA_R_CASE(17) DFPCA_R_CASE(18) DFPCA_R_CASE(19)
    DFPCA_R_CASE(20) DFPCA_R_CASE(21) DFPCA_R_CASE(22) DFPCA_R_CASE(23) DFPCA_R_CASE(24)
    DFPCA_R_CASE(32) DFPCA_R_CASE(48)
#undef DFPCA_R_CASE
    default:
      break;
  }
}

void launch_tphase2_r(dfpca_context* ctx, const TPhase2Spec& s, const Taps2P& tp, int R) {
  switch (R) {
#define DFPCA_T_CASE(r)                                \
  case r:                                              \
    conv_detail::launch_tphase2<r>(ctx, s, tp);        \
    break;
    DFPCA_T_CASE(1) DFPCA_T_CASE(2) DFPCA_T_CASE(3) DFPCA_T_CASE(4) DFPCA_T_CASE(5) DFPCA_T_CASE(6)
    DFPCA_T_CASE(7) DFPCA_T_CASE(8) DFPCA_T_CASE(9) DFPCA_T_CASE(10) DFPCA_T_CASE(11) DFPCA_T_CASE(12)
    DFPCA_T_CASE(13) DFPCA_T_CASE(14) DFPCA_T_CASE(15) DFPCA_T_CASE(16) DFPCA_T_CASE(17) DFPCA_T_CASE(18)
    DFPCA_T_CASE(19) DFPCA_T_CASE(20) DFPCA_T_CASE(21) DFPCA_T_CASE(22) DFPCA_T_CASE(23) DFPCA_T_CASE(24)
    DFPCA_T_CASE(32) DFPCA_T_CASE(48)
#undef DFPCA_T_CASE
    default:
      break;
  }
}

}  // namespace

bool run_tphase2_mma(dfpca_context* ctx, const TPhase2Spec& s);

// Crossover radius of the t-phase: from this radius on the banded Toeplitz
// products on the DMMA pipe (conv_mma.cu) beat the direct FMA kernels
// (measured, profiles/r06_tphase_crossover.txt: direct 0.281 vs 0.289 ms at
// R = 16, 0.372 vs 0.312 ms at R = 20, 0.738 vs 0.383 ms at R = 39).
// DFPCA_TPHASE_MMA_R overrides it (0 = always the DMMA variant, a large value
// = never).
int tphase_mma_from() {
  static const int r = [] {
    const char* e = std::getenv("DFPCA_TPHASE_MMA_R");
    return e && *e ? std::atoi(e) : 18;
  }();
  return r;
}

bool run_tphase2(dfpca_context* ctx, const TPhase2Spec& s) {
  const int Rmax = std::max(s.R[0], s.R[1]);
  if (Rmax >= tphase_mma_from() && run_tphase2_mma(ctx, s)) return true;
  if (Rmax < 1 || Rmax > kMaxTemplR) return false;
  const int R = tiled_radius(Rmax);
  if (sizeof(double) * 3 * s.n1 * (s.n2 + 1) > 200 * 1024) return false;
  Taps2P tp{};
  for (int ax = 0; ax < 2; ++ax)
    for (int r = 0; r < 3; ++r)
      for (int o = -s.R[ax]; o <= s.R[ax]; ++o) tp.t[ax][r][o + R] = s.taps[ax][r][o + s.R[ax]];
  launch_tphase2_r(ctx, s, tp, R);
  return true;
}

bool run_pass_mma(dfpca_context* ctx, const PassSpec& s);

// Crossover radius of the column passes (the s-phase): banded Toeplitz
// products on the DMMA pipe (conv_mma.cu) from this radius on
// (profiles/r06_pass_crossover.txt: direct 0.523 vs 0.542 ms at R = 32,
// 0.729 vs 0.561 ms at R = 39); DFPCA_PASS_MMA_R overrides it.
int pass_mma_from() {
  static const int r = [] {
    const char* e = std::getenv("DFPCA_PASS_MMA_R");
    return e && *e ? std::atoi(e) : 36;
  }();
  return r;
}

void run_pass(dfpca_context* ctx, const PassSpec& s, double* taps_dev) {
  const int R = s.R;
  if (R >= pass_mma_from() && s.in.inner > 1 && run_pass_mma(ctx, s)) return;
  const bool tiled_ok = R <= kMaxTemplR && s.in.n <= conv_detail::kMaxN && s.in.n >= 1 &&
                        (s.in.inner == 1 || s.in.inner >= 16) &&
                        s.in.outer * ((s.in.inner + conv_detail::kTC - 1) / conv_detail::kTC) < (1ll << 31) &&
                        s.in.inner < (1ll << 31);
  if (tiled_ok) {
    // taps centred in the kernel's radius (zero padding for the 32 / 48 buckets)
    const int RT = tiled_radius(R);
    TapsP tp{};
    for (int r = 0; r < s.n_out; ++r)
      for (int o = -R; o <= R; ++o) tp.t[r][o + RT] = s.taps[r][o + R];
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
