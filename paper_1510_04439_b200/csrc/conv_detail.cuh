// K3 internals shared by conv.cu (dispatch) and the per-radius instantiation
// units conv_r*.cu (kernels).  The kernels are templated on the stencil radius
// R; each radius is instantiated in exactly one conv_r*.cu so the three units
// compile in parallel.
#pragma once

#include "conv.cuh"

namespace dfpca_gpu {
namespace conv_detail {

constexpr int kThreads = 256;
constexpr int kTC = 64;     // columns per tile of the columns kernel
constexpr int kLines = 32;  // lines per CTA of the lines kernel
constexpr int kJBr = 8;     // outputs per thread: lines kernel and fused t-phase
constexpr int kMaxN = 128;  // longest axis staged whole in shared memory

struct TapsP {
  double t[3][2 * kMaxTemplR + 1];
};

struct Taps2P {
  double t[2][3][2 * kMaxTemplR + 1];
};

struct TPhaseOut {
  double* m[6];
  double* v[3];
  // upper-triangle trim (t1_margin >= 0): pair-grid row s (global s_base + s)
  // produces t1 planes >= (s_base + s) / rn - t1_margin only
  long long s_base;
  long long rn;
  int t1_margin;
};

// Tiled pass along one axis with radius R (R <= kMaxTemplR, n <= kMaxN).
template <int R>
void launch_pass(dfpca_context* ctx, const PassSpec& s, const TapsP& tp);

// Fused two-axis t-phase with (common) radius R.
template <int R>
void launch_tphase2(dfpca_context* ctx, const TPhase2Spec& s, const Taps2P& tp);

}  // namespace conv_detail
}  // namespace dfpca_gpu
