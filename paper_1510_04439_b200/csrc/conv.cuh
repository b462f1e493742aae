// K3: separable axis passes of the kernel-moment convolutions.
#pragma once

#include "common.cuh"

namespace dfpca_gpu {

// Largest stencil radius with a register-tiled specialisation; wider stencils
// use the generic pass.
constexpr int kMaxTemplR = 24;

// A strided view of a row-major array: element (o, j, i) lives at
// p[o * os + j * js + i] for o < outer, j < n, i < inner (inner contiguous).
struct View {
  double* p;
  i64 outer, os;
  i64 n, js;
  i64 inner;
};

// One multi-order pass along an axis: outputs out[r] = taps(order[r]) * in.
struct PassSpec {
  View in;
  int n_out;
  View out[3];
  const double* taps[3];  // host pointers to 2R+1 taps each
  int R;
};

void run_pass(dfpca_context* ctx, const PassSpec& spec, double* taps_dev_scratch);

}  // namespace dfpca_gpu
