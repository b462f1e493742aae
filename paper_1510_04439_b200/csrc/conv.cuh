// K3: separable axis passes of the kernel-moment convolutions.
#pragma once

#include "common.cuh"

namespace dfpca_gpu {

// Largest stencil radius with a register-tiled specialisation: every radius up
// to 24 has its own instantiation, 25..32 and 33..48 run the radius-32 / -48
// kernels with zero-padded taps (a zero tap adds +0, leaving every sum
// unchanged); wider stencils use the generic pass.
constexpr int kMaxTemplR = 48;

// A strided view of a row-major array: element (o, j, i) lives at
// p[o * os + j * js + i] for o < outer, j < n, i < inner (inner contiguous).
struct View {
  double* p;
  i64 outer, os;
  i64 n, js;
  i64 inner;
  // Upper-triangle restriction of the 2-d covariance s-phase (arrays laid out
  // [s1][s2][t], only s <= t is ever solved):
  //   tri = 1: pass along s2 (outer = s1): skip s1 rows beyond those the s1
  //            pass of the same t columns will read;
  //   tri = 2: pass along s1 (inner = s2 * tri_G + t): read s1 < s1_out + R,
  //            write s1 < s1_out, s1_out = t_max / tri_rn + 1;
  //   tri = 3: pass along s2 after the s1 pass (outer = s1): only the
  //            planes s1 < s1_out.
  int tri = 0;
  int tri_R = 0;
  i64 tri_G = 0;   // t extent
  i64 tri_rn = 0;  // s nodes per s1 row
  i64 tri_n1 = 0;  // s1 extent (local planes)
  // slab of a sharded covariance (shard.hpp): local plane 0 is global s1 plane
  // tri_row0, outputs stop at global plane tri_row_hi (< 0: no limit), and
  // local column 0 is global t = tri_t0
  i64 tri_row0 = 0;
  i64 tri_row_hi = -1;
  i64 tri_t0 = 0;
  // output window along the axis (columns kernel): rows [lo, hi) are written,
  // rows [0, min(n, hi + R)) are read; hi < 0: the whole axis
  i64 lo = 0;
  i64 hi = -1;
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

// Fused t-phase of the 2-d covariance (two trailing axes t1, t2): per pair-grid
// row, both axis passes run in shared memory and only the 9 t-partials reach
// HBM.  mass_out[i] receives t-orders (a1, a2) in the order
// (0,0) (1,0) (2,0) (0,1) (1,1) (0,2); value_out: (0,0) (1,0) (0,1).
// taps[axis][order] point at 2R+1 host doubles (axis 0 = t1, 1 = t2).
struct TPhase2Spec {
  const double* pw;
  const double* pv;
  i64 rows;      // pair-grid rows (s nodes) in this call
  i64 n1, n2;    // t-plane shape
  double* mass_out[6];
  double* value_out[3];
  const double* taps[2][3];
  int R[2];
  bool value_only = false;  // pw unused: only the 3 value t-partials
  // Upper-triangle trim: row s (global pair-grid row s_base + s, plane
  // (s_base + s) / rn) computes only t1 >= plane - t1_margin -- the
  // s-phase (View::tri) never reads the planes below.  t1_margin < 0: all.
  i64 s_base = 0, rn = 1;
  int t1_margin = -1;
};
// Returns false when the plane does not fit (caller uses run_pass instead).
bool run_tphase2(dfpca_context* ctx, const TPhase2Spec& spec);

}  // namespace dfpca_gpu
