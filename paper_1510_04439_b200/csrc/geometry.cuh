// Device replays of the reference's per-observation grid geometry, shared by
// binning (binning.cu) and scores (scores.cu): locate_cell (surface.hpp:42-66),
// the hull test (grid.hpp:209-215) and the corner masses in axis order
// (binning.hpp:135-145, scores.hpp:227-236), all without FMA contraction.
#pragma once

#include "common.cuh"

namespace dfpca_gpu {

struct ObsGeom {
  // Per observation: the 2^d corner flats and masses (axis-0 bit = corner bit 0).
  i64 flat[8];
  double mass[8];
};

__device__ inline void locate_cell_dev(const double* axis, i64 n, double x, i64& cell,
                                       double& frac) {
  if (x <= axis[0]) {
    cell = 0;
    frac = 0.0;
    return;
  }
  if (x >= axis[n - 1]) {
    cell = n - 2;
    frac = 1.0;
    return;
  }
  i64 lo = 0, hi = n - 1;
  while (hi - lo > 1) {
    const i64 mid = (lo + hi) / 2;
    if (axis[mid] <= x)
      lo = mid;
    else
      hi = mid;
  }
  cell = lo;
  frac = __ddiv_rn(__dsub_rn(x, axis[lo]), __dsub_rn(axis[lo + 1], axis[lo]));
}

template <int D = 0>
__device__ inline bool hull_contains_dev(const DevGrid& g, const double* x) {
  const int d = D > 0 ? D : g.d;
#pragma unroll
  for (int k = 0; k < d; ++k) {
    const double lo = g.axes[k][0], hi = g.axes[k][g.shape[k] - 1];
    const double tol = __dmul_rn(1e-12, __dsub_rn(hi, lo));
    if (x[k] < __dsub_rn(lo, tol) || x[k] > __dadd_rn(hi, tol)) return false;
  }
  return true;
}

// D > 0: the dimension as a template constant (loops unrolled, ObsGeom in
// registers); D = 0: runtime g.d.
template <int D = 0>
__device__ inline void corner_geometry(const DevGrid& g, const double* x, ObsGeom& geo) {
  i64 cell[kMaxDim];
  double frac[kMaxDim];
  const int d = D > 0 ? D : g.d;
#pragma unroll
  for (int k = 0; k < d; ++k) locate_cell_dev(g.axes[k], g.shape[k], x[k], cell[k], frac[k]);
  const int corners = 1 << d;
#pragma unroll
  for (int c = 0; c < corners; ++c) {
    double m = 1.0;
    i64 flat = 0;
#pragma unroll
    for (int k = 0; k < d; ++k) {
      const bool up = (c >> k) & 1;
      m = __dmul_rn(m, up ? frac[k] : __dsub_rn(1.0, frac[k]));
      flat += (cell[k] + (up ? 1 : 0)) * g.strides[k];
    }
    geo.flat[c] = flat;
    geo.mass[c] = m;
  }
}


}  // namespace dfpca_gpu
