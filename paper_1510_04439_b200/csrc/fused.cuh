// Fused last-axis convolution + per-node solve for the 2-d covariance.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace dfpca_gpu {

struct S1SolveSpec {
  const double* in[14];  // canonical order, see s1_p4_input_order()
  i64 n;                 // s1 extent
  i64 inner;             // s2 extent * cols
  i64 cols;              // t columns in this chunk
  i64 t0;                // first t column
  i64 G;                 // grid nodes (row length of the covariance)
  i64 s2n;               // s2 extent
  const double* taps[3]; // s1 taps, orders 0..2 (2R+1 host doubles each)
  int R;
  const std::uint8_t* mask;  // device mask or nullptr
  double* out;               // G x G covariance (pre-centering)
  unsigned long long* cnt;   // empty-window counter
  i64* list;                 // empty-window node list
  i64 cap;
};

// Returns false when the shape/radius has no specialisation.
bool run_s1_solve_p4(dfpca_context* ctx, const S1SolveSpec& s);

// {budget, a, b, c}: budget 2 = mass-like, 1 = value-like; (a, b, c) the
// orders on axes (s2, t1, t2).
std::vector<std::array<int, 4>> s1_p4_input_order();

}  // namespace dfpca_gpu
