// Fused last-axis (s1) moment pass + per-node solve for the 2-d covariance.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace dfpca_gpu {

struct S1SolveSpec {
  const double* in[14];  // s2-level partials, canonical order (s1_p4_input_order)
  i64 n;                 // s1 extent (rows of the compact inputs)
  i64 inner;             // s2 extent * cols (row length of the compact inputs)
  i64 cols;              // t columns in this chunk
  i64 t0;                // first t column of the chunk
  i64 G;                 // grid nodes (covariance row length)
  i64 s2n;               // s2 extent
  const double* taps[3]; // s1 taps, orders 0..2 (2R+1 host doubles each)
  int R;
  const std::uint8_t* mask;  // device mask or nullptr
  double* out;               // G x G covariance (upper triangle written)
  unsigned long long* cnt;   // empty-window counter
  i64* list;                 // empty-window node list
  i64 cap;
};

// Returns false when there is no specialisation (the caller falls back to the
// separate s1 pass + solve).
bool run_s1_solve_p4(dfpca_context* ctx, const S1SolveSpec& s);

// {budget, a, b, c}: budget 2 = mass-like, 1 = value-like; (a, b, c) the
// orders on axes (s2, t1, t2), lexicographic.
std::vector<std::array<int, 4>> s1_p4_input_order();

}  // namespace dfpca_gpu
