// Slab sharding of the covariance smoother across ranks (one GPU each):
// partition plan and exchange schedule (host code, no device state).
//
// The 2d-dim pair grids and the covariance are split along the leading s
// axis s1.  Rank r owns s1 planes [a_r, b_r) of the output
// covariance and works on the halo-extended planes [ha_r, hb_r) =
// [a_r - R, b_r + R) clipped to the grid, R = the s1 stencil radius.  Every
// stage between the pair grids and the covariance is pointwise in s except
// the s1 pass, so the only inputs a rank lacks are pair-grid rows and the
// lower-triangle entries it does not compute:
//
//   exchange 1 (pair grids):  a rank computes the SYRK tiles (tm <= tn) of its
//     own rows -- the same tiles, hence the same bits, as the one-GPU build --
//     and receives (a) the halo rows of its neighbours and (b) the mirror
//     entries (s, t), tile(t) < tile(s), whose tile another rank computed;
//   exchange 2 (covariance):  a rank smooths and centres its rows for t >= s
//     and receives the transposed blocks of the rows before it, so every
//     rank ends with complete, exactly symmetric rows of the covariance.
//
// Slab boundaries are multiples of the 64-row GEMM tile (plane granularity
// `unit`) and balance the upper-triangle work, which dominates every stage.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace dfpca_gpu {

using i64 = std::int64_t;

constexpr i64 kShardRowTile = 64;  // GEMM tile rows (gemm.cu BM)

struct ShardPlan {
  int world = 1;
  i64 n1 = 0;   // s1 planes
  i64 rn = 0;   // s nodes per s1 plane (G / n1)
  i64 G = 0;    // grid nodes
  i64 R = 0;    // s1 halo (planes)
  i64 unit = 1;  // partition granularity (planes)
  std::vector<i64> bounds;  // world + 1 plane boundaries

  i64 a(int r) const { return bounds[static_cast<std::size_t>(r)]; }
  i64 b(int r) const { return bounds[static_cast<std::size_t>(r) + 1]; }
  i64 ha(int r) const { return a(r) - R > 0 ? a(r) - R : 0; }
  i64 hb(int r) const { return b(r) + R < n1 ? b(r) + R : n1; }
  bool empty(int r) const { return a(r) >= b(r); }
  int owner_of_plane(i64 x) const {
    for (int r = 0; r < world; ++r)
      if (x >= a(r) && x < b(r)) return r;
    return -1;
  }
};

// Plane boundaries balancing sum_{x in slab} (n1 - x - 1/2), the share of
// the upper triangle s <= t held by the rows of plane x.
ShardPlan make_shard_plan(i64 n1, i64 rn, i64 R, int world);

// One rectangular block of an exchange, in global (s, t) node indices:
// dst receives entries (s, t), s in [r0, r1), t in [c0, c1); the value is
// src's local row s, column t (transpose = false) or row t, column s
// (transpose = true).  Blocks with src == dst are local copies.
struct ShardBlock {
  int src = 0, dst = 0;
  i64 r0 = 0, r1 = 0, c0 = 0, c1 = 0;
  bool transpose = false;
  i64 elems() const { return (r1 - r0) * (c1 - c0); }
};

// phase 0: the pair-grid window of every rank (rows [ha, hb) planes, columns
// [ha * rn, G)); phase 1: the lower-triangle blocks of the covariance rows.
std::vector<ShardBlock> shard_blocks(const ShardPlan& plan, int phase);

}  // namespace dfpca_gpu
