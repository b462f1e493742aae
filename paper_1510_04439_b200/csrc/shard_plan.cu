// Host-side slab plan and exchange schedule (see shard.hpp).
#include <algorithm>
#include <cmath>
#include <numeric>

#include "shard.hpp"

namespace dfpca_gpu {

ShardPlan make_shard_plan(i64 n1, i64 rn, i64 R, int world) {
  ShardPlan p;
  p.world = world < 1 ? 1 : world;
  p.n1 = n1;
  p.rn = rn;
  p.G = n1 * rn;
  p.R = R;
  const i64 g = std::gcd(rn, kShardRowTile);
  p.unit = kShardRowTile / (g > 0 ? g : 1);
  const i64 units = (n1 + p.unit - 1) / p.unit;
  // cumulative upper-triangle weight at every unit boundary
  std::vector<double> cum(static_cast<std::size_t>(units) + 1, 0.0);
  for (i64 u = 0; u < units; ++u) {
    double w = 0.0;
    for (i64 x = u * p.unit; x < std::min(n1, (u + 1) * p.unit); ++x) w += static_cast<double>(n1 - x) - 0.5;
    cum[static_cast<std::size_t>(u) + 1] = cum[static_cast<std::size_t>(u)] + w;
  }
  // contiguous unit ranges per rank minimising the largest load (then the
  // sum of squared loads, so ties stay balanced): a small DP over unit
  // boundaries (units <= n1, a few hundred at most in practice).  A rank's
  // load is its upper-triangle weight plus a per-plane term for the planes
  // its moment passes cover, halo included (the t-phase of [a - R, b + R)):
  // beta = 0.14 n1 triangle units per plane (the d = 3 ranks' fit, ~0.7 ms
  // per halo-extended plane against 0.12 ms per unit at n1 = 32, rn = 1024,
  // then the best of 0.10-0.30 by projection: N = 2 0.79 -> 0.87, N = 4
  // 0.67 -> 0.72, N = 8 0.49 -> 0.51), faded out for small
  // planes (rn < 32 n1: d = 2 64^2, where fixed per-rank costs dominate and
  // the planes-only balance measured better).
  const int W = p.world;
  const std::size_t U = static_cast<std::size_t>(units);
  const double beta = 0.14 * static_cast<double>(n1) *
                      std::min(1.0, static_cast<double>(rn) / (32.0 * static_cast<double>(n1)));
  auto load = [&](std::size_t a, std::size_t b) {
    if (b <= a) return 0.0;
    const i64 pa = static_cast<i64>(a) * p.unit, pb = std::min(n1, static_cast<i64>(b) * p.unit);
    const i64 planes = std::min(n1, pb + R) - std::max<i64>(0, pa - R);
    return cum[b] - cum[a] + beta * static_cast<double>(planes);
  };
  // f[k][j]: best (max, sumsq) for units [0, j) split into k ranks
  const double inf = 1e300;
  std::vector<std::vector<std::pair<double, double>>> f(
      static_cast<std::size_t>(W) + 1, std::vector<std::pair<double, double>>(U + 1, {inf, inf}));
  std::vector<std::vector<std::size_t>> arg(static_cast<std::size_t>(W) + 1, std::vector<std::size_t>(U + 1, 0));
  f[0][0] = {0.0, 0.0};
  for (int k = 1; k <= W; ++k)
    for (std::size_t j = 0; j <= U; ++j)
      for (std::size_t i = j + 1; i-- > 0;) {  // rank k takes units [i, j) (possibly none; ties: later ranks idle)
        const auto& prev = f[static_cast<std::size_t>(k) - 1][i];
        if (prev.first >= inf) continue;
        const double l = load(i, j);
        const std::pair<double, double> cand{std::max(prev.first, l), prev.second + l * l};
        auto& cur = f[static_cast<std::size_t>(k)][j];
        if (cand.first < cur.first - 1e-9 || (cand.first <= cur.first + 1e-9 && cand.second < cur.second - 1e-9)) {
          cur = cand;
          arg[static_cast<std::size_t>(k)][j] = i;
        }
      }
  p.bounds.assign(static_cast<std::size_t>(W) + 1, 0);
  std::size_t j = U;
  for (int k = W; k >= 1; --k) {
    const std::size_t i = arg[static_cast<std::size_t>(k)][j];
    p.bounds[static_cast<std::size_t>(k)] = std::min(n1, static_cast<i64>(j) * p.unit);
    j = i;
  }
  p.bounds[0] = 0;
  p.bounds[static_cast<std::size_t>(p.world)] = n1;
  return p;
}

std::vector<ShardBlock> shard_blocks(const ShardPlan& plan, int phase) {
  std::vector<ShardBlock> out;
  const i64 rn = plan.rn;
  for (int q = 0; q < plan.world; ++q) {
    if (plan.empty(q)) continue;
    if (phase == 0) {
      const i64 ha = plan.ha(q), hb = plan.hb(q);
      for (int p = 0; p < plan.world; ++p) {
        if (plan.empty(p)) continue;
        const i64 s0 = std::max(plan.a(p), ha), s1 = std::min(plan.b(p), hb);
        if (s0 >= s1) continue;
        // direct: rows of p, columns from p's own slab start (tile(t) >= tile(s))
        ShardBlock d;
        d.src = p;
        d.dst = q;
        d.r0 = s0 * rn;
        d.r1 = s1 * rn;
        d.c0 = std::max(plan.a(p), ha) * rn;
        d.c1 = plan.G;
        d.transpose = false;
        if (d.elems() > 0) out.push_back(d);
        // mirror: columns before p's slab, from the owners of those rows
        for (int pp = 0; pp < p; ++pp) {
          if (plan.empty(pp)) continue;
          const i64 t0 = std::max(plan.a(pp), ha), t1 = std::min(plan.b(pp), plan.a(p));
          if (t0 >= t1) continue;
          ShardBlock m;
          m.src = pp;
          m.dst = q;
          m.r0 = s0 * rn;
          m.r1 = s1 * rn;
          m.c0 = t0 * rn;
          m.c1 = t1 * rn;
          m.transpose = true;
          out.push_back(m);
        }
      }
    } else {
      // covariance rows of q, columns of every earlier rank p: Gamma(t, s) of p
      for (int p = 0; p < q; ++p) {
        if (plan.empty(p)) continue;
        ShardBlock m;
        m.src = p;
        m.dst = q;
        m.r0 = plan.a(q) * rn;
        m.r1 = plan.b(q) * rn;
        m.c0 = plan.a(p) * rn;
        m.c1 = plan.b(p) * rn;
        m.transpose = true;
        out.push_back(m);
      }
    }
  }
  return out;
}

}  // namespace dfpca_gpu
