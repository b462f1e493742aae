// Drop-in binned local-linear smoothers (reference fft_smoother.hpp: same
// declarations and default arguments) running on the GPU.
//
// Block plans and PairGridSource modes only trade memory for recomputation in
// the reference, whose outputs are bit-invariant to both (fft_smoother.hpp:
// 24-29, 494-497); the device computes the whole grid at once, so a plan is
// validated exactly as the reference does (same error names, same order) and
// otherwise has no effect.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "dfpca/binning.hpp"
#include "dfpca/dataset.hpp"
#include "dfpca/errors.hpp"
#include "dfpca/gpu.hpp"
#include "dfpca/grid.hpp"
#include "dfpca/surface.hpp"

namespace dfpca {

enum class MomentTarget { Mean, Squares };

struct BlockPlan {
  std::vector<Box> blocks;
  std::vector<Index> halo;

  Box core(std::size_t b, const std::vector<Index>& shape) const {
    Box c = blocks[b];
    for (std::size_t k = 0; k < c.dim(); ++k) {
      if (c.lo[k] > 0) c.lo[k] += halo[k];
      if (c.hi[k] < shape[k]) c.hi[k] -= halo[k];
    }
    return c;
  }
};

namespace detail {
inline Index kernel_radius_nodes(double h, double spacing) { return static_cast<Index>(std::ceil(h / spacing)); }

inline std::vector<Index> radii(const EvaluationGrid& grid, const Bandwidth& h) {
  std::vector<Index> r;
  for (std::size_t k = 0; k < grid.dim(); ++k) r.push_back(kernel_radius_nodes(h[k], grid.spacing(k)));
  return r;
}
}  // namespace detail

inline BlockPlan single_block_plan(const EvaluationGrid& grid, const Bandwidth& h) {
  return BlockPlan{{Box::full(grid.shape())}, detail::radii(grid, h)};
}

inline BlockPlan make_block_plan(const EvaluationGrid& grid, const Bandwidth& h, Index n_blocks) {
  if (n_blocks < 1) throw err::invalid_argument("block count must be positive");
  const auto& shape = grid.shape();
  n_blocks = std::min(n_blocks, shape[0]);
  BlockPlan plan{{}, detail::radii(grid, h)};
  for (Index b = 0; b < n_blocks; ++b) {
    Box blk = Box::full(shape);
    blk.lo[0] = std::max<Index>(0, shape[0] * b / n_blocks - plan.halo[0]);
    blk.hi[0] = std::min<Index>(shape[0], shape[0] * (b + 1) / n_blocks + plan.halo[0]);
    plan.blocks.push_back(blk);
  }
  return plan;
}

inline void validate_block_plan(const BlockPlan& plan, const EvaluationGrid& grid, const Bandwidth& h) {
  const std::size_t d = grid.dim();
  if (plan.blocks.empty() || plan.halo.size() != d)
    throw err::invalid_argument("block plan does not match the grid dimension");
  const auto r = detail::radii(grid, h);
  for (std::size_t k = 0; k < d; ++k)
    if (plan.halo[k] < r[k])
      throw err::halo_too_small("halo of " + std::to_string(plan.halo[k]) + " node(s) on axis " +
                                std::to_string(k) + " is below the kernel radius of " + std::to_string(r[k]));
  const auto& shape = grid.shape();
  Index covered = 0;
  std::vector<Box> cores;
  for (std::size_t b = 0; b < plan.blocks.size(); ++b) {
    const Box& blk = plan.blocks[b];
    if (blk.dim() != d) throw err::invalid_argument("block dimension mismatch");
    const Box c = plan.core(b, shape);
    for (std::size_t k = 0; k < d; ++k) {
      if (blk.lo[k] < 0 || blk.hi[k] > shape[k] || blk.lo[k] >= blk.hi[k])
        throw err::invalid_argument("block range outside the grid");
      if (c.extent(k) < plan.halo[k])
        throw err::block_too_small("block " + std::to_string(b) + " core extent " + std::to_string(c.extent(k)) +
                                   " on axis " + std::to_string(k) + " is smaller than its halo of " +
                                   std::to_string(plan.halo[k]));
    }
    covered += c.volume();
    cores.push_back(c);
  }
  for (std::size_t a = 0; a < cores.size(); ++a)
    for (std::size_t b = a + 1; b < cores.size(); ++b) {
      bool apart = false;
      for (std::size_t k = 0; k < d && !apart; ++k)
        apart = cores[a].hi[k] <= cores[b].lo[k] || cores[b].hi[k] <= cores[a].lo[k];
      if (!apart) throw err::invalid_argument("block cores overlap");
    }
  if (covered != grid.size()) throw err::invalid_argument("block cores do not tile the grid exactly");
}

/// Pair-product grids over the product domain (reference PairGridSource): the
/// full grids come from the device (dfpca_pair_grids); extract() slices any
/// box of them.
class PairGridSource {
 public:
  enum class Mode { Auto, Materialize, Rebuild };
  static constexpr std::size_t kMaterializeBudget = 640ull << 20;

  explicit PairGridSource(const BinnedData& binned, Mode mode = Mode::Auto) : binned_(binned) {
    if (!binned.has_covariance_path) throw err::invalid_argument("binned data lacks the covariance path");
    const auto g = static_cast<std::size_t>(binned.grid.size());
    materialized_ = mode == Mode::Materialize || (mode == Mode::Auto && 2 * g * g * sizeof(double) <= kMaterializeBudget);
  }
  bool materialized() const { return materialized_; }
  Box full_box() const {
    std::vector<Index> s2 = binned_.grid.shape();
    s2.insert(s2.end(), binned_.grid.shape().begin(), binned_.grid.shape().end());
    return Box::full(s2);
  }
  void extract(const Box& box, std::vector<double>& pw, std::vector<double>& pv) const {
    if (full_pw_.empty()) {
      const auto g = static_cast<std::size_t>(binned_.grid.size());
      full_pw_.resize(g * g);
      full_pv_.resize(g * g);
      gpu::check(dfpca_pair_grids(gpu::context(), gpu::device_binned(binned_), full_pw_.data(), full_pv_.data()));
    }
    const Box all = full_box();
    const auto st = detail::strides_of(all.hi);
    pw.clear();
    pv.clear();
    std::vector<Index> idx(box.lo);
    if (box.volume() == 0) return;
    do {
      const auto f = static_cast<std::size_t>(detail::flatten(idx, st));
      pw.push_back(full_pw_[f]);
      pv.push_back(full_pv_[f]);
    } while (detail::advance(idx, box));
  }

 private:
  const BinnedData& binned_;
  bool materialized_ = false;
  mutable std::vector<double> full_pw_, full_pv_;
};

namespace detail {

struct PlanDesc {
  std::vector<int64_t> lo, hi, halo;
  dfpca_plan p{};
  PlanDesc(const BlockPlan& plan, std::size_t d) {
    for (const auto& b : plan.blocks)
      for (std::size_t k = 0; k < d; ++k) {
        lo.push_back(k < b.lo.size() ? b.lo[k] : 0);
        hi.push_back(k < b.hi.size() ? b.hi[k] : 0);
      }
    halo.assign(plan.halo.begin(), plan.halo.end());
    p.n_blocks = plan.halo.size() == d ? static_cast<int64_t>(plan.blocks.size()) : 0;
    p.blocks_lo = lo.data();
    p.blocks_hi = hi.data();
    p.halo = halo.data();
  }
};

}  // namespace detail

inline SurfaceEstimate fft_local_linear(const BinnedData& binned, const EvaluationGrid& grid, const Bandwidth& h,
                                        MomentTarget target, const BlockPlan& plan) {
  // reference order of checks (fft_smoother.hpp:502-507); the device repeats them
  grid.require_equispaced("binned smoothing");
  h.validate(grid);
  if (!binned.has_mean_path) throw err::invalid_argument("binned data lacks the mean path");
  if (binned.grid.shape() != grid.shape()) throw err::invalid_argument("binned data does not conform to the grid");
  validate_block_plan(plan, grid, h);
  SurfaceEstimate out;
  out.grid = grid;
  out.kind = target == MomentTarget::Mean ? SurfaceKind::Mean : SurfaceKind::DiagPlusNoise;
  out.values.resize(static_cast<std::size_t>(grid.size()));
  gpu::GridDesc gd(grid);
  detail::PlanDesc pd(plan, grid.dim());
  dfpca_surface* s = nullptr;
  gpu::check(dfpca_local_linear(gpu::context(), gpu::device_binned(binned), gd.get(), h.h.data(),
                                target == MomentTarget::Mean ? DFPCA_TARGET_MEAN : DFPCA_TARGET_SQUARES, &pd.p,
                                out.values.data(), &s));
  out.device.reset(s, gpu::SurfaceDeleter{});
  return out;
}

inline SurfaceEstimate fft_local_linear(const BinnedData& binned, const EvaluationGrid& grid, const Bandwidth& h,
                                        MomentTarget target) {
  return fft_local_linear(binned, grid, h, target, single_block_plan(grid, h));
}

inline SurfaceEstimate fft_covariance(const BinnedData& binned, const EvaluationGrid& grid, const Bandwidth& h,
                                      const SurfaceEstimate& mean, const BlockPlan& plan,
                                      PairGridSource::Mode mode = PairGridSource::Mode::Auto) {
  (void)mode;  // memory/recompute trade-off of the reference only
  grid.require_equispaced("binned covariance smoothing");
  h.validate(grid);
  if (!binned.has_covariance_path) throw err::invalid_argument("binned data lacks the covariance path");
  if (binned.grid.shape() != grid.shape()) throw err::invalid_argument("binned data does not conform to the grid");
  if (binned.per_sample.empty())
    throw err::no_pairs("covariance smoothing needs at least one sample with two observations");
  if (mean.values.size() != static_cast<std::size_t>(grid.size()))
    throw err::invalid_argument("mean surface does not conform to the grid");
  validate_block_plan(plan, grid, h);
  gpu::GridDesc gd(grid);
  detail::PlanDesc pd(plan, grid.dim());
  dfpca_surface* s = nullptr;
  gpu::check(dfpca_covariance(gpu::context(), gpu::device_binned(binned), gd.get(), h.h.data(), mean.values.data(),
                              &pd.p, &s));
  SurfaceEstimate out;
  out.grid = grid;
  out.kind = SurfaceKind::Covariance;
  out.device.reset(s, gpu::SurfaceDeleter{});
  const auto g = static_cast<std::size_t>(grid.size());
  out.values.resize(g * g);
  gpu::check(dfpca_surface_download(gpu::context(), s, out.values.data()));
  return out;
}

inline SurfaceEstimate fft_covariance(const BinnedData& binned, const EvaluationGrid& grid, const Bandwidth& h,
                                      const SurfaceEstimate& mean,
                                      PairGridSource::Mode mode = PairGridSource::Mode::Auto) {
  return fft_covariance(binned, grid, h, mean, single_block_plan(grid, h), mode);
}

inline SurfaceEstimate blockwise_apply(const BlockPlan& plan, const BinnedData& binned, const EvaluationGrid& grid,
                                       const Bandwidth& h, MomentTarget target) {
  return fft_local_linear(binned, grid, h, target, plan);
}

inline SurfaceEstimate blockwise_apply(const BlockPlan& plan, const BinnedData& binned, const EvaluationGrid& grid,
                                       const Bandwidth& h, const SurfaceEstimate& mean) {
  return fft_covariance(binned, grid, h, mean, plan);
}

}  // namespace dfpca
