// Multi-GPU extension of the drop-in (no reference counterpart: the
// reference's only parallel knob is set_max_threads, parallel.hpp:23).
// One process per GPU; every rank calls the same functions with the same
// (replicated) inputs.  The covariance is split into s1-plane slabs
// (paper_1510_04439_b200/csrc/shard.hpp): each rank returns
// complete, exactly symmetric rows [row0, row0 + rows) of the covariance the
// one-GPU fft_covariance (fft_smoother.hpp:585) computes -- bit for bit --
// and randomized_eig_sharded returns the one-GPU EigenSystem on every rank.
//
//   std::array<unsigned char, 128> id{};
//   if (rank == 0) dfpca::gpu::nccl_unique_id(id.data());
//   /* broadcast id with MPI / a file / torch.distributed */
//   dfpca::gpu::init_distributed(world, rank, id.data());
//   auto slab = dfpca::gpu::fft_covariance_sharded(binned, grid, h, mean);
//   auto eig  = dfpca::gpu::randomized_eig_sharded(slab, 99, 20, grid, seed);
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "dfpca/eigensolve.hpp"
#include "dfpca/fft_smoother.hpp"
#include "dfpca/gpu.hpp"

namespace dfpca {
namespace gpu {

/// 128 bytes identifying a new NCCL communicator (call on one rank).
inline void nccl_unique_id(void* id128) {
  if (dfpca_nccl_unique_id(id128) != 0) throw err::device_error("libnccl could not provide a unique id");
}

/// Joins this process's context (device DFPCA_DEVICE / set_device) to a
/// communicator of `world` ranks.
inline void init_distributed(int world, int rank, const void* id128) {
  check(dfpca_nccl_init(context(), world, rank, id128));
}

/// This rank's rows of the covariance.
struct CovarianceSlab {
  EvaluationGrid grid;
  Index row0 = 0;
  Index rows = 0;
  std::vector<double> values;  // rows x G, row-major (s * G + t with s - row0)
  std::shared_ptr<dfpca_surface> device;
};

inline CovarianceSlab fft_covariance_sharded(const BinnedData& binned, const EvaluationGrid& grid,
                                             const Bandwidth& h, const SurfaceEstimate& mean) {
  grid.require_equispaced("binned covariance smoothing");
  h.validate(grid);
  if (mean.values.size() != static_cast<std::size_t>(grid.size()))
    throw err::invalid_argument("mean surface does not conform to the grid");
  GridDesc gd(grid);
  dfpca_surface* s = nullptr;
  check(dfpca_covariance_sharded(context(), device_binned(binned), gd.get(), h.h.data(), mean.values.data(),
                                 nullptr, &s));
  CovarianceSlab out;
  out.grid = grid;
  out.device.reset(s, SurfaceDeleter{});
  int64_t r0 = 0, nr = 0;
  check(dfpca_surface_rows(s, &r0, &nr));
  out.row0 = r0;
  out.rows = nr;
  out.values.resize(static_cast<std::size_t>(nr * grid.size()));
  check(dfpca_surface_download(context(), s, out.values.data()));
  return out;
}

/// randomized_eig (eigensolve.hpp:245-279) over the ranks' slabs: the
/// products with the covariance run per rank and are all-gathered.
inline EigenSystem randomized_eig_sharded(const CovarianceSlab& slab, std::size_t q, std::size_t L_max,
                                          const EvaluationGrid& grid, std::uint64_t seed) {
  if (q < L_max)
    throw err::sketch_too_small("sketch size " + std::to_string(q) + " is below the requested component count " +
                                std::to_string(L_max));
  const auto G = static_cast<std::size_t>(grid.size());
  const std::size_t cap = std::max<std::size_t>(L_max, 1);
  std::vector<double> ev(cap), ef(cap * G), fve(cap);
  double total = 0.0;
  int64_t n = 0;
  GridDesc gd(grid);
  check(dfpca_randomized_eig(context(), slab.device.get(), gd.get(), static_cast<int64_t>(q),
                             static_cast<int64_t>(L_max), seed, ev.data(), ef.data(), fve.data(), &total, &n));
  EigenSystem out;
  out.total_variance = total;
  for (int64_t l = 0; l < n; ++l) {
    out.eigenvalues.push_back(ev[static_cast<std::size_t>(l)]);
    out.fve.push_back(fve[static_cast<std::size_t>(l)]);
    out.eigenfunctions.emplace_back(ef.begin() + l * static_cast<int64_t>(G),
                                    ef.begin() + (l + 1) * static_cast<int64_t>(G));
  }
  return out;
}

}  // namespace gpu
}  // namespace dfpca
