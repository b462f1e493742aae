// Drop-in for the reference's dfpca/scores.hpp (noise variance, component
// scores, reconstruction) over libdfpca_cuda.so: the same declarations; the
// batch work runs on the GPU (dfpca_estimate_sigma2, dfpca_scores,
// dfpca_reconstruct).  estimate_sigma2, integration scores and
// reconstruct_on_grid are bit-identical to the reference; PACE scores agree to
// ~1e-15 (the reference's Eigen products are vectorized, version dependent).
// reconstruct_at stays a host evaluation (one multilinear interpolation per
// component), and holdout_prediction_error batches each held-out location's
// re-scoring into one GPU call.
//
// Host-side glue (argument validation, error names and message text, and
// the expressions whose bits the results depend on) follows the reference's
// code line for line where the drop-in contract requires identical behaviour.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "dfpca/dataset.hpp"
#include "dfpca/eigensolve.hpp"
#include "dfpca/errors.hpp"
#include "dfpca/gpu.hpp"
#include "dfpca/grid.hpp"
#include "dfpca/surface.hpp"

namespace dfpca {

enum class ScoreMethod { Pace, Integration };

inline std::string score_method_name(ScoreMethod m) { return m == ScoreMethod::Pace ? "pace" : "integration"; }

inline ScoreMethod parse_score_method(const std::string& s) {
  if (s == "pace") return ScoreMethod::Pace;
  if (s == "integration") return ScoreMethod::Integration;
  throw err::invalid_argument("unknown score method '" + s + "' (expected pace|integration)");
}

struct FpcaModel {
  SurfaceEstimate mean;
  EigenSystem eig;
  double sigma2 = 0.0;
  std::vector<std::vector<double>> scores;
  std::vector<std::string> sample_ids;

  Bandwidth mean_bandwidth;
  Bandwidth cov_bandwidth;
  Bandwidth diag_bandwidth;
  double fve_threshold = 0.0;
  std::uint64_t seed = 0;
  ScoreMethod score_method = ScoreMethod::Pace;

  std::size_t n_components() const { return eig.eigenvalues.size(); }
  const EvaluationGrid& grid() const { return mean.grid; }

  void validate() const {
    if (!(sigma2 >= 0.0) || !std::isfinite(sigma2))
      throw err::invalid_argument("model noise variance must be finite and nonnegative");
    if (mean.kind != SurfaceKind::Mean) throw err::invalid_argument("model mean surface has the wrong kind");
    const std::size_t L = n_components();
    for (const auto& row : scores) {
      if (row.size() != L) throw err::invalid_argument("score row length differs from component count");
      for (double a : row)
        if (!std::isfinite(a)) throw err::invalid_argument("scores must be finite");
    }
    if (!sample_ids.empty() && sample_ids.size() != scores.size())
      throw err::invalid_argument("sample id count differs from score row count");
  }
};

inline double estimate_sigma2(const SurfaceEstimate& diag_plus_noise, const SurfaceEstimate& cov,
                              const SurfaceEstimate& mean) {
  if (diag_plus_noise.kind != SurfaceKind::DiagPlusNoise || cov.kind != SurfaceKind::Covariance ||
      mean.kind != SurfaceKind::Mean)
    throw err::invalid_argument("estimate_sigma2 got surfaces of the wrong kind");
  const EvaluationGrid& grid = mean.grid;
  const Index g = grid.size();
  if (diag_plus_noise.grid.size() != g || cov.grid.size() != g)
    throw err::invalid_argument("estimate_sigma2 surfaces must share one grid");
  gpu::GridDesc gd(grid);
  double out = 0.0;
  gpu::check(dfpca_estimate_sigma2(gpu::context(), gd.get(), diag_plus_noise.values.data(),
                                   gpu::device_surface(cov), mean.values.data(), &out));
  return out;
}

namespace detail {
constexpr double kSigmaFloorRel = 1e-6;
}  // namespace detail

namespace gpu {

/// compute_scores for a batch of samples in one GPU call; sparse_warning (if
/// given) receives integration_scores' per-sample flag.
inline std::vector<std::vector<double>> compute_scores_batch(const std::vector<const Sample*>& samples,
                                                             const FpcaModel& model, ScoreMethod method,
                                                             std::vector<char>* sparse_warning = nullptr) {
  const EvaluationGrid& grid = model.grid();
  const std::size_t d = grid.dim(), L = model.n_components(), n = samples.size();
  const auto G = static_cast<std::size_t>(grid.size());
  std::vector<int64_t> off(n + 1, 0);
  std::vector<double> coords, values;
  for (std::size_t i = 0; i < n; ++i) {
    off[i + 1] = off[i] + static_cast<int64_t>(samples[i]->n_obs());
    coords.insert(coords.end(), samples[i]->coords.begin(), samples[i]->coords.begin() +
                                                              static_cast<std::ptrdiff_t>(samples[i]->n_obs() * d));
    values.insert(values.end(), samples[i]->values.begin(), samples[i]->values.end());
  }
  std::vector<double> funcs;
  funcs.reserve(L * G);
  for (const auto& f : model.eig.eigenfunctions) funcs.insert(funcs.end(), f.begin(), f.end());
  std::vector<double> out(std::max<std::size_t>(n * L, 1));
  std::vector<int32_t> warn(std::max<std::size_t>(n, 1), 0);
  GridDesc gd(grid);
  check(dfpca_scores(context(), gd.get(), static_cast<int64_t>(n), off.data(), coords.empty() ? nullptr : coords.data(),
                     values.empty() ? nullptr : values.data(), model.mean.values.data(), static_cast<int64_t>(L),
                     model.eig.eigenvalues.data(), funcs.empty() ? nullptr : funcs.data(), model.sigma2,
                     method == ScoreMethod::Pace ? 0 : 1, out.data(), warn.data()));
  std::vector<std::vector<double>> rows(n);
  for (std::size_t i = 0; i < n; ++i) rows[i].assign(out.begin() + static_cast<std::ptrdiff_t>(i * L),
                                                    out.begin() + static_cast<std::ptrdiff_t>((i + 1) * L));
  if (sparse_warning) {
    sparse_warning->resize(n);
    for (std::size_t i = 0; i < n; ++i) (*sparse_warning)[i] = warn[i] != 0;
  }
  return rows;
}

}  // namespace gpu

inline std::vector<double> pace_scores(const Sample& sample, const FpcaModel& model) {
  if (model.n_components() == 0) return {};
  return gpu::compute_scores_batch({&sample}, model, ScoreMethod::Pace)[0];
}

inline std::vector<double> integration_scores(const Sample& sample, const FpcaModel& model,
                                              bool* sparse_warning = nullptr) {
  if (sparse_warning) *sparse_warning = sample.n_obs() * 4 < static_cast<std::size_t>(model.grid().size());
  if (model.n_components() == 0) return {};
  return gpu::compute_scores_batch({&sample}, model, ScoreMethod::Integration)[0];
}

inline ScoreMethod choose_score_method(const FunctionalDataset& data, const EvaluationGrid& grid) {
  return data.median_obs_per_sample() >= 0.25 * static_cast<double>(grid.size()) ? ScoreMethod::Integration
                                                                                 : ScoreMethod::Pace;
}

inline std::vector<double> compute_scores(const Sample& sample, const FpcaModel& model, ScoreMethod method,
                                          bool* sparse_warning = nullptr) {
  return method == ScoreMethod::Pace ? pace_scores(sample, model) : integration_scores(sample, model, sparse_warning);
}

inline std::vector<double> reconstruct_on_grid(const FpcaModel& model, const std::vector<double>& scores) {
  const std::size_t L = model.n_components();
  if (scores.size() != L) throw err::invalid_argument("score vector length differs from component count");
  const auto G = static_cast<std::size_t>(model.grid().size());
  std::vector<double> funcs;
  funcs.reserve(L * G);
  for (const auto& f : model.eig.eigenfunctions) funcs.insert(funcs.end(), f.begin(), f.end());
  std::vector<double> out(G);
  gpu::GridDesc gd(model.grid());
  gpu::check(dfpca_reconstruct(gpu::context(), gd.get(), model.mean.values.data(), static_cast<int64_t>(L),
                               funcs.empty() ? nullptr : funcs.data(), 1, scores.empty() ? nullptr : scores.data(),
                               out.data()));
  return out;
}

inline std::vector<double> reconstruct_on_grid(const FpcaModel& model, std::size_t sample_index) {
  if (sample_index >= model.scores.size()) throw err::invalid_argument("sample index outside the fitted score table");
  return reconstruct_on_grid(model, model.scores[sample_index]);
}

inline double reconstruct_at(const FpcaModel& model, const std::vector<double>& scores, const double* coord) {
  const std::size_t L = model.n_components();
  if (scores.size() != L) throw err::invalid_argument("score vector length differs from component count");
  double x = interp_multilinear(model.grid(), model.mean.values, coord);
  if (is_outside(x)) return outside_value();
  for (std::size_t l = 0; l < L; ++l) {
    const double p = interp_multilinear(model.grid(), model.eig.eigenfunctions[l], coord);
    if (is_outside(p)) return outside_value();
    x += scores[l] * p;
  }
  return x;
}

inline double reconstruct_at(const FpcaModel& model, std::size_t sample_index, const double* coord) {
  if (sample_index >= model.scores.size()) throw err::invalid_argument("sample index outside the fitted score table");
  return reconstruct_at(model, model.scores[sample_index], coord);
}

struct HoldoutResult {
  std::vector<double> per_location;
  double mean = 0.0;
  double standard_error = 0.0;
};

inline HoldoutResult holdout_prediction_error(const FunctionalDataset& data,
                                              const std::vector<std::vector<double>>& locations,
                                              const FpcaModel& model, ScoreMethod method, double match_tol = 1e-9) {
  if (locations.size() < 2) throw err::invalid_argument("leave-one-location-out needs at least two locations");
  const std::size_t d = data.dim;
  for (const auto& s : locations)
    if (s.size() != d) throw err::invalid_argument("held-out location has the wrong dimension");
  std::vector<double> tol(d);
  for (std::size_t k = 0; k < d; ++k) tol[k] = match_tol * (model.grid().hull_hi(k) - model.grid().hull_lo(k));

  HoldoutResult out;
  out.per_location.assign(locations.size(), 0.0);
  for (std::size_t i = 0; i < locations.size(); ++i) {
    const double* s = locations[i].data();
    // every sample with an observation at the location, re-scored in one batch
    std::vector<Sample> reduced;
    std::vector<std::vector<double>> held;
    for (const auto& sample : data.samples) {
      Sample r;
      std::vector<double> hv;
      for (std::size_t j = 0; j < sample.n_obs(); ++j) {
        const double* c = sample.coord(j, d);
        bool at = true;
        for (std::size_t k = 0; k < d; ++k)
          if (std::abs(c[k] - s[k]) > tol[k]) {
            at = false;
            break;
          }
        if (at) {
          hv.push_back(sample.values[j]);
        } else {
          r.coords.insert(r.coords.end(), c, c + d);
          r.values.push_back(sample.values[j]);
        }
      }
      if (hv.empty()) continue;
      reduced.push_back(std::move(r));
      held.push_back(std::move(hv));
    }
    if (reduced.empty()) continue;
    std::vector<const Sample*> ptrs;
    for (const auto& r : reduced) ptrs.push_back(&r);
    const auto sc = gpu::compute_scores_batch(ptrs, model, method);
    for (std::size_t q = 0; q < reduced.size(); ++q) {
      const double pred = reconstruct_at(model, sc[q], s);
      if (is_outside(pred)) continue;
      for (double y : held[q]) out.per_location[i] += (y - pred) * (y - pred);
    }
  }
  const auto m = static_cast<double>(out.per_location.size());
  for (double e : out.per_location) out.mean += e;
  out.mean /= m;
  double var = 0.0;
  for (double e : out.per_location) var += (e - out.mean) * (e - out.mean);
  var /= (m - 1.0);
  out.standard_error = std::sqrt(var / m);
  return out;
}

}  // namespace dfpca
