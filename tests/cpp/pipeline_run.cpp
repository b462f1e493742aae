// TEST HARNESS: the reference's own fit_pipeline (pipeline.hpp) on a
// simulated dataset (simulate.hpp), compiled two ways from this one source --
// against the drop-in headers first (include/, the GPU path through
// libdfpca_cuda.so) or against the reference alone (the oracle build) -- and
// printed as one JSON line, so tests/test_gpu_pipeline.py can compare them.
//
//   pipeline_run sim1|grid2d|random2d randomized|dense
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "dfpca/pipeline.hpp"
#include "dfpca/simulate.hpp"

using namespace dfpca;

static void print_list(const char* key, const std::vector<double>& v, bool last = false) {
  std::printf("\"%s\": [", key);
  for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
  std::printf("]%s", last ? "" : ", ");
}

int main(int argc, char** argv) {
  const std::string which = argc > 1 ? argv[1] : "sim1";
  const std::string eig = argc > 2 ? argv[2] : "randomized";
  const bool d2 = which != "sim1";
  SimSpec spec = sim1_spec(200, 100, 100);
  if (d2) {
    // SURVEY.md 8(d) config 2's process on a 24^2 midpoint grid: exp bump
    // mean, 2 prod_k sin(2 pi l t_k), lambda 16, 4, 1, 0.25, sigma^2 = 1/16;
    // every node observed (grid2d) or 40 uniform random points (random2d)
    spec = SimSpec{};
    spec.name = which;
    spec.n = 60;
    spec.grid = EvaluationGrid::midpoint({0.0, 0.0}, {1.0, 1.0}, {24, 24});
    spec.design = which == "grid2d" ? SimDesign::GridNodes : SimDesign::UniformRandom;
    spec.points_per_sample = which == "grid2d" ? 0 : 40;
    spec.mean = [](const double* t) { return std::exp((t[0] - 0.5) * (t[0] - 0.5) + (t[1] - 0.5) * (t[1] - 0.5)); };
    const double pi = std::acos(-1.0);
    for (int l = 1; l <= 4; ++l)
      spec.eigenfunctions.push_back(
          [pi, l](const double* t) { return 2.0 * std::sin(2.0 * l * pi * t[0]) * std::sin(2.0 * l * pi * t[1]); });
    spec.lambda = {16.0, 4.0, 1.0, 0.25};
    spec.sigma2 = 1.0 / 16.0;
  }
  const auto generated = generate(spec);
  const FunctionalDataset& data = generated.first;
  RunConfig cfg;
  cfg.grid_nodes = {d2 ? Index{24} : Index{100}};
  const double h = d2 ? 0.15 : 0.25;  // tests/acceptance.cpp:103-105 for sim1
  for (BandwidthChoice* c : {&cfg.bw_mean, &cfg.bw_cov, &cfg.bw_diag}) {
    c->mode = BandwidthMode::Explicit;
    c->values.assign(d2 ? 2 : 1, h);
  }
  cfg.max_components = 5;
  cfg.eig_method = eig == "dense" ? EigMethod::Dense : EigMethod::Randomized;
  cfg.threads = 4;
  set_max_threads(cfg.threads);
  try {
    const auto fit = fit_pipeline(data, cfg);
    const FpcaModel& m = fit.first;
    const FitReport& r = fit.second;
    std::printf("{\"ok\": true, \"sigma2\": %.17g, \"total_variance\": %.17g, \"n_components\": %zu, ", m.sigma2,
                r.total_variance, r.n_components);
    print_list("eigenvalues", r.eigenvalues);
    print_list("fve", r.fve);
    print_list("h_cov", r.h_cov.h);
    std::vector<double> sc;
    for (std::size_t i = 0; i < 5 && i < m.scores.size(); ++i) sc.insert(sc.end(), m.scores[i].begin(), m.scores[i].end());
    print_list("scores_head", sc);
    std::vector<double> phi0 = m.eig.eigenfunctions.empty() ? std::vector<double>{} : m.eig.eigenfunctions[0];
    print_list("phi0", phi0);
    std::printf("\"score_method\": \"%s\", \"fit_s\": %.6f}\n", score_method_name(r.score_method).c_str(), [&] {
      double t = 0.0;
      for (const auto& s : r.timings) t += s.seconds;
      return t;
    }());
  } catch (const Error& e) {
    std::printf("{\"ok\": false, \"error\": \"%s\"}\n", e.what());
    return 1;
  }
  return 0;
}
