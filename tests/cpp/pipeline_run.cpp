// TEST HARNESS: the reference's own fit_pipeline (pipeline.hpp) on a
// simulated dataset (simulate.hpp), compiled two ways from this one source --
// against the drop-in headers first (include/, the GPU path through
// libdfpca_cuda.so) or against the reference alone (the oracle build) -- and
// printed as one JSON line, so tests/test_gpu_pipeline.py can compare them.
//
//   pipeline_run sim1|sim2 randomized|dense
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
  const bool d3 = which == "sim2";
  const SimSpec spec = d3 ? sim2_spec(60, 8) : sim1_spec(200, 100, 100);
  const auto generated = generate(spec);
  const FunctionalDataset& data = generated.first;
  RunConfig cfg;
  cfg.grid_nodes = {d3 ? Index{8} : Index{100}};
  const double h = d3 ? 0.3 : 0.25;  // tests/acceptance.cpp:103-105 for sim1
  for (BandwidthChoice* c : {&cfg.bw_mean, &cfg.bw_cov, &cfg.bw_diag}) {
    c->mode = BandwidthMode::Explicit;
    c->values.assign(d3 ? 3 : 1, h);
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
