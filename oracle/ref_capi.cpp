// TEST INFRASTRUCTURE ONLY -- the parity oracle.
//
// extern "C" driver over the reference implementation itself: the reference's
// own headers (/root/reference/proj/include/dfpca/*.hpp) are compiled
// UNCHANGED against the shims in oracle/shim (Eigen subset, FFTW, LAPACKE)
// into oracle/_ref/libdfpca_ref.so by oracle/Makefile.  Nothing from the
// product links this; only tests/, __graft_entry__.smoke() and bench.py's
// CPU baseline / reference arm load it.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "dfpca/bandwidth.hpp"
#include "dfpca/binning.hpp"
#include "dfpca/dataset.hpp"
#include "dfpca/eigensolve.hpp"
#include "dfpca/errors.hpp"
#include "dfpca/fft_smoother.hpp"
#include "dfpca/grid.hpp"
#include "dfpca/io.hpp"
#include "dfpca/parallel.hpp"
#include "dfpca/scores.hpp"
#include "dfpca/simulate.hpp"
#include "dfpca/smoother.hpp"

using namespace dfpca;

namespace {

thread_local std::string g_err;
thread_local int g_cls = 0;

template <class F>
int guarded(F&& f) {
  g_err.clear();
  g_cls = 0;
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    g_cls = static_cast<int>(e.error_class());
  } catch (const std::exception& e) {
    g_err = std::string("InternalError: ") + e.what();
    g_cls = 4;
  }
  return g_cls;
}

EvaluationGrid make_grid(int dim, const int64_t* shape, const double* axes, const uint8_t* mask) {
  std::vector<std::vector<double>> ax(static_cast<std::size_t>(dim));
  std::size_t off = 0, total = 1;
  for (int k = 0; k < dim; ++k) {
    ax[static_cast<std::size_t>(k)].assign(axes + off, axes + off + shape[k]);
    off += static_cast<std::size_t>(shape[k]);
    total *= static_cast<std::size_t>(shape[k]);
  }
  if (mask) return EvaluationGrid(std::move(ax), std::vector<std::uint8_t>(mask, mask + total));
  return EvaluationGrid(std::move(ax));
}

FunctionalDataset make_data(int dim, int64_t n, const int64_t* offsets, const double* coords,
                            const double* values) {
  FunctionalDataset d;
  d.dim = static_cast<std::size_t>(dim);
  d.samples.resize(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    Sample& s = d.samples[static_cast<std::size_t>(i)];
    s.id = std::to_string(i);
    s.coords.assign(coords + offsets[i] * dim, coords + offsets[i + 1] * dim);
    s.values.assign(values + offsets[i], values + offsets[i + 1]);
  }
  return d;
}

BlockPlan plan_for(const EvaluationGrid& g, const Bandwidth& h, int64_t n_blocks) {
  return n_blocks > 0 ? make_block_plan(g, h, n_blocks) : single_block_plan(g, h);
}

void put_eig(const EigenSystem& es, int64_t L_cap, int64_t G, double* evals, double* efuncs, double* fve,
             double* total, int64_t* n_out) {
  const int64_t L = std::min<int64_t>(static_cast<int64_t>(es.eigenvalues.size()), L_cap);
  for (int64_t l = 0; l < L; ++l) {
    evals[l] = es.eigenvalues[static_cast<std::size_t>(l)];
    fve[l] = es.fve[static_cast<std::size_t>(l)];
    std::memcpy(efuncs + l * G, es.eigenfunctions[static_cast<std::size_t>(l)].data(),
                sizeof(double) * static_cast<std::size_t>(G));
  }
  *total = es.total_variance;
  *n_out = L;
}

}  // namespace

extern "C" {

const char* ref_last_error(int* cls) {
  if (cls) *cls = g_cls;
  return g_err.c_str();
}

void ref_set_threads(int n) { set_max_threads(n); }

int ref_linear_bin(int dim, const int64_t* shape, const double* axes, const uint8_t* mask, int64_t n,
                   const int64_t* offsets, const double* coords, const double* values, int mean_path,
                   int cov_path, void** out) {
  return guarded([&] {
    auto g = make_grid(dim, shape, axes, mask);
    auto data = make_data(dim, n, offsets, coords, values);
    auto* b = new BinnedData(linear_bin(data, g, BinOptions{mean_path != 0, cov_path != 0}));
    *out = b;
  });
}

int ref_binned_from_host(int dim, const int64_t* shape, const double* axes, const uint8_t* mask,
                         int64_t n_samples, const int64_t* sample_sizes, int has_mean, const double* mass,
                         const double* wvalue, const double* wsquare, int has_cov, int64_t n_pair,
                         const int64_t* sample_index, const double* pair_weight, const double* ps_mass,
                         const double* ps_value, const double* diag_mass, const double* diag_value,
                         void** out) {
  return guarded([&] {
    auto* b = new BinnedData();
    b->grid = make_grid(dim, shape, axes, mask);
    const auto G = static_cast<std::size_t>(b->grid.size());
    b->has_mean_path = has_mean != 0;
    b->has_covariance_path = has_cov != 0;
    for (int64_t i = 0; i < n_samples; ++i) b->sample_sizes.push_back(static_cast<std::size_t>(sample_sizes[i]));
    if (has_mean) {
      b->mass.assign(mass, mass + G);
      b->wvalue.assign(wvalue, wvalue + G);
      b->wsquare.assign(wsquare, wsquare + G);
    }
    if (has_cov) {
      const std::size_t codes = b->offset_codes();
      b->diag_mass.assign(diag_mass, diag_mass + G * codes);
      b->diag_value.assign(diag_value, diag_value + G * codes);
      for (int64_t i = 0; i < n_pair; ++i) {
        BinnedData::SampleGrids sg;
        sg.sample_index = static_cast<std::size_t>(sample_index[i]);
        sg.pair_weight = pair_weight[i];
        sg.mass.assign(ps_mass + i * G, ps_mass + (i + 1) * G);
        sg.value.assign(ps_value + i * G, ps_value + (i + 1) * G);
        b->per_sample.push_back(std::move(sg));
      }
    }
    *out = b;
  });
}

int ref_binned_info(void* h, int64_t* n_samples, int64_t* n_pair, int64_t* G, int64_t* codes) {
  auto* b = static_cast<BinnedData*>(h);
  *n_samples = static_cast<int64_t>(b->sample_sizes.size());
  *n_pair = static_cast<int64_t>(b->per_sample.size());
  *G = b->grid.size();
  *codes = static_cast<int64_t>(b->offset_codes());
  return 0;
}

int ref_binned_download(void* h, double* mass, double* wvalue, double* wsquare, int64_t* sample_index,
                        double* pair_weight, double* ps_mass, double* ps_value, double* diag_mass,
                        double* diag_value, int64_t* sample_sizes) {
  auto* b = static_cast<BinnedData*>(h);
  const auto G = static_cast<std::size_t>(b->grid.size());
  auto cp = [](double* dst, const std::vector<double>& src) {
    if (dst && !src.empty()) std::memcpy(dst, src.data(), sizeof(double) * src.size());
  };
  cp(mass, b->mass);
  cp(wvalue, b->wvalue);
  cp(wsquare, b->wsquare);
  cp(diag_mass, b->diag_mass);
  cp(diag_value, b->diag_value);
  for (std::size_t i = 0; i < b->per_sample.size(); ++i) {
    if (sample_index) sample_index[i] = static_cast<int64_t>(b->per_sample[i].sample_index);
    if (pair_weight) pair_weight[i] = b->per_sample[i].pair_weight;
    if (ps_mass) std::memcpy(ps_mass + i * G, b->per_sample[i].mass.data(), sizeof(double) * G);
    if (ps_value) std::memcpy(ps_value + i * G, b->per_sample[i].value.data(), sizeof(double) * G);
  }
  if (sample_sizes)
    for (std::size_t i = 0; i < b->sample_sizes.size(); ++i) sample_sizes[i] = static_cast<int64_t>(b->sample_sizes[i]);
  return 0;
}

void ref_binned_free(void* h) { delete static_cast<BinnedData*>(h); }

int ref_local_linear(void* h, int dim, const int64_t* shape, const double* axes, const uint8_t* mask,
                     const double* bw, int target, int64_t n_blocks, double* out) {
  return guarded([&] {
    auto* b = static_cast<BinnedData*>(h);
    auto g = make_grid(dim, shape, axes, mask);
    Bandwidth hb{std::vector<double>(bw, bw + dim)};
    const MomentTarget t = target == 0 ? MomentTarget::Mean : MomentTarget::Squares;
    auto est = n_blocks > 0 ? blockwise_apply(plan_for(g, hb, n_blocks), *b, g, hb, t)
                            : fft_local_linear(*b, g, hb, t);
    std::memcpy(out, est.values.data(), sizeof(double) * est.values.size());
  });
}

int ref_covariance(void* h, int dim, const int64_t* shape, const double* axes, const uint8_t* mask,
                   const double* bw, const double* mean, int64_t n_blocks, int mode, double* out) {
  return guarded([&] {
    auto* b = static_cast<BinnedData*>(h);
    auto g = make_grid(dim, shape, axes, mask);
    Bandwidth hb{std::vector<double>(bw, bw + dim)};
    SurfaceEstimate mu;
    mu.grid = g;
    mu.kind = SurfaceKind::Mean;
    mu.values.assign(mean, mean + g.size());
    const auto m = static_cast<PairGridSource::Mode>(mode);
    auto est = fft_covariance(*b, g, hb, mu, plan_for(g, hb, n_blocks), m);
    std::memcpy(out, est.values.data(), sizeof(double) * est.values.size());
  });
}

int ref_pair_grids(void* h, int mode, double* pw, double* pv) {
  return guarded([&] {
    auto* b = static_cast<BinnedData*>(h);
    PairGridSource src(*b, static_cast<PairGridSource::Mode>(mode));
    std::vector<double> a, c;
    src.extract(src.full_box(), a, c);
    std::memcpy(pw, a.data(), sizeof(double) * a.size());
    std::memcpy(pv, c.data(), sizeof(double) * c.size());
  });
}

int ref_randomized_eig(int dim, const int64_t* shape, const double* axes, const uint8_t* mask,
                       const double* cov, int64_t q, int64_t L_max, uint64_t seed, double* evals,
                       double* efuncs, double* fve, double* total, int64_t* n_out) {
  return guarded([&] {
    SurfaceEstimate s;
    s.grid = make_grid(dim, shape, axes, mask);
    s.kind = SurfaceKind::Covariance;
    const auto G = s.grid.size();
    s.values.assign(cov, cov + G * G);
    auto S = matrixize(s);
    auto es = randomized_eig(S, static_cast<std::size_t>(q), static_cast<std::size_t>(L_max), s.grid, seed);
    put_eig(es, L_max, G, evals, efuncs, fve, total, n_out);
  });
}

int ref_dense_eig(int dim, const int64_t* shape, const double* axes, const uint8_t* mask, const double* cov,
                  int64_t L_max, double* evals, double* efuncs, double* fve, double* total, int64_t* n_out) {
  return guarded([&] {
    SurfaceEstimate s;
    s.grid = make_grid(dim, shape, axes, mask);
    s.kind = SurfaceKind::Covariance;
    const auto G = s.grid.size();
    s.values.assign(cov, cov + G * G);
    auto S = matrixize(s);
    auto es = dense_eig(S, static_cast<std::size_t>(L_max), s.grid);
    put_eig(es, L_max, G, evals, efuncs, fve, total, n_out);
  });
}

int ref_eig_residuals(int dim, const int64_t* shape, const double* axes, const uint8_t* mask,
                      const double* cov, int64_t L, const double* evals, const double* efuncs, double* out) {
  return guarded([&] {
    SurfaceEstimate s;
    s.grid = make_grid(dim, shape, axes, mask);
    s.kind = SurfaceKind::Covariance;
    const auto G = s.grid.size();
    s.values.assign(cov, cov + G * G);
    auto S = matrixize(s);
    EigenSystem es;
    for (int64_t l = 0; l < L; ++l) {
      es.eigenvalues.push_back(evals[l]);
      es.eigenfunctions.emplace_back(efuncs + l * G, efuncs + (l + 1) * G);
    }
    auto r = eig_residuals(S, es, s.grid);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}

int ref_estimate_mean(int dim, const int64_t* shape, const double* axes, const uint8_t* mask, int64_t n,
                      const int64_t* offsets, const double* coords, const double* values, const double* bw,
                      int squares, double* out) {
  return guarded([&] {
    auto g = make_grid(dim, shape, axes, mask);
    auto data = make_data(dim, n, offsets, coords, values);
    Bandwidth hb{std::vector<double>(bw, bw + dim)};
    auto est = squares ? estimate_diag_plus_noise(data, g, hb) : estimate_mean(data, g, hb);
    std::memcpy(out, est.values.data(), sizeof(double) * est.values.size());
  });
}

int ref_estimate_covariance(int dim, const int64_t* shape, const double* axes, const uint8_t* mask,
                            int64_t n, const int64_t* offsets, const double* coords, const double* values,
                            const double* bw, const double* mean, double* out) {
  return guarded([&] {
    auto g = make_grid(dim, shape, axes, mask);
    auto data = make_data(dim, n, offsets, coords, values);
    Bandwidth hb{std::vector<double>(bw, bw + dim)};
    SurfaceEstimate mu;
    mu.grid = g;
    mu.kind = SurfaceKind::Mean;
    mu.values.assign(mean, mean + g.size());
    auto est = estimate_covariance(data, g, hb, mu);
    std::memcpy(out, est.values.data(), sizeof(double) * est.values.size());
  });
}

// ---- noise variance, scores, reconstruction (scores.hpp) ----

static FpcaModel make_model(int dim, const int64_t* shape, const double* axes, const uint8_t* mask,
                            const double* mean, int64_t L, const double* evals, const double* efuncs,
                            double sigma2) {
  FpcaModel m;
  m.mean.grid = make_grid(dim, shape, axes, mask);
  m.mean.kind = SurfaceKind::Mean;
  const auto G = static_cast<std::size_t>(m.mean.grid.size());
  m.mean.values.assign(mean, mean + G);
  for (int64_t l = 0; l < L; ++l) {
    m.eig.eigenvalues.push_back(evals[l]);
    m.eig.eigenfunctions.emplace_back(efuncs + l * G, efuncs + (l + 1) * G);
  }
  m.sigma2 = sigma2;
  return m;
}

int ref_estimate_sigma2(int dim, const int64_t* shape, const double* axes, const uint8_t* mask,
                        const double* diag, const double* cov, const double* mean, double* out) {
  return guarded([&] {
    EvaluationGrid g = make_grid(dim, shape, axes, mask);
    const auto G = static_cast<std::size_t>(g.size());
    SurfaceEstimate dn{g, std::vector<double>(diag, diag + G), SurfaceKind::DiagPlusNoise};
    SurfaceEstimate cv{g, std::vector<double>(cov, cov + G * G), SurfaceKind::Covariance};
    SurfaceEstimate mu{g, std::vector<double>(mean, mean + G), SurfaceKind::Mean};
    *out = estimate_sigma2(dn, cv, mu);
  });
}

// method 0 = pace, 1 = integration; scores[n][L]; sparse[n] (integration only)
int ref_scores(int dim, const int64_t* shape, const double* axes, const uint8_t* mask, int64_t n,
               const int64_t* offsets, const double* coords, const double* values, const double* mean,
               int64_t L, const double* evals, const double* efuncs, double sigma2, int method, double* scores,
               int* sparse) {
  return guarded([&] {
    FpcaModel m = make_model(dim, shape, axes, mask, mean, L, evals, efuncs, sigma2);
    FunctionalDataset data = make_data(dim, n, offsets, coords, values);
    for (int64_t i = 0; i < n; ++i) {
      bool w = false;
      const auto sc = compute_scores(data.samples[static_cast<std::size_t>(i)], m,
                                     method == 0 ? ScoreMethod::Pace : ScoreMethod::Integration, &w);
      for (int64_t l = 0; l < L; ++l) scores[i * L + l] = sc[static_cast<std::size_t>(l)];
      if (sparse) sparse[i] = w ? 1 : 0;
    }
  });
}

int ref_reconstruct(int dim, const int64_t* shape, const double* axes, const uint8_t* mask, const double* mean,
                    int64_t L, const double* evals, const double* efuncs, const double* sc, double* out) {
  return guarded([&] {
    FpcaModel m = make_model(dim, shape, axes, mask, mean, L, evals, efuncs, 0.0);
    const auto r = reconstruct_on_grid(m, std::vector<double>(sc, sc + L));
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}

// ---- the CV bandwidth objective (bandwidth.hpp:56-163) ----
// target 0 = mean, 1 = covariance, 2 = diag (squares)
int ref_cv_score(int dim, const int64_t* shape, const double* axes, const uint8_t* mask, int64_t n,
                 const int64_t* offsets, const double* coords, const double* values, int target, int64_t max_units,
                 uint64_t seed, const double* h, double* out, int64_t* n_units) {
  return guarded([&] {
    EvaluationGrid g = make_grid(dim, shape, axes, mask);
    FunctionalDataset data = make_data(dim, n, offsets, coords, values);
    const CvTarget t = target == 0 ? CvTarget::Mean : target == 1 ? CvTarget::Covariance : CvTarget::DiagPlusNoise;
    CvObjective obj(data, g, t, CvOptions{static_cast<std::size_t>(max_units), seed});
    Bandwidth bw;
    bw.h.assign(h, h + dim);
    *out = cv_score(bw, obj);
    if (n_units) *n_units = static_cast<int64_t>(obj.n_units());
  });
}

// ---- io.hpp (long-format tables, grid files) --------------------------------
struct RefTable {
  int dim = 0;
  std::vector<int64_t> off{0}, id_off{0};
  std::vector<double> coords, values;
  std::string ids;
};

int ref_read_long_format(const char* path, void** out) {
  return guarded([&] {
    const FunctionalDataset data = read_long_format(path);
    auto* t = new RefTable;
    t->dim = static_cast<int>(data.dim);
    for (const auto& s : data.samples) {
      t->coords.insert(t->coords.end(), s.coords.begin(), s.coords.end());
      t->values.insert(t->values.end(), s.values.begin(), s.values.end());
      t->off.push_back(static_cast<int64_t>(t->values.size()));
      t->ids += s.id;
      t->id_off.push_back(static_cast<int64_t>(t->ids.size()));
    }
    *out = t;
  });
}

void ref_table_info(void* h, int* dim, int64_t* n_samples, int64_t* n_obs, int64_t* id_bytes) {
  const auto* t = static_cast<RefTable*>(h);
  *dim = t->dim;
  *n_samples = static_cast<int64_t>(t->off.size()) - 1;
  *n_obs = static_cast<int64_t>(t->values.size());
  *id_bytes = static_cast<int64_t>(t->ids.size());
}

void ref_table_copy(void* h, int64_t* off, double* coords, double* values, int64_t* id_off, char* ids) {
  const auto* t = static_cast<RefTable*>(h);
  std::memcpy(off, t->off.data(), sizeof(int64_t) * t->off.size());
  if (!t->coords.empty()) std::memcpy(coords, t->coords.data(), sizeof(double) * t->coords.size());
  if (!t->values.empty()) std::memcpy(values, t->values.data(), sizeof(double) * t->values.size());
  std::memcpy(id_off, t->id_off.data(), sizeof(int64_t) * t->id_off.size());
  if (!t->ids.empty()) std::memcpy(ids, t->ids.data(), t->ids.size());
}

void ref_table_free(void* h) { delete static_cast<RefTable*>(h); }

int ref_write_long_format(const char* path, int dim, int64_t n, const int64_t* off, const double* coords,
                          const double* values, const int64_t* id_off, const char* ids) {
  return guarded([&] {
    FunctionalDataset data;
    data.dim = static_cast<std::size_t>(dim);
    for (int64_t i = 0; i < n; ++i) {
      Sample s;
      s.id.assign(ids + id_off[i], ids + id_off[i + 1]);
      s.coords.assign(coords + off[i] * dim, coords + off[i + 1] * dim);
      s.values.assign(values + off[i], values + off[i + 1]);
      data.samples.push_back(std::move(s));
    }
    write_long_format(path, data);
  });
}

int ref_write_grid(const char* path, int dim, const int64_t* shape, const double* axes, const uint8_t* mask) {
  return guarded([&] { write_grid(path, make_grid(dim, shape, axes, mask)); });
}

// shape: capacity 16; axes: capacity sum(shape) (call with axes == NULL first)
int ref_read_grid(const char* path, int* dim, int64_t* shape, double* axes, uint8_t* mask, int* has_mask) {
  return guarded([&] {
    const EvaluationGrid g = read_grid(path);
    *dim = static_cast<int>(g.dim());
    *has_mask = g.has_mask() ? 1 : 0;
    std::size_t off = 0;
    for (std::size_t k = 0; k < g.dim() && k < 16; ++k) {
      shape[k] = static_cast<int64_t>(g.axis(k).size());
      if (axes) std::memcpy(axes + off, g.axis(k).data(), sizeof(double) * g.axis(k).size());
      off += g.axis(k).size();
    }
    if (mask && g.has_mask())
      for (Index f = 0; f < g.size(); ++f) mask[f] = g.in_mask(f) ? 1 : 0;
  });
}

// ---- simulate.hpp: the configs' inputs drawn by the reference's generator ----
// kind 1 sim1_spec, 2 sim2_spec, 3 the 2-d analogue of sim2 (SURVEY 8(d)
// configs 2/3), 4 config 4's sparse design (a thin custom generator over the
// reference's RandomStream with generate()'s substream layout).  Two calls:
// coords == NULL sizes offsets[n+1].
int ref_simulate(int kind, int dim, const int64_t* shape, const double* axes, const uint8_t* mask, int64_t n,
                 int64_t ppp, uint64_t seed, int64_t* offsets, double* coords, double* values) {
  return guarded([&] {
    const EvaluationGrid g = make_grid(dim, shape, axes, mask);
    FunctionalDataset data;
    if (kind == 1 || kind == 2 || kind == 3) {
      SimSpec spec;
      if (kind == 1) {
        spec = sim1_spec(static_cast<std::size_t>(n), static_cast<std::size_t>(ppp), shape[0], seed);
        spec.grid = g;
      } else if (kind == 2) {
        spec = sim2_spec(static_cast<std::size_t>(n), shape[0], seed);
        spec.grid = g;
      } else {
        spec.name = "images2";
        spec.n = static_cast<std::size_t>(n);
        spec.design = SimDesign::GridNodes;
        spec.grid = g;
        spec.seed = seed;
        spec.mean = [](const double* t) {
          double q = 0.0;
          for (std::size_t k = 0; k < 2; ++k) q += (t[k] - 0.5) * (t[k] - 0.5);
          return std::exp(q);
        };
        const double pi = std::acos(-1.0);
        for (int l = 1; l <= 4; ++l)
          spec.eigenfunctions.push_back([pi, l](const double* t) {
            double p = std::sqrt(4.0);
            for (std::size_t k = 0; k < 2; ++k) p *= std::sin(2.0 * l * pi * t[k]);
            return p;
          });
        spec.lambda = {16.0, 4.0, 1.0, 0.25};
        spec.sigma2 = 1.0 / 16.0;
      }
      spec.store_grid_truth = false;
      data = generate(spec).first;
    } else if (kind == 4) {
      const double pi = std::acos(-1.0);
      const double lam[4] = {16.0, 4.0, 1.0, 0.25};
      data.dim = 2;
      data.samples.resize(static_cast<std::size_t>(n));
      for (int64_t i = 0; i < n; ++i) {
        const auto iu = static_cast<std::uint64_t>(i);
        RandomStream sr = RandomStream::substream(seed, 3 * iu);
        double a[4];
        for (int l = 0; l < 4; ++l) a[l] = std::sqrt(lam[l]) * sr.normal();
        RandomStream cr = RandomStream::substream(seed, 3 * iu + 1);
        const std::size_t ni = 5 + static_cast<std::size_t>(cr.below(16));
        Sample& s = data.samples[static_cast<std::size_t>(i)];
        for (std::size_t j = 0; j < ni; ++j) {
          double p[2];
          for (;;) {
            for (std::size_t k = 0; k < 2; ++k) p[k] = g.hull_lo(k) + (g.hull_hi(k) - g.hull_lo(k)) * cr.uniform();
            const double u = (p[0] - 0.5) / 0.45, v = (p[1] - 0.5) / 0.3;
            if (u * u + v * v <= 1.0) break;
          }
          s.coords.push_back(p[0]);
          s.coords.push_back(p[1]);
        }
        RandomStream nr = RandomStream::substream(seed, 3 * iu + 2);
        for (std::size_t j = 0; j < ni; ++j) {
          const double* t = s.coords.data() + 2 * j;
          double q = 0.0;
          for (std::size_t k = 0; k < 2; ++k) q += (t[k] - 0.5) * (t[k] - 0.5);
          double x = std::exp(q);
          for (int l = 0; l < 4; ++l) {
            double ph = std::sqrt(4.0);
            for (std::size_t k = 0; k < 2; ++k) ph *= std::sin(2.0 * (l + 1) * pi * t[k]);
            x += a[l] * ph;
          }
          s.values.push_back(x + std::sqrt(1.0 / 16.0) * nr.normal());
        }
      }
    } else {
      throw err::invalid_argument("unknown simulation kind");
    }
    offsets[0] = 0;
    for (std::size_t i = 0; i < data.samples.size(); ++i)
      offsets[i + 1] = offsets[i] + static_cast<int64_t>(data.samples[i].values.size());
    if (!coords || !values) return;
    for (std::size_t i = 0; i < data.samples.size(); ++i) {
      const Sample& s = data.samples[i];
      std::memcpy(coords + offsets[i] * dim, s.coords.data(), sizeof(double) * s.coords.size());
      std::memcpy(values + offsets[i], s.values.data(), sizeof(double) * s.values.size());
    }
  });
}

// ---- fft_covariance restricted to one pair of output boxes ------------------
// The body of the reference's (bs, bt) loop (fft_smoother.hpp:627-719) run for
// core boxes S and T (d-dim, [lo, hi)) and for (T, S), then the centering and
// symmetrization (fft_smoother.hpp:723-736) of the S x T entries: the
// reference's values for a sub-block of a covariance too large to compute
// whole on the host (config 5, 1.07e9 points).  The block sits inside
// fft_covariance's own plan-invariance guarantee (fft_smoother.hpp:24-29).
// Empty kernel windows raise (no enlargement ladder here).  out: |S| x |T|.
int ref_covariance_block(void* h, int dim, const int64_t* shape, const double* axes, const uint8_t* mask,
                         const double* bw, const double* mean, const int64_t* s_lo, const int64_t* s_hi,
                         const int64_t* t_lo, const int64_t* t_hi, double* out) {
  return guarded([&] {
    auto* b = static_cast<BinnedData*>(h);
    const auto grid = make_grid(dim, shape, axes, mask);
    const std::size_t d = grid.dim();
    Bandwidth hb{std::vector<double>(bw, bw + dim)};
    hb.validate(grid);
    PairGridSource source(*b, PairGridSource::Mode::Rebuild);
    std::vector<double> spacing2(2 * d), h2(2 * d);
    std::vector<Index> shape2 = grid.shape();
    shape2.insert(shape2.end(), grid.shape().begin(), grid.shape().end());
    for (std::size_t k = 0; k < d; ++k) {
      spacing2[k] = spacing2[d + k] = grid.spacing(k);
      h2[k] = h2[d + k] = hb[k];
    }
    detail::MomentEngineBank bank(h2, spacing2, shape2);
    const std::size_t nm = bank.basis.count(), nl = bank.basis.count_linear();
    Box bs{std::vector<Index>(s_lo, s_lo + dim), std::vector<Index>(s_hi, s_hi + dim)};
    Box bt{std::vector<Index>(t_lo, t_lo + dim), std::vector<Index>(t_hi, t_hi + dim)};
    // raw[a][b] for the pair (A, B) of boxes, box-major over A then B
    auto raw_block = [&](const Box& A, const Box& B) {
      Box core2{A.lo, A.hi};
      core2.lo.insert(core2.lo.end(), B.lo.begin(), B.lo.end());
      core2.hi.insert(core2.hi.end(), B.hi.begin(), B.hi.end());
      const Box in_box = bank.engines[0]->required_input_box(core2);
      std::vector<double> pw_in, pv_in;
      source.extract(in_box, pw_in, pv_in);
      const auto core_n = static_cast<std::size_t>(core2.volume());
      std::vector<std::vector<double>> S(nm), T(nl);
      for (std::size_t i = 0; i < nm; ++i) {
        S[i].assign(core_n, 0.0);
        bank.engines[i]->run(pw_in.data(), in_box, S[i].data(), core2);
      }
      for (std::size_t i = 0; i < nl; ++i) {
        T[i].assign(core_n, 0.0);
        bank.engines[i]->run(pv_in.data(), in_box, T[i].data(), core2);
      }
      std::vector<Index> core_ext(2 * d);
      for (std::size_t k = 0; k < 2 * d; ++k) core_ext[k] = core2.extent(k);
      const std::vector<Index> core_str = detail::strides_of(core_ext);
      auto pair_nodes = [&](Index local, Index& s_flat, Index& t_flat) {
        s_flat = 0;
        t_flat = 0;
        for (std::size_t k = 0; k < d; ++k) {
          s_flat += (core2.lo[k] + (local / core_str[k]) % core_ext[k]) * grid.strides()[k];
          t_flat += (core2.lo[d + k] + (local / core_str[d + k]) % core_ext[d + k]) * grid.strides()[k];
        }
      };
      std::vector<double> res(core_n, outside_value());
      detail::solve_binned_box(
          bank.basis, S, T, core2.volume(),
          [&](Index local) {
            Index s_flat, t_flat;
            pair_nodes(local, s_flat, t_flat);
            return grid.in_mask(s_flat) && grid.in_mask(t_flat);
          },
          [&](Index, double, Eigen::MatrixXd&, Eigen::VectorXd&) { return false; },
          [&](Index local, double v) { res[static_cast<std::size_t>(local)] = v; },
          "binned covariance smoother (block)");
      return res;
    };
    const std::vector<double> st = raw_block(bs, bt);
    const std::vector<double> ts = raw_block(bt, bs);
    const std::vector<Index>& str = grid.strides();
    auto flat_of = [&](const Box& B, Index local) {
      Index f = 0, r = local;
      for (std::size_t k = d; k-- > 0;) {
        const Index e = B.hi[k] - B.lo[k];
        f += (B.lo[k] + r % e) * str[k];
        r /= e;
      }
      return f;
    };
    const Index ns = bs.volume(), nt = bt.volume();
    for (Index i = 0; i < ns; ++i) {
      const Index a = flat_of(bs, i);
      for (Index j = 0; j < nt; ++j) {
        const Index c = flat_of(bt, j);
        double v_ab = st[static_cast<std::size_t>(i * nt + j)];
        double v_ba = ts[static_cast<std::size_t>(j * ns + i)];
        if (grid.in_mask(a) && grid.in_mask(c)) {
          v_ab -= mean[a] * mean[c];
          v_ba -= mean[c] * mean[a];
        }
        double v = v_ab;
        if (a != c) {
          const double lo_hi = a < c ? v_ab : v_ba;  // the entry the reference tests for "outside"
          if (!is_outside(lo_hi)) v = 0.5 * (a < c ? v_ab + v_ba : v_ba + v_ab);
        }
        out[i * nt + j] = v;
      }
    }
  });
}

}  // extern "C"
