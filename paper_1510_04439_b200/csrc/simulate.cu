// Seeded synthetic datasets: a restatement of the reference's generator
// (simulate.hpp:163-245, RandomStream rng.hpp:30-78) for the models
// BASELINE.json's configs are quoted on.  Host code only: the
// draws are sequential per sample (one mt19937_64 substream each), so samples
// are generated in parallel on host threads and every value is bit-identical
// to the reference's generate() (tests/test_simulate.py checks that against
// the compiled reference).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "dfpca_cuda.h"

namespace {

std::uint64_t splitmix64(std::uint64_t x) {  // rng.hpp:12-17
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// RandomStream (rng.hpp:30-78): mt19937_64, 53-bit uniforms on (0,1),
// Box-Muller pairs (cos first, sin cached).
class Stream {
 public:
  static Stream substream(std::uint64_t seed, std::uint64_t index) {
    return Stream(splitmix64(seed) ^ splitmix64(index + 0x51ed2701a9e5a3d5ULL));
  }
  double uniform() { return (static_cast<double>(eng_() >> 11) + 0.5) * 0x1.0p-53; }
  double normal() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    const double u1 = uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare_ = r * std::sin(a);
    spare_ok_ = true;
    return r * std::cos(a);
  }
  std::uint64_t below(std::uint64_t n) {
    return static_cast<std::uint64_t>(uniform() * static_cast<double>(n)) % (n == 0 ? 1 : n);
  }

 private:
  explicit Stream(std::uint64_t seed) : eng_(splitmix64(seed)) {}  // rng.hpp:32-33
  std::mt19937_64 eng_;
  double spare_ = 0.0;
  bool spare_ok_ = false;
};

const double kPi = std::acos(-1.0);

// The models.  Each evaluates exactly the reference's expressions, in its
// order, so the doubles are the reference's.
struct Model {
  int kind;
  int dim;
  std::vector<double> lambda;
  double sigma2;

  double mean(const double* t) const {
    if (kind == DFPCA_SIM_SIM1) return t[0] + std::sin(t[0]);  // simulate.hpp:113
    double q = 0.0;  // simulate.hpp:132-136 (and its 2-d analogue)
    for (int k = 0; k < dim; ++k) q += (t[k] - 0.5) * (t[k] - 0.5);
    return std::exp(q);
  }
  double phi(int l, const double* t) const {  // l = 0-based component
    if (kind == DFPCA_SIM_SIM1) {  // simulate.hpp:115-117
      if (l == 0) return -std::cos(kPi * t[0] / 10.0) / std::sqrt(5.0);
      return std::sin(kPi * t[0] / 10.0) / std::sqrt(5.0);
    }
    // simulate.hpp:140-146: sqrt(2^d) prod_k sin(2 l pi t_k), l = 1..4
    const int ll = l + 1;
    double p = std::sqrt(dim == 3 ? 8.0 : 4.0);
    for (int k = 0; k < dim; ++k) p *= std::sin(2.0 * ll * kPi * t[k]);
    return p;
  }
};

Model model_of(int kind) {
  if (kind == DFPCA_SIM_SIM1) return {kind, 1, {4.0, 1.0}, 0.25};
  if (kind == DFPCA_SIM_SIM2) return {kind, 3, {16.0, 4.0, 1.0, 0.25}, 1.0 / 16.0};
  return {kind, 2, {16.0, 4.0, 1.0, 0.25}, 1.0 / 16.0};
}

// Config 4's domain: ellipse ((x-.5)/.45)^2 + ((y-.5)/.3)^2 <= 1.
bool in_ellipse(const double* c) {
  const double a = (c[0] - 0.5) / 0.45, b = (c[1] - 0.5) / 0.3;
  return a * a + b * b <= 1.0;
}

template <class F>
void parallel_samples(int64_t n, F&& f) {
  const int64_t hw = std::max<int64_t>(1, std::thread::hardware_concurrency());
  const int64_t nt = std::min<int64_t>(hw, std::max<int64_t>(1, n / 4));
  if (nt <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  for (int64_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (int64_t i = t; i < n; i += nt) f(i);
    });
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" DFPCA_API int dfpca_simulate(int kind, const dfpca_grid* grid, int64_t n, int64_t points_per_sample,
                                        uint64_t seed, int64_t* offsets, double* coords, double* values) {
  if (kind < DFPCA_SIM_SIM1 || kind > DFPCA_SIM_SPARSE2 || !grid || n <= 0 || !offsets) return 3;
  const Model m = model_of(kind);
  if (grid->dim != m.dim) return 3;
  const int d = m.dim;
  int64_t G = 1;
  for (int k = 0; k < d; ++k) {
    if (grid->shape[k] < 2 || !grid->axes[k]) return 3;
    G *= grid->shape[k];
  }
  const std::size_t L = m.lambda.size();
  double lo[DFPCA_MAX_DIM], hi[DFPCA_MAX_DIM];
  for (int k = 0; k < d; ++k) {
    lo[k] = grid->axes[k][0];  // hull_lo / hull_hi (grid.hpp:206-207)
    hi[k] = grid->axes[k][grid->shape[k] - 1];
  }

  // Observation coordinates of the deterministic designs (simulate.hpp:180-195).
  std::vector<double> fixed;
  if (kind == DFPCA_SIM_SIM2 || kind == DFPCA_SIM_IMAGES2) {
    for (int64_t f = 0; f < G; ++f) {
      if (grid->mask && !grid->mask[f]) continue;
      double c[DFPCA_MAX_DIM];
      int64_t r = f;
      for (int k = d - 1; k >= 0; --k) {
        c[k] = grid->axes[k][r % grid->shape[k]];
        r /= grid->shape[k];
      }
      fixed.insert(fixed.end(), c, c + d);
    }
  } else if (kind == DFPCA_SIM_SIM1) {
    if (points_per_sample <= 0) return 3;
    const int64_t p = points_per_sample;
    for (int64_t j = 0; j < p; ++j)
      fixed.push_back(p == 1 ? 0.5 * (lo[0] + hi[0])
                             : lo[0] + (hi[0] - lo[0]) * static_cast<double>(j) / static_cast<double>(p - 1));
  }

  // Sizes: fixed designs share one count; config 4 draws N_i ~ U{5..20} as
  // the first draw of the coordinate substream 3i+1.
  offsets[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t ni;
    if (kind == DFPCA_SIM_SPARSE2) {
      Stream cr = Stream::substream(seed, 3 * static_cast<std::uint64_t>(i) + 1);
      ni = 5 + static_cast<int64_t>(cr.below(16));
    } else {
      ni = static_cast<int64_t>(fixed.size()) / d;
    }
    offsets[i + 1] = offsets[i] + ni;
  }
  if (!coords || !values) return 0;

  const double noise_sd = std::sqrt(m.sigma2);
  parallel_samples(n, [&](int64_t i) {
    const auto iu = static_cast<std::uint64_t>(i);
    Stream score = Stream::substream(seed, 3 * iu);
    double a[8];
    for (std::size_t l = 0; l < L; ++l) a[l] = std::sqrt(m.lambda[l]) * score.normal();
    const int64_t o0 = offsets[i], ni = offsets[i + 1] - offsets[i];
    double* c = coords + o0 * d;
    if (kind == DFPCA_SIM_SPARSE2) {
      Stream cr = Stream::substream(seed, 3 * iu + 1);
      cr.below(16);  // the count drawn above
      for (int64_t j = 0; j < ni; ++j) {
        double p[2];
        do {
          for (int k = 0; k < 2; ++k) p[k] = lo[k] + (hi[k] - lo[k]) * cr.uniform();
        } while (!in_ellipse(p));
        c[j * 2] = p[0];
        c[j * 2 + 1] = p[1];
      }
    } else {
      std::copy(fixed.begin(), fixed.end(), c);
    }
    Stream noise = Stream::substream(seed, 3 * iu + 2);
    for (int64_t j = 0; j < ni; ++j) {  // simulate.hpp:226-240
      const double* t = c + j * d;
      double x = m.mean(t);
      for (std::size_t l = 0; l < L; ++l) x += a[l] * m.phi(static_cast<int>(l), t);
      values[o0 + j] = x + noise_sd * noise.normal();
    }
  });
  return 0;
}
