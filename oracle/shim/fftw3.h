// Stand-in for the five FFTW3 calls of the reference's conv.hpp
// (conv.hpp:103-125, 188-192).  TEST INFRASTRUCTURE ONLY (oracle/_ref).
// Real-input transforms of any length by direct O(n^2) summation with a
// precomputed twiddle table: FFTW's r2c is the unnormalized forward DFT
// (k = 0..n/2), c2r the unnormalized inverse of a Hermitian spectrum.
#pragma once

#include <cmath>
#include <vector>

typedef double fftw_complex[2];

#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

struct fftw_plan_s {
  int n;
  std::vector<double> cs, sn;  // cos / sin (2 pi j / n), j < n
};
typedef fftw_plan_s* fftw_plan;

inline fftw_plan dfpca_shim_make_plan(int n) {
  auto* p = new fftw_plan_s;
  p->n = n;
  p->cs.resize(static_cast<std::size_t>(n));
  p->sn.resize(static_cast<std::size_t>(n));
  const double two_pi = 6.283185307179586476925286766559;
  for (int j = 0; j < n; ++j) {
    p->cs[static_cast<std::size_t>(j)] = std::cos(two_pi * j / n);
    p->sn[static_cast<std::size_t>(j)] = std::sin(two_pi * j / n);
  }
  return p;
}

inline fftw_plan fftw_plan_dft_r2c_1d(int n, double*, fftw_complex*, unsigned) {
  return dfpca_shim_make_plan(n);
}
inline fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex*, double*, unsigned) {
  return dfpca_shim_make_plan(n);
}
inline void fftw_destroy_plan(fftw_plan p) { delete p; }

inline void fftw_execute_dft_r2c(fftw_plan p, double* in, fftw_complex* out) {
  const int n = p->n;
  for (int k = 0; k <= n / 2; ++k) {
    double re = 0.0, im = 0.0;
    for (int j = 0; j < n; ++j) {
      const std::size_t t = static_cast<std::size_t>((static_cast<long long>(j) * k) % n);
      re += in[j] * p->cs[t];
      im -= in[j] * p->sn[t];
    }
    out[k][0] = re;
    out[k][1] = im;
  }
}

inline void fftw_execute_dft_c2r(fftw_plan p, fftw_complex* in, double* out) {
  const int n = p->n;
  for (int j = 0; j < n; ++j) {
    double acc = in[0][0];
    for (int k = 1; k < (n + 1) / 2; ++k) {
      const std::size_t t = static_cast<std::size_t>((static_cast<long long>(j) * k) % n);
      acc += 2.0 * (in[k][0] * p->cs[t] - in[k][1] * p->sn[t]);
    }
    if (n % 2 == 0) acc += in[n / 2][0] * ((j % 2 == 0) ? 1.0 : -1.0);
    out[j] = acc;
  }
}
