// Drop-in matrixization and random-projection eigensolver (reference
// eigensolve.hpp: matrixize, default_sketch_size, randomized_eig,
// select_components_fve, eig_residuals, EigenSystem) running on the GPU: the
// sketch, range capture (DMMA products), Cholesky QR (Householder QR for
// ill-conditioned sketches), Rayleigh-Ritz projection, the small symmetric
// eigensolve (tridiagonalization, bisection, inverse iteration), lift and
// Riemann MGS all happen on the device (dfpca_randomized_eig), on the
// device-resident covariance when the surface came from fft_covariance.
// dense_eig (the LAPACK comparator, also the pipeline's default) runs the
// library's own device eigensolver (dfpca_dense_eig: Householder
// tridiagonalization, Sturm bisection, inverse iteration, back-transform).
//
// MatrixizedCovariance::dense_matrix / apply use Eigen::MatrixXd when Eigen is
// available (as in the reference) and a small column-major dfpca::DenseMatrix
// otherwise.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "dfpca/errors.hpp"
#include "dfpca/gpu.hpp"
#include "dfpca/grid.hpp"
#include "dfpca/surface.hpp"

#if defined(DFPCA_USE_EIGEN) && __has_include(<Eigen/Dense>)
#include <Eigen/Dense>
namespace dfpca {
using DenseMatrix = Eigen::MatrixXd;
}
#else
namespace dfpca {
/// Column-major dense matrix with the Eigen calls the eigensolve API needs.
class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(Index r, Index c) : r_(r), c_(c), a_(static_cast<std::size_t>(r * c), 0.0) {}
  void resize(Index r, Index c) {
    r_ = r;
    c_ = c;
    a_.assign(static_cast<std::size_t>(r * c), 0.0);
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double& operator()(Index i, Index j) { return a_[static_cast<std::size_t>(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return a_[static_cast<std::size_t>(j * r_ + i)]; }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> a_;
};
}  // namespace dfpca
#endif

namespace dfpca {

struct MatrixizedCovariance {
  static constexpr std::size_t kDenseBudget = 2ull << 30;
  static constexpr std::size_t kSlabBytes = 64ull << 20;

  const SurfaceEstimate* cov = nullptr;
  Index m = 0;
  std::vector<Index> node_of_row;
  std::vector<Index> row_of_node;  // -1 for masked-out nodes
  bool dense = false;
  DenseMatrix dense_matrix;

  /// Sigma * V (host product; the eigensolver itself never calls this).
  DenseMatrix apply(const DenseMatrix& V) const {
    if (V.rows() != m) throw err::invalid_argument("provider input has wrong row count");
    const auto g = static_cast<std::size_t>(cov->grid.size());
    DenseMatrix out(m, V.cols());
    for (Index i = 0; i < m; ++i) {
      const double* row = cov->values.data() + static_cast<std::size_t>(node_of_row[static_cast<std::size_t>(i)]) * g;
      for (Index c = 0; c < V.cols(); ++c) {
        double s = 0.0;
        for (Index j = 0; j < m; ++j) s += row[node_of_row[static_cast<std::size_t>(j)]] * V(j, c);
        out(i, c) = s;
      }
    }
    return out;
  }
};

inline MatrixizedCovariance matrixize(const SurfaceEstimate& cov,
                                      std::size_t dense_budget = MatrixizedCovariance::kDenseBudget) {
  if (cov.kind != SurfaceKind::Covariance) throw err::invalid_argument("matrixize expects a covariance surface");
  const auto g = static_cast<std::size_t>(cov.grid.size());
  if (cov.values.size() != g * g) throw err::invalid_argument("covariance surface has wrong length");
  MatrixizedCovariance out;
  out.cov = &cov;
  out.row_of_node.assign(g, -1);
  for (std::size_t f = 0; f < g; ++f)
    if (cov.grid.in_mask(static_cast<Index>(f))) {
      out.row_of_node[f] = out.m++;
      out.node_of_row.push_back(static_cast<Index>(f));
    }
  if (out.m == 0) throw err::invalid_argument("no in-mask nodes to decompose");
  out.dense = static_cast<std::size_t>(out.m) * static_cast<std::size_t>(out.m) * sizeof(double) <= dense_budget;
  if (out.dense) {
    out.dense_matrix.resize(out.m, out.m);
    for (Index i = 0; i < out.m; ++i)
      for (Index j = 0; j < out.m; ++j)
        out.dense_matrix(i, j) = cov.values[static_cast<std::size_t>(out.node_of_row[static_cast<std::size_t>(i)]) * g +
                                            static_cast<std::size_t>(out.node_of_row[static_cast<std::size_t>(j)])];
  }
  return out;
}

struct EigenSystem {
  std::vector<double> eigenvalues;                  // positive, descending
  std::vector<std::vector<double>> eigenfunctions;  // full-grid surfaces
  std::vector<double> fve;                          // cumulative FVE
  double total_variance = 0.0;
};

inline std::size_t default_sketch_size(std::size_t L_max, Index m) {
  return std::min(std::max<std::size_t>(2 * L_max + 10, 99), static_cast<std::size_t>(m));
}

namespace gpu {
/// Device copy of a covariance surface (the one fft_covariance left, or an upload).
inline dfpca_surface* device_surface(const SurfaceEstimate& s) {
  if (s.device) return s.device.get();
  GridDesc gd(s.grid);
  dfpca_surface* h = nullptr;
  check(dfpca_surface_upload(context(), gd.get(), DFPCA_SURFACE_COVARIANCE, s.values.data(),
                             static_cast<int64_t>(s.values.size()), &h));
  const_cast<SurfaceEstimate&>(s).device.reset(h, SurfaceDeleter{});
  return h;
}
}  // namespace gpu

/// dense_eig (eigensolve.hpp:205-228): full symmetric eigendecomposition on
/// the GPU (cuSOLVER syevd) followed by the reference's finalization.
inline EigenSystem dense_eig(const MatrixizedCovariance& S, std::size_t L_max, const EvaluationGrid& grid) {
  if (!S.dense)
    throw err::invalid_argument("dense eigendecomposition needs the dense provider; "
                                "the matrix exceeded the memory budget");
  const auto G = static_cast<std::size_t>(grid.size());
  const std::size_t cap = std::max<std::size_t>(L_max, 1);
  std::vector<double> ev(cap), ef(cap * G), fve(cap);
  double total = 0.0;
  int64_t n = 0;
  gpu::GridDesc gd(grid);
  gpu::check(dfpca_dense_eig(gpu::context(), gpu::device_surface(*S.cov), gd.get(), static_cast<int64_t>(L_max),
                             ev.data(), ef.data(), fve.data(), &total, &n));
  EigenSystem out;
  out.total_variance = total;
  for (int64_t l = 0; l < n; ++l) {
    out.eigenvalues.push_back(ev[static_cast<std::size_t>(l)]);
    out.fve.push_back(fve[static_cast<std::size_t>(l)]);
    out.eigenfunctions.emplace_back(ef.begin() + l * static_cast<int64_t>(G), ef.begin() + (l + 1) * static_cast<int64_t>(G));
  }
  return out;
}

inline EigenSystem randomized_eig(const MatrixizedCovariance& S, std::size_t q, std::size_t L_max,
                                  const EvaluationGrid& grid, std::uint64_t seed) {
  if (q < L_max)
    throw err::sketch_too_small("sketch size " + std::to_string(q) + " is below the requested component count " +
                                std::to_string(L_max));
  const auto G = static_cast<std::size_t>(grid.size());
  const std::size_t cap = std::max<std::size_t>(L_max, 1);
  std::vector<double> ev(cap), ef(cap * G), fve(cap);
  double total = 0.0;
  int64_t n = 0;
  gpu::GridDesc gd(grid);
  gpu::check(dfpca_randomized_eig(gpu::context(), gpu::device_surface(*S.cov), gd.get(), static_cast<int64_t>(q),
                                  static_cast<int64_t>(L_max), seed, ev.data(), ef.data(), fve.data(), &total, &n));
  EigenSystem out;
  out.total_variance = total;
  for (int64_t l = 0; l < n; ++l) {
    out.eigenvalues.push_back(ev[static_cast<std::size_t>(l)]);
    out.fve.push_back(fve[static_cast<std::size_t>(l)]);
    out.eigenfunctions.emplace_back(ef.begin() + l * static_cast<int64_t>(G), ef.begin() + (l + 1) * static_cast<int64_t>(G));
  }
  return out;
}

inline std::size_t select_components_fve(const EigenSystem& eig, double threshold) {
  if (!(threshold > 0.0) || threshold > 1.0) throw err::invalid_argument("FVE threshold must lie in (0, 1]");
  for (std::size_t l = 0; l < eig.fve.size(); ++l)
    if (eig.fve[l] >= threshold - 1e-12) return l + 1;
  return eig.eigenvalues.size();
}

inline std::vector<double> eig_residuals(const MatrixizedCovariance& S, const EigenSystem& eig,
                                         const EvaluationGrid& grid) {
  const std::size_t L = eig.eigenvalues.size();
  if (L == 0) return {};
  std::vector<double> flat;
  for (const auto& f : eig.eigenfunctions) flat.insert(flat.end(), f.begin(), f.end());
  std::vector<double> out(L);
  gpu::GridDesc gd(grid);
  gpu::check(dfpca_eig_residuals(gpu::context(), gpu::device_surface(*S.cov), gd.get(), static_cast<int64_t>(L),
                                 eig.eigenvalues.data(), flat.data(), out.data()));
  return out;
}

}  // namespace dfpca
