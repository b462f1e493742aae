// Run-time binding of LAPACK for the oracle build (TEST INFRASTRUCTURE ONLY):
// dsyevd from scipy's bundled OpenBLAS, whose exported names carry a scipy_
// prefix.  Used by dense_eig (through lapacke.h) and by the Eigen shim's
// SelfAdjointEigenSolver.
#include <dlfcn.h>

#include <stdexcept>
#include <string>

#include "lapacke.h"

#ifndef DFPCA_OPENBLAS_PATH
#error "build with -DDFPCA_OPENBLAS_PATH=\"/path/to/libscipy_openblas.so\""
#endif

namespace {
using lapacke_dsyevd_t = lapack_int (*)(int, char, char, lapack_int, double*, lapack_int, double*);

lapacke_dsyevd_t resolve() {
  static lapacke_dsyevd_t fn = [] {
    void* h = dlopen(DFPCA_OPENBLAS_PATH, RTLD_NOW | RTLD_LOCAL);
    if (!h) throw std::runtime_error(std::string("oracle: cannot load LAPACK: ") + dlerror());
    void* s = dlsym(h, "scipy_LAPACKE_dsyevd");
    if (!s) throw std::runtime_error("oracle: scipy_LAPACKE_dsyevd missing");
    return reinterpret_cast<lapacke_dsyevd_t>(s);
  }();
  return fn;
}
}  // namespace

lapack_int LAPACKE_dsyevd(int layout, char jobz, char uplo, lapack_int n, double* a, lapack_int lda,
                          double* w) {
  return resolve()(layout, jobz, uplo, n, a, lda, w);
}

namespace Eigen {
namespace shim {
int syevd(int n, double* a, double* w) {
  if (n == 0) return 0;
  return static_cast<int>(resolve()(LAPACK_COL_MAJOR, 'V', 'L', n, a, n, w));
}
}  // namespace shim
}  // namespace Eigen
