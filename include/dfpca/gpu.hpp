// Host glue between the drop-in dfpca:: headers and the C-ABI of
// libdfpca_cuda.so (include/dfpca_cuda.h): one lazily created device context
// per process (device from DFPCA_DEVICE, default 0), grid descriptors, and the
// mapping of ABI status codes back to dfpca::Error.  Link with -ldfpca_cuda.
#pragma once

#include <cstdlib>
#include <memory>
#include <mutex>
#include <string>

#include "dfpca/errors.hpp"
#include "dfpca/grid.hpp"
#include "dfpca_cuda.h"

namespace dfpca {
namespace gpu {

inline int& device_ref() {
  static int dev = [] {
    const char* e = std::getenv("DFPCA_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  return dev;
}

/// Selects the CUDA device used by subsequent calls (before the first call).
inline void set_device(int device) { device_ref() = device; }

inline dfpca_context* context() {
  static std::once_flag once;
  static dfpca_context* ctx = nullptr;
  static int status = 0;
  std::call_once(once, [] { status = dfpca_context_create(device_ref(), &ctx); });
  if (status != 0 || !ctx)
    throw err::device_error("no CUDA device " + std::to_string(device_ref()) +
                            " for the GPU hot path (there is no CPU fallback)");
  return ctx;
}

/// Rethrows a nonzero ABI status as the reference's dfpca::Error.
inline void check(int status) {
  if (status == 0) return;
  int cls = 0;
  const char* name = nullptr;
  const char* msg = nullptr;
  dfpca_last_error(context(), &cls, &name, &msg);
  const auto ec = cls >= 1 && cls <= 5 ? static_cast<ErrorClass>(cls) : ErrorClass::Numeric;
  throw Error(ec, name ? name : "DeviceError", msg ? msg : "");
}

/// dfpca_grid view of an EvaluationGrid (the grid must outlive it).
struct GridDesc {
  dfpca_grid g{};
  explicit GridDesc(const EvaluationGrid& grid) {
    if (grid.dim() > DFPCA_MAX_DIM)
      throw err::invalid_argument("the GPU path supports grids of dimension <= " + std::to_string(DFPCA_MAX_DIM));
    g.dim = static_cast<int32_t>(grid.dim());
    for (std::size_t k = 0; k < grid.dim(); ++k) {
      g.shape[k] = grid.shape()[k];
      g.axes[k] = grid.axis(k).data();
    }
    g.mask = grid.has_mask() ? grid.mask()->data() : nullptr;
  }
  const dfpca_grid* get() const { return &g; }
};

struct BinnedDeleter {
  void operator()(dfpca_binned* b) const { dfpca_binned_free(b); }
};
struct SurfaceDeleter {
  void operator()(dfpca_surface* s) const { dfpca_surface_free(s); }
};

}  // namespace gpu
}  // namespace dfpca
