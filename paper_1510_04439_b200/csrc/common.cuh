// Device-side helpers shared by the kernels of libdfpca_cuda.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>

#include "internal.hpp"

namespace dfpca_gpu {

constexpr int kMaxDim = DFPCA_MAX_DIM;       // data dimension d
constexpr int kMaxDim2 = 2 * DFPCA_MAX_DIM;  // product-grid dimension 2d

// Grid geometry passed by value to kernels.
struct DevGrid {
  int d;
  i64 shape[kMaxDim];
  i64 strides[kMaxDim];
  const double* axes[kMaxDim];  // device pointers
};

// Launch bookkeeping: every kernel launch goes through this so the context
// can report how many of its own kernels ran (bench.py "gpu_launches").
// With profiling enabled (dfpca_profile_enable) each launch is bracketed by
// CUDA events on the launching stream and attributed to the kernel's name.
// Every launch is a programmatic dependent launch (below): each kernel of
// the library begins with pdl_wait().
#define DFPCA_LAUNCH(ctx, kernel, grid, block, smem, ...) DFPCA_LAUNCH_PDL(ctx, kernel, grid, block, smem, __VA_ARGS__)

// Programmatic dependent launch (PDL): the kernel may be scheduled while the
// previous kernel on the stream drains (its launch latency and rasterization
// overlap that kernel's tail).  Every kernel launched this way calls
// pdl_wait() first, which blocks until the previous grid has completed and
// its memory is visible -- so ordering is exactly that of a plain launch.
// DFPCA_PDL=0 turns the attribute off (A/B).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("DFPCA_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

#define DFPCA_LAUNCH_PDL(ctx, kernel, grid, block, smem, ...)                                     \
  do {                                                                                           \
    const int dfpca_prof_slot_ = (ctx)->profile ? (ctx)->kernel_begin(#kernel) : -1;            \
    cudaLaunchConfig_t dfpca_cfg_{};                                                             \
    dfpca_cfg_.gridDim = dim3(grid);                                                             \
    dfpca_cfg_.blockDim = dim3(block);                                                           \
    dfpca_cfg_.dynamicSmemBytes = (smem);                                                        \
    dfpca_cfg_.stream = (ctx)->stream;                                                           \
    cudaLaunchAttribute dfpca_attr_[1];                                                          \
    dfpca_attr_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                      \
    dfpca_attr_[0].val.programmaticStreamSerializationAllowed = ::dfpca_gpu::pdl_enabled() ? 1 : 0; \
    dfpca_cfg_.attrs = dfpca_attr_;                                                              \
    dfpca_cfg_.numAttrs = 1;                                                                     \
    ::dfpca_gpu::cuda_check(cudaLaunchKernelEx(&dfpca_cfg_, kernel, __VA_ARGS__), #kernel);      \
    if (dfpca_prof_slot_ >= 0) (ctx)->kernel_end(dfpca_prof_slot_);                              \
    ++(ctx)->launches;                                                                           \
  } while (0)

// Raises (never lowers) a kernel's dynamic shared-memory limit.  The
// attribute is process-wide, so ranks running as threads of one process
// (shard.cu) must not race a smaller value in between another rank's
// attribute call and launch.
template <class K>
inline void allow_smem(K kern, std::size_t bytes) {
  static std::mutex mu;
  static std::map<const void*, std::size_t> cur;
  std::lock_guard<std::mutex> lk(mu);
  std::size_t& c = cur[reinterpret_cast<const void*>(kern)];
  if (bytes > c) {
    DFPCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    c = bytes;
  }
}

inline unsigned grid_for(i64 n, int block, i64 cap = 148ll * 32) {
  i64 g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// Reference kernel_axis (kernel.hpp:37-43) evaluated on the host when taps
// are built; device code uses the same expression order.
__host__ __device__ inline double kernel_axis_value(double u, double h) {
  const double z = u / h;
  const double t = 1.0 - z * z;
  return t > 0.0 ? 0.75 * t / h : 0.0;
}

}  // namespace dfpca_gpu
