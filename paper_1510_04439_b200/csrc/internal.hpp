// Host-side internals of libdfpca_cuda.so: error plumbing, device buffers,
// the grid descriptor, the context and the device-resident handles.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "dfpca_cuda.h"

namespace dfpca_gpu {

using i64 = std::int64_t;
class Transport;  // shard.cu: NCCL (or in-process) rank exchanges
void host_mark(const char* what);  // DFPCA_HOST_TRACE: a host timestamp on stderr

// Error classes of the reference (errors.hpp:11-17).
enum : int { kParse = 2, kConfig = 3, kNumeric = 4, kVersion = 5 };

struct Failure {
  int cls = 0;
  std::string name;
  std::string msg;
  i64 sample = -1;
  i64 obs = -1;
};

[[noreturn]] void fail(int cls, const char* name, const std::string& msg);
[[noreturn]] void fail_at(int cls, const char* name, const std::string& msg, i64 sample, i64 obs);
void cuda_check(cudaError_t e, const char* what);

#define DFPCA_CUDA(call) ::dfpca_gpu::cuda_check((call), #call)

// Stream the current API call runs on; device buffers are allocated
// stream-ordered on it (cudaMallocAsync from the device's default pool, whose
// release threshold is raised at context creation so blocks are cached) and
// freed on the same stream, also when a handle is released outside any call
// (dfpca_*_free), so the pool can hand the block to the next call at once.
extern thread_local cudaStream_t g_alloc_stream;

// Move-only owning device array.
template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(std::size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p_ = o.p_; n_ = o.n_; s_ = o.s_; o.p_ = nullptr; o.n_ = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(std::size_t n) {
    if (n == n_ && p_) return;
    release();
    if (n == 0) return;
    DFPCA_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), g_alloc_stream));
    n_ = n;
    s_ = g_alloc_stream;
  }
  void release() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  std::size_t bytes() const { return n_ * sizeof(T); }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
  cudaStream_t s_ = nullptr;  // allocation stream, reused for the free
};

// Validated copy of an EvaluationGrid (grid.hpp:92-230).
struct Grid {
  int d = 0;
  i64 shape[DFPCA_MAX_DIM] = {0, 0, 0};
  i64 strides[DFPCA_MAX_DIM] = {0, 0, 0};
  i64 G = 0;
  std::vector<double> axes[DFPCA_MAX_DIM];
  double spacing[DFPCA_MAX_DIM] = {0, 0, 0};
  bool equispaced = false;
  bool has_mask = false;
  std::vector<std::uint8_t> mask;
  i64 in_mask_count = 0;

  bool same_shape(const Grid& o) const {
    if (d != o.d) return false;
    for (int k = 0; k < d; ++k)
      if (shape[k] != o.shape[k]) return false;
    return true;
  }
  double hull_lo(int k) const { return axes[k].front(); }
  double hull_hi(int k) const { return axes[k].back(); }
  double cell_volume() const {
    double v = 1.0;
    for (int k = 0; k < d; ++k) v *= spacing[k];
    return v;
  }
};

Grid make_grid(const dfpca_grid* g);

class Context;

// Stage timer: CUDA events on the context stream, collected at sync points.
struct StageMark {
  std::string name;
  cudaEvent_t start = nullptr;
  cudaEvent_t stop = nullptr;
};

}  // namespace dfpca_gpu

// ---- opaque handles --------------------------------------------------------

struct dfpca_context {
  // Serialises API calls on this context: the reference's functions are
  // reentrant, so several host threads may share one context (the C++
  // drop-in's process-wide context, include/dfpca/gpu.hpp); each call holds
  // the lock for its whole run (scratch, caches, stage timers, stream).
  std::recursive_mutex api_mu;
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  dfpca_gpu::Failure err;
  std::map<std::string, double> stage_ms;
  std::vector<dfpca_gpu::StageMark> marks;
  std::vector<cudaEvent_t> event_pool;  // timing events reused across calls (stage / kernel marks)
  cudaEvent_t take_event() {
    if (event_pool.empty()) {
      cudaEvent_t e = nullptr;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  void give_event(cudaEvent_t e) {
    if (e) event_pool.push_back(e);
  }
  std::int64_t launches = 0;
  // multi-GPU (dfpca_nccl_init): this process's rank of a sharded covariance
  std::shared_ptr<dfpca_gpu::Transport> transport;

  // Device tables that depend only on the grid and bandwidth (smooth.cu),
  // built on first use.
  std::map<std::string, std::unique_ptr<dfpca_gpu::DevBuf<double>>> table_cache;
  // Second stream for host-to-device copies that overlap compute (binning
  // chunks), and a reusable event to order it after the context stream.
  cudaStream_t copy_ = nullptr;
  cudaEvent_t fence_ = nullptr;
  cudaStream_t copy_stream() {
    if (!copy_) cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking);
    return copy_;
  }
  cudaEvent_t fence() {
    if (!fence_) cudaEventCreateWithFlags(&fence_, cudaEventDisableTiming);
    return fence_;
  }
  // Second compute stream (binning counts of later chunks) and a small
  // pinned host array for asynchronous scalar read-backs, zeroed on request.
  cudaStream_t aux_ = nullptr;
  cudaStream_t aux_stream() {
    if (!aux_) cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking);
    return aux_;
  }
  unsigned long long* pinned_ = nullptr;
  std::size_t pinned_n_ = 0;
  unsigned long long* pinned_u64(std::size_t n) {
    if (n > pinned_n_) {
      if (pinned_) cudaFreeHost(pinned_);
      pinned_ = nullptr;
      pinned_n_ = 0;
      if (cudaHostAlloc(reinterpret_cast<void**>(&pinned_), n * sizeof(unsigned long long), cudaHostAllocDefault) ==
          cudaSuccess)
        pinned_n_ = n;
    }
    if (!pinned_) throw std::bad_alloc();
    for (std::size_t i = 0; i < n; ++i) pinned_[i] = 0;
    return pinned_;
  }
  // Pinned upload slots, worker streams and events of the table reader
  // (longfmt.cu), created on first use.
  std::shared_ptr<void> io_state;
  // Reusable scratch (grown on demand, never shrunk while the context lives).
  dfpca_gpu::DevBuf<unsigned char> scratch;
  unsigned char* scratch_bytes(std::size_t n) {
    if (scratch.size() < n) scratch.alloc(n);
    return scratch.get();
  }

  void begin_stage(const std::string& name);
  void end_stage();
  void collect_stages();  // after a stream sync

  // Per-kernel device timing (profiling mode).
  struct KernelStat {
    double ms = 0.0;
    std::int64_t count = 0;
  };
  bool profile = false;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> kernel_marks;
  std::map<std::string, KernelStat> kernel_stats;
  int kernel_begin(const char* name);
  void kernel_end(int slot);
};

struct dfpca_binned {
  dfpca_gpu::Grid grid;
  std::int64_t n_samples = 0;
  std::int64_t n_pair = 0;
  std::int64_t codes = 1;  // 3^d
  bool has_mean = false;
  bool has_cov = false;
  // Structure flags computed at binning time.
  bool identical_mass = false;  // every per-sample mass grid bitwise equal
  // Shared constant design: identical masses, M(s) == shared_m0 > 0 at every
  // node, and a diagonal-only mass band equal to shared_dm0 at every node (the
  // GridNodes design: every subject observed once at every node).  Then
  // pw(u,v) = sw - shared_dm0 [u == v] exactly as the reference builds it,
  // with sw the ordered sum of (w_i M0) M0 (see smooth.cu, run_covariance).
  bool shared_const = false;
  double shared_m0 = 0.0, shared_dm0 = 0.0;

  dfpca_gpu::DevBuf<double> mass, wvalue, wsquare;  // G
  dfpca_gpu::DevBuf<double> ps_mass, ps_value;      // n_pair * G
  dfpca_gpu::DevBuf<double> pair_weight;            // n_pair
  dfpca_gpu::DevBuf<double> diag_mass, diag_value;  // G * codes
  std::vector<std::int64_t> sample_index;           // n_pair
  std::vector<double> pair_weight_h;                // n_pair
  std::vector<std::int64_t> sample_sizes;           // n_samples
  // pair-grid route (pairs.cu), decided on first use: -1 unknown, 0 SYRK,
  // 1 sparse records; pair_nnz = nonzeros of every per-sample mass grid
  mutable int pair_route = -1;
  mutable std::vector<std::int64_t> pair_nnz;
};

namespace dfpca_gpu {
// Sets identical_mass-derived structure flags (shared_const, shared_m0/dm0).
void detect_shared_design(dfpca_context* ctx, dfpca_binned* b);
// Host <-> device copies of caller buffers (longfmt.cu): pinned memory is
// copied directly, large pageable buffers through the pinned slots on host
// worker threads.  copy_h2d is ordered before later work on ctx->stream;
// copy_d2h returns when the bytes are in `dst`.
bool copy_is_staged(const void* host, std::int64_t bytes);
void copy_h2d(dfpca_context* ctx, void* d_dst, const void* src, std::int64_t bytes);
void copy_d2h(dfpca_context* ctx, void* dst, const void* d_src, std::int64_t bytes);
}  // namespace dfpca_gpu

struct dfpca_surface {
  dfpca_gpu::Grid grid;
  int kind = DFPCA_SURFACE_MEAN;
  std::int64_t n = 0;
  dfpca_gpu::DevBuf<double> values;
  // covariance slab of a sharded run (shard.hpp): values hold global rows
  // [row0, row0 + rows) of the G x G covariance; rows = G when unsharded
  std::int64_t row0 = 0;
  std::int64_t rows = -1;
};

// Device-resident observations of a FunctionalDataset (CSR), for the CV
// objective (cv.cu): host copies give the units' targets and responses.
struct dfpca_dataset {
  int dim = 0;
  std::int64_t n_samples = 0, n_obs = 0;
  std::vector<std::int64_t> offsets_h;
  std::vector<double> coords_h, values_h;
  dfpca_gpu::DevBuf<std::int64_t> offsets;
  dfpca_gpu::DevBuf<double> coords, values, obs_w;
};

namespace dfpca_gpu {
// Backs the device pool up to `bytes` in one allocation when it holds less (capi.cu).
void pool_ensure(dfpca_context* ctx, std::uint64_t bytes);
}  // namespace dfpca_gpu
