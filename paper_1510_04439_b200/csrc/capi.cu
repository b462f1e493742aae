// extern "C" entry points of libdfpca_cuda.so (include/dfpca_cuda.h):
// argument validation in the reference's order, error mapping to the
// reference's error names, handle management and stage timing.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <iterator>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"

namespace dfpca_gpu {

thread_local cudaStream_t g_alloc_stream = nullptr;

// out[i] = values[index[i] - lo]: entries of a device-resident surface
// (SurfaceEstimate::values[i] without downloading the G^2 array).
__global__ void k_gather_values(const double* __restrict__ values, i64 lo, const i64* __restrict__ index, i64 n,
                                double* __restrict__ out) {
  pdl_wait();
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    out[i] = values[index[i] - lo];
}

void gather_values(dfpca_context* ctx, const double* values, i64 lo, const i64* index, i64 n, double* out) {
  DFPCA_LAUNCH(ctx, k_gather_values, grid_for(n, 256), 256, 0, values, lo, index, n, out);
}

dfpca_binned* run_linear_bin(dfpca_context* ctx, const Grid& grid, i64 n_samples,
                             const i64* obs_offsets, const double* coords, const double* values,
                             bool mean_path, bool cov_path, bool device_inputs = false);
void run_local_linear(dfpca_context* ctx, const dfpca_binned* b, const Grid& grid, const double* h,
                      int target, double* out_host, dfpca_surface** out_surface);
void run_covariance(dfpca_context* ctx, const dfpca_binned* b, const Grid& grid, const double* h,
                    const double* mean_host, dfpca_surface** out);
}  // namespace dfpca_gpu
#include "pairs.cuh"
#include "shard.hpp"
namespace dfpca_gpu {
void run_covariance_sharded(dfpca_context* ctx, Transport& tr, const dfpca_binned* b, const Grid& grid,
                            const double* h, const double* mean_host, dfpca_surface** out);
struct EigOut {
  i64 q = 0, L = 0;
  unsigned long long seed = 0;
  std::vector<double> values, functions, fve;
  double total = 0.0;
  i64 n = 0;
};
void run_covariance_emulated(dfpca_context* ctx, int world, const dfpca_binned* b, const Grid& grid,
                             const double* h, const double* mean_host, dfpca_surface** out,
                             std::vector<EigOut>* eig);
void nccl_unique_id(void* out);
void run_covariance_dryrun(dfpca_context* ctx, int world, int rank, const dfpca_binned* b, const Grid& grid,
                           const double* h, const double* mean_host, dfpca_surface** out);
std::shared_ptr<Transport> make_nccl_transport(int world, int rank, const void* id);
i64 nccl_selftest(dfpca_context* ctx);
dfpca_dataset* upload_dataset(dfpca_context* ctx, int dim, i64 n, const i64* offsets, const double* coords,
                              const double* values);
std::vector<i64> cv_units(i64 n_samples, const i64* offsets, int target, i64 max_units, std::uint64_t seed);
double run_cv_objective(dfpca_context* ctx, const dfpca_dataset* ds, int target, i64 n_units, const i64* units,
                        const double* h, i64* used_out);
dfpca_table* read_long_format_file(dfpca_context* ctx, const char* path);
dfpca_table* parse_long_format_bytes(dfpca_context* ctx, const char* name, const char* bytes, i64 S);
void table_copy(dfpca_context* ctx, const dfpca_table* t, i64* offsets, double* coords, double* values, i64* id_off,
                char* id_chars);
void table_shape(const dfpca_table* t, int* dim, i64* n_samples, i64* n_obs, i64* id_bytes);
void table_delete(dfpca_table* t);
dfpca_binned* bin_table(dfpca_context* ctx, const dfpca_table* t, const Grid& grid, bool mean_path, bool cov_path);
void run_estimate_sigma2(dfpca_context* ctx, const Grid& grid, const double* diag_plus_noise,
                         const dfpca_surface* cov, const double* mean, double* sigma2);
void run_scores(dfpca_context* ctx, const Grid& grid, i64 n, const i64* offsets, const double* coords,
                const double* values, const double* mean, i64 L, const double* eigenvalues,
                const double* eigenfunctions, double sigma2, int method, double* scores, int* sparse_warning,
                i64* bad_sample);
void run_reconstruct(dfpca_context* ctx, const Grid& grid, const double* mean, i64 L, const double* eigenfunctions,
                     i64 n, const double* scores, double* out);
void run_randomized_eig(dfpca_context* ctx, const dfpca_surface* cov, const Grid& grid, i64 q,
                        i64 L_max, unsigned long long seed, double* eigenvalues, double* eigenfunctions,
                        double* fve, double* total_variance, i64* n_components);
void run_eig_residuals(dfpca_context* ctx, const dfpca_surface* cov, const Grid& grid, i64 L,
                       const double* eigenvalues, const double* eigenfunctions, double* residuals);
void run_dense_eig(dfpca_context* ctx, const dfpca_surface* cov, const Grid& grid, i64 L_max, double* eigenvalues,
                   double* eigenfunctions, double* fve, double* total_variance, i64* n_components);

void fail(int cls, const char* name, const std::string& msg) {
  Failure f;
  f.cls = cls;
  f.name = name;
  f.msg = msg;
  throw f;
}

void fail_at(int cls, const char* name, const std::string& msg, i64 sample, i64 obs) {
  Failure f;
  f.cls = cls;
  f.name = name;
  f.msg = msg;
  f.sample = sample;
  f.obs = obs;
  throw f;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  fail(kNumeric, "DeviceError", std::string(what) + ": " + cudaGetErrorString(e));
}

// EvaluationGrid invariants (grid.hpp:99-126): >= 1 axis, >= 2 nodes per
// axis, strictly increasing, mask size; spacing = mean gap; equispaced when
// every gap is within 1e-9 of it.
Grid make_grid(const dfpca_grid* g) {
  if (!g) fail(kConfig, "InvalidArgument", "grid descriptor is null");
  if (g->dim < 1) fail(kConfig, "InvalidArgument", "grid needs at least one axis");
  if (g->dim > DFPCA_MAX_DIM)
    fail(kConfig, "InvalidArgument", "grid dimension above " + std::to_string(DFPCA_MAX_DIM));
  Grid out;
  out.d = g->dim;
  for (int k = 0; k < out.d; ++k) {
    const i64 n = g->shape[k];
    if (n < 2) fail(kConfig, "InvalidArgument", "grid axis " + std::to_string(k) + " needs >= 2 nodes");
    out.axes[k].assign(g->axes[k], g->axes[k] + n);
    for (i64 j = 1; j < n; ++j)
      if (!(out.axes[k][j] > out.axes[k][j - 1]))
        fail(kConfig, "InvalidArgument", "grid axis " + std::to_string(k) + " is not strictly increasing");
    out.shape[k] = n;
  }
  out.strides[out.d - 1] = 1;
  for (int k = out.d - 2; k >= 0; --k) out.strides[k] = out.strides[k + 1] * out.shape[k + 1];
  out.G = out.strides[0] * out.shape[0];
  out.equispaced = true;
  for (int k = 0; k < out.d; ++k) {
    const auto& ax = out.axes[k];
    const double gap = (ax.back() - ax.front()) / static_cast<double>(ax.size() - 1);
    out.spacing[k] = gap;
    for (std::size_t j = 1; j < ax.size(); ++j)
      if (std::abs((ax[j] - ax[j - 1]) - gap) > 1e-9 * gap) {
        out.equispaced = false;
        break;
      }
  }
  out.has_mask = g->mask != nullptr;
  out.in_mask_count = out.G;
  if (out.has_mask) {
    out.mask.assign(g->mask, g->mask + out.G);
    out.in_mask_count = 0;
    for (auto m : out.mask) out.in_mask_count += (m != 0);
  }
  return out;
}

DevGrid upload_grid_axes(dfpca_context* ctx, const Grid& g, DevBuf<double>& storage) {
  i64 total = 0;
  for (int k = 0; k < g.d; ++k) total += g.shape[k];
  storage.alloc(static_cast<std::size_t>(total));
  std::vector<double> flat;
  flat.reserve(static_cast<std::size_t>(total));
  for (int k = 0; k < g.d; ++k) flat.insert(flat.end(), g.axes[k].begin(), g.axes[k].end());
  DFPCA_CUDA(cudaMemcpyAsync(storage.get(), flat.data(), sizeof(double) * total, cudaMemcpyHostToDevice,
                             ctx->stream));
  DevGrid dg{};
  dg.d = g.d;
  i64 off = 0;
  for (int k = 0; k < g.d; ++k) {
    dg.shape[k] = g.shape[k];
    dg.strides[k] = g.strides[k];
    dg.axes[k] = storage.get() + off;
    off += g.shape[k];
  }
  DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  return dg;
}

// Bandwidth::validate (dataset.hpp:86-103) against the grid hull.
void validate_bandwidth(const Grid& grid, const double* h) {
  if (!h) fail(kConfig, "InvalidBandwidth", "bandwidth dimension mismatch");
  for (int k = 0; k < grid.d; ++k) {
    const double ext = grid.hull_hi(k) - grid.hull_lo(k);
    if (!(h[k] > 0.0))
      fail(kConfig, "InvalidBandwidth", "bandwidth axis " + std::to_string(k) + " must be positive");
    if (h[k] > ext * (1.0 + 1e-12))
      fail(kConfig, "InvalidBandwidth", "bandwidth axis " + std::to_string(k) + " exceeds the axis extent");
  }
}

static i64 radius_nodes(double h, double spacing) { return static_cast<i64>(std::ceil(h / spacing)); }

// validate_block_plan (fft_smoother.hpp:101-145).
void validate_plan(const dfpca_plan* plan, const Grid& grid, const double* h) {
  if (!plan) return;  // single-block plan: valid by construction
  const int d = grid.d;
  if (plan->n_blocks <= 0 || !plan->halo)
    fail(kConfig, "InvalidArgument", "block plan does not match the grid dimension");
  for (int k = 0; k < d; ++k) {
    const i64 r = radius_nodes(h[k], grid.spacing[k]);
    if (plan->halo[k] < r)
      fail(kConfig, "HaloTooSmall",
           "halo of " + std::to_string(plan->halo[k]) + " node(s) on axis " + std::to_string(k) +
               " is below the kernel radius of " + std::to_string(r));
  }
  i64 covered = 0;
  std::vector<std::vector<i64>> lo(plan->n_blocks), hi(plan->n_blocks);
  for (i64 b = 0; b < plan->n_blocks; ++b) {
    const i64* blo = plan->blocks_lo + b * d;
    const i64* bhi = plan->blocks_hi + b * d;
    lo[b].resize(d);
    hi[b].resize(d);
    i64 vol = 1;
    for (int k = 0; k < d; ++k) {
      if (blo[k] < 0 || bhi[k] > grid.shape[k] || blo[k] >= bhi[k])
        fail(kConfig, "InvalidArgument", "block range outside the grid");
      i64 cl = blo[k], ch = bhi[k];
      if (cl > 0) cl += plan->halo[k];
      if (ch < grid.shape[k]) ch -= plan->halo[k];
      if (ch - cl < plan->halo[k])
        fail(kConfig, "BlockTooSmall",
             "block " + std::to_string(b) + " core extent " + std::to_string(ch - cl) + " on axis " +
                 std::to_string(k) + " is smaller than its halo of " + std::to_string(plan->halo[k]));
      lo[b][k] = cl;
      hi[b][k] = ch;
      vol *= (ch - cl);
    }
    covered += vol;
  }
  for (i64 a = 0; a < plan->n_blocks; ++a)
    for (i64 b = a + 1; b < plan->n_blocks; ++b) {
      bool separated = false;
      for (int k = 0; k < d; ++k)
        if (hi[a][k] <= lo[b][k] || hi[b][k] <= lo[a][k]) {
          separated = true;
          break;
        }
      if (!separated) fail(kConfig, "InvalidArgument", "block cores overlap");
    }
  if (covered != grid.G) fail(kConfig, "InvalidArgument", "block cores do not tile the grid exactly");
}

}  // namespace dfpca_gpu

using namespace dfpca_gpu;

// ---- context stage timing ---------------------------------------------------
namespace {
// DFPCA_HOST_TRACE=1: host wall-clock stamps at stage boundaries (stderr), to
// find host gaps between the device stages
double host_us() {
  static const auto t0 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
}
bool host_trace() {
  static const bool on = std::getenv("DFPCA_HOST_TRACE") != nullptr;
  return on;
}
}  // namespace

namespace dfpca_gpu {
void host_mark(const char* what) {
  if (host_trace()) std::fprintf(stderr, "[host %10.1f us] %s\n", host_us(), what);
}
}  // namespace dfpca_gpu

void dfpca_context::begin_stage(const std::string& name) {
  if (host_trace()) std::fprintf(stderr, "[host %10.1f us] begin %s\n", host_us(), name.c_str());
  StageMark m;
  m.name = name;
  m.start = take_event();
  m.stop = take_event();
  cudaEventRecord(m.start, stream);
  marks.push_back(m);
}
void dfpca_context::end_stage() {
  if (host_trace()) std::fprintf(stderr, "[host %10.1f us] end\n", host_us());
  for (auto it = marks.rbegin(); it != marks.rend(); ++it)
    if (it->stop && !it->name.empty() && it->name[0] != '#') {
      cudaEventRecord(it->stop, stream);
      it->name = "#" + it->name;  // closed
      return;
    }
}
int dfpca_context::kernel_begin(const char* name) {
  cudaEvent_t a = take_event(), b = take_event();
  cudaEventRecord(a, stream);
  std::string n(name);
  if (!n.empty() && n.front() == '(') n = n.substr(1);
  const auto p = n.find('<');  // strip template arguments for grouping
  kernel_marks.push_back({n.substr(0, p == std::string::npos ? n.size() : p), {a, b}});
  return static_cast<int>(kernel_marks.size()) - 1;
}
void dfpca_context::kernel_end(int slot) { cudaEventRecord(kernel_marks[static_cast<std::size_t>(slot)].second.second, stream); }

void dfpca_context::collect_stages() {
  cudaStreamSynchronize(stream);
  for (auto& km : kernel_marks) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, km.second.first, km.second.second) == cudaSuccess) {
      auto& st = kernel_stats[km.first];
      st.ms += ms;
      st.count += 1;
    }
    give_event(km.second.first);
    give_event(km.second.second);
  }
  kernel_marks.clear();
  for (auto& m : marks) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, m.start, m.stop) == cudaSuccess) {
      const std::string name = m.name[0] == '#' ? m.name.substr(1) : m.name;
      stage_ms[name] += ms;
    }
    give_event(m.start);
    give_event(m.stop);
  }
  marks.clear();
}

namespace {

// The failure of the calling thread's last call per context: dfpca_last_error
// reads it after the call has released the context lock, so another thread's
// call on the same context cannot clear or overwrite it in between.
thread_local std::map<const dfpca_context*, Failure> t_last_err;

int record(dfpca_context* ctx) {
  t_last_err[ctx] = ctx->err;
  return ctx->err.cls;
}

template <class F>
int guarded(dfpca_context* ctx, F&& f) {
  if (!ctx) return kConfig;
  std::lock_guard<std::recursive_mutex> lock(ctx->api_mu);
  ctx->err = Failure{};
  ctx->stage_ms.clear();
  struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
    ~StreamScope() { g_alloc_stream = prev; }
  } scope(ctx->stream);
  try {
    DFPCA_CUDA(cudaSetDevice(ctx->device));
    ctx->begin_stage("total");
    f();
    ctx->end_stage();
    ctx->collect_stages();
    return record(ctx);
  } catch (const Failure& e) {
    ctx->err = e;
  } catch (const std::bad_alloc&) {
    ctx->err = Failure{kNumeric, "DeviceError", "host allocation failed", -1, -1};
  } catch (const std::exception& e) {
    ctx->err = Failure{kNumeric, "DeviceError", e.what(), -1, -1};
  }
  // leave the stream usable for the next call
  cudaStreamSynchronize(ctx->stream);
  cudaGetLastError();
  for (auto& m : ctx->marks) {
    ctx->give_event(m.start);
    ctx->give_event(m.stop);
  }
  ctx->marks.clear();
  for (auto& km : ctx->kernel_marks) {
    ctx->give_event(km.second.first);
    ctx->give_event(km.second.second);
  }
  ctx->kernel_marks.clear();
  return record(ctx);
}

}  // namespace

// Blocks freed into a stream-ordered pool that already holds them are handed
// out again without mapping new pages: allocate `bytes` (at most 55 % of the
// free memory) and free it into the pool, whose release threshold keeps it.
bool pool_reserve(dfpca_context* ctx, std::uint64_t bytes) {
  std::size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return false;
  const std::size_t want = std::min<std::size_t>(static_cast<std::size_t>(bytes), static_cast<std::size_t>(0.55 * free_b));
  void* p = nullptr;
  bool ok = true;
  if (want > 0) {
    ok = cudaMallocAsync(&p, want, ctx->stream) == cudaSuccess;
    if (ok) cudaFreeAsync(p, ctx->stream);
    ok = cudaStreamSynchronize(ctx->stream) == cudaSuccess && ok;
  }
  cudaGetLastError();
  return ok;
}

namespace dfpca_gpu {
// Backs the pool up to `bytes` in one allocation when it holds less: a
// large call's first run then maps its memory at once instead of growing
// the pool block by block (cold start).
void pool_ensure(dfpca_context* ctx, std::uint64_t bytes) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) != cudaSuccess) return;
  std::uint64_t reserved = 0;
  if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) != cudaSuccess) return;
  if (reserved < bytes) pool_reserve(ctx, bytes);
}
}  // namespace dfpca_gpu

extern "C" {

int dfpca_context_create(int device, dfpca_context** out) {
  if (!out) return kConfig;
  *out = nullptr;
  // Module loading stays CUDA's default (lazy): EAGER would also load every
  // kernel of cuSOLVER at the first dense_eig (31.7 s cold for config 1,
  // against 90 ms lazy); lazy loading costs a few ms on each path's first call.
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0 || device < 0 || device >= n) return kNumeric;
  auto* ctx = new dfpca_context();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return kNumeric;
  }
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    std::uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    // Up-front backing of the pool (DFPCA_POOL_RESERVE_GB, default 16;
    // dfpca_context_reserve adds more later).  Without one the pool grows in
    // pieces and calls stall while it maps more (config-3 covariance 1.3 ms
    // warm, with stalls of 3-60 ms on calls whose allocations did not fit the
    // fragments); 16 GB (~0.2 s at creation, ~13 ms per GB) covers the d = 2
    // configurations, and 96 GB (+1.25 s) the d = 3 32^3 one.
    const char* e = std::getenv("DFPCA_POOL_RESERVE_GB");
    const double gb = e ? std::atof(e) : 16.0;
    if (gb > 0) pool_reserve(ctx, static_cast<std::uint64_t>(gb * (1ull << 30)));
  }
  *out = ctx;
  return 0;
}

int dfpca_context_reserve(dfpca_context* ctx, uint64_t bytes) {
  if (!ctx) return kConfig;
  cudaSetDevice(ctx->device);
  return pool_reserve(ctx, bytes) ? 0 : kNumeric;
}

int dfpca_context_destroy(dfpca_context* ctx) {
  if (!ctx) return 0;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  {
    g_alloc_stream = ctx->stream;
    ctx->scratch.release();
    ctx->table_cache.clear();
    cudaStreamSynchronize(ctx->stream);
    g_alloc_stream = nullptr;
  }
  if (ctx->copy_) {
    cudaStreamSynchronize(ctx->copy_);
    cudaStreamDestroy(ctx->copy_);
  }
  if (ctx->fence_) cudaEventDestroy(ctx->fence_);
  for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->aux_) {
    cudaStreamSynchronize(ctx->aux_);
    cudaStreamDestroy(ctx->aux_);
  }
  if (ctx->pinned_) cudaFreeHost(ctx->pinned_);
  ctx->io_state.reset();
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return 0;
}

int dfpca_last_error(const dfpca_context* ctx, int* error_class, const char** name, const char** message) {
  if (!ctx) return kConfig;
  const Failure& e = t_last_err[ctx];
  if (error_class) *error_class = e.cls;
  if (name) *name = e.name.c_str();
  if (message) *message = e.msg.c_str();
  return 0;
}

int dfpca_last_error_location(const dfpca_context* ctx, int64_t* sample, int64_t* obs) {
  if (!ctx) return kConfig;
  const Failure& e = t_last_err[ctx];
  if (sample) *sample = e.sample;
  if (obs) *obs = e.obs;
  return 0;
}

int dfpca_stage_time(const dfpca_context* ctx, const char* stage, double* ms) {
  if (!ctx || !stage || !ms) return kConfig;
  auto it = ctx->stage_ms.find(stage);
  *ms = it == ctx->stage_ms.end() ? 0.0 : it->second;
  return 0;
}

int64_t dfpca_kernel_launches(const dfpca_context* ctx) { return ctx ? ctx->launches : 0; }

int dfpca_profile_enable(dfpca_context* ctx, int on) {
  if (!ctx) return kConfig;
  ctx->profile = on != 0;
  ctx->kernel_stats.clear();
  return 0;
}

int dfpca_kernel_stat(const dfpca_context* ctx, int64_t index, const char** name, double* ms,
                      int64_t* count) {
  if (!ctx) return kConfig;
  if (index < 0 || index >= static_cast<int64_t>(ctx->kernel_stats.size())) return kConfig;
  auto it = ctx->kernel_stats.begin();
  std::advance(it, index);
  if (name) *name = it->first.c_str();
  if (ms) *ms = it->second.ms;
  if (count) *count = it->second.count;
  return 0;
}

int dfpca_host_register(void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return kConfig;
  return cudaHostRegister(ptr, static_cast<std::size_t>(bytes), cudaHostRegisterDefault) == cudaSuccess ? 0
                                                                                                           : kNumeric;
}

int dfpca_host_unregister(void* ptr) {
  if (!ptr) return kConfig;
  return cudaHostUnregister(ptr) == cudaSuccess ? 0 : kNumeric;
}

int dfpca_linear_bin(dfpca_context* ctx, const dfpca_grid* grid, int64_t n_samples,
                     const int64_t* obs_offsets, const double* coords, const double* values,
                     int mean_path, int covariance_path, dfpca_binned** out) {
  return guarded(ctx, [&] {
    if (!out) fail(kConfig, "InvalidArgument", "null output handle");
    *out = nullptr;
    Grid g = make_grid(grid);
    if (n_samples > 0 && !obs_offsets) fail(kConfig, "InvalidArgument", "null observation offsets");
    *out = run_linear_bin(ctx, g, n_samples, obs_offsets, coords, values, mean_path != 0,
                          covariance_path != 0);
  });
}

int dfpca_binned_info(const dfpca_binned* b, int64_t* n_samples, int64_t* n_pair_samples,
                      int64_t* grid_size, int64_t* offset_codes, int* has_mean_path,
                      int* has_covariance_path) {
  if (!b) return kConfig;
  if (n_samples) *n_samples = b->n_samples;
  if (n_pair_samples) *n_pair_samples = b->n_pair;
  if (grid_size) *grid_size = b->grid.G;
  if (offset_codes) *offset_codes = b->codes;
  if (has_mean_path) *has_mean_path = b->has_mean ? 1 : 0;
  if (has_covariance_path) *has_covariance_path = b->has_cov ? 1 : 0;
  return 0;
}

int dfpca_binned_download(dfpca_context* ctx, const dfpca_binned* b, double* mass, double* wvalue,
                          double* wsquare, int64_t* sample_index, double* pair_weight, double* ps_mass,
                          double* ps_value, double* diag_mass, double* diag_value, int64_t* sample_sizes) {
  return guarded(ctx, [&] {
    if (!b) fail(kConfig, "InvalidArgument", "null binned handle");
    cudaStream_t st = ctx->stream;
    const i64 G = b->grid.G;
    auto d2h = [&](double* dst, const DevBuf<double>& src, i64 n) {
      if (!dst || n <= 0 || !src.get()) return;
      if (copy_is_staged(dst, static_cast<i64>(sizeof(double)) * n))
        copy_d2h(ctx, dst, src.get(), static_cast<i64>(sizeof(double)) * n);
      else
        DFPCA_CUDA(cudaMemcpyAsync(dst, src.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    };
    if (b->has_mean) {
      d2h(mass, b->mass, G);
      d2h(wvalue, b->wvalue, G);
      d2h(wsquare, b->wsquare, G);
    }
    if (b->has_cov) {
      d2h(ps_mass, b->ps_mass, b->n_pair * G);
      d2h(ps_value, b->ps_value, b->n_pair * G);
      d2h(diag_mass, b->diag_mass, G * b->codes);
      d2h(diag_value, b->diag_value, G * b->codes);
      for (i64 i = 0; i < b->n_pair; ++i) {
        if (sample_index) sample_index[i] = b->sample_index[static_cast<std::size_t>(i)];
        if (pair_weight) pair_weight[i] = b->pair_weight_h[static_cast<std::size_t>(i)];
      }
    }
    if (sample_sizes)
      for (i64 i = 0; i < b->n_samples; ++i) sample_sizes[i] = b->sample_sizes[static_cast<std::size_t>(i)];
    DFPCA_CUDA(cudaStreamSynchronize(st));
  });
}

int dfpca_binned_upload(dfpca_context* ctx, const dfpca_grid* grid, int64_t n_samples,
                        const int64_t* sample_sizes, int has_mean_path, const double* mass,
                        const double* wvalue, const double* wsquare, int has_covariance_path,
                        int64_t n_pair_samples, const int64_t* sample_index, const double* pair_weight,
                        const double* ps_mass, const double* ps_value, const double* diag_mass,
                        const double* diag_value, dfpca_binned** out) {
  return guarded(ctx, [&] {
    if (!out) fail(kConfig, "InvalidArgument", "null output handle");
    *out = nullptr;
    Grid g = make_grid(grid);
    // argument validation up front: counts, and the arrays a count makes
    // mandatory (a NULL grid array of the mean path or a NULL band means
    // zeros; the per-sample bookkeeping must be given)
    if (n_samples < 0) fail(kConfig, "InvalidArgument", "negative sample count");
    if (has_covariance_path && n_pair_samples < 0) fail(kConfig, "InvalidArgument", "negative pair-sample count");
    if (n_samples > 0 && !sample_sizes) fail(kConfig, "InvalidArgument", "null sample_sizes");
    if (has_covariance_path && n_pair_samples > 0 && (!sample_index || !pair_weight))
      fail(kConfig, "InvalidArgument", "null sample_index or pair_weight");
    auto b = std::make_unique<dfpca_binned>();
    b->grid = g;
    b->n_samples = n_samples;
    b->has_mean = has_mean_path != 0;
    b->has_cov = has_covariance_path != 0;
    b->codes = 1;
    for (int k = 0; k < g.d; ++k) b->codes *= 3;
    if (sample_sizes) b->sample_sizes.assign(sample_sizes, sample_sizes + n_samples);
    cudaStream_t st = ctx->stream;
    const i64 G = g.G;
    auto h2d = [&](DevBuf<double>& dst, const double* src, i64 n) {
      dst.alloc(static_cast<std::size_t>(n));
      if (n == 0) return;
      if (src)
        copy_h2d(ctx, dst.get(), src, static_cast<i64>(sizeof(double)) * n);
      else
        DFPCA_CUDA(cudaMemsetAsync(dst.get(), 0, sizeof(double) * n, st));
    };
    if (b->has_mean) {
      h2d(b->mass, mass, G);
      h2d(b->wvalue, wvalue, G);
      h2d(b->wsquare, wsquare, G);
    }
    if (b->has_cov) {
      b->n_pair = n_pair_samples;
      h2d(b->ps_mass, ps_mass, n_pair_samples * G);
      h2d(b->ps_value, ps_value, n_pair_samples * G);
      h2d(b->pair_weight, pair_weight, n_pair_samples);
      h2d(b->diag_mass, diag_mass, G * b->codes);
      h2d(b->diag_value, diag_value, G * b->codes);
      b->sample_index.assign(sample_index, sample_index + n_pair_samples);
      b->pair_weight_h.assign(pair_weight, pair_weight + n_pair_samples);
      // structure flag: identical per-sample masses (host check on upload;
      // NULL masses are all zeros, hence identical)
      bool same = n_pair_samples >= 1;
      for (i64 i = 1; ps_mass && i < n_pair_samples && same; ++i)
        same = std::memcmp(ps_mass + i * G, ps_mass, sizeof(double) * G) == 0;
      b->identical_mass = same;
      dfpca_gpu::detect_shared_design(ctx, b.get());
    }
    DFPCA_CUDA(cudaStreamSynchronize(st));
    *out = b.release();
  });
}

int dfpca_binned_free(dfpca_binned* b) {
  delete b;
  return 0;
}

int dfpca_local_linear(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid, const double* h,
                       int target, const dfpca_plan* plan, double* out, dfpca_surface** out_surface) {
  return guarded(ctx, [&] {
    if (out_surface) *out_surface = nullptr;
    Grid g = make_grid(grid);
    // fft_smoother.hpp:502-507, in order
    if (!g.equispaced) fail(kConfig, "GridNotEquispaced", "binned smoothing requires equispaced grid axes");
    validate_bandwidth(g, h);
    if (!b || !b->has_mean) fail(kConfig, "InvalidArgument", "binned data lacks the mean path");
    if (!b->grid.same_shape(g)) fail(kConfig, "InvalidArgument", "binned data does not conform to the grid");
    validate_plan(plan, g, h);
    run_local_linear(ctx, b, g, h, target, out, out_surface);
  });
}

}  // extern "C"

namespace {
// fft_smoother.hpp:589-600, in order
Grid validate_covariance(const dfpca_binned* b, const dfpca_grid* grid, const double* h, const double* mean,
                         const dfpca_plan* plan, dfpca_surface** out) {
  if (!out) fail(kConfig, "InvalidArgument", "null output handle");
  *out = nullptr;
  Grid g = make_grid(grid);
  if (!g.equispaced)
    fail(kConfig, "GridNotEquispaced", "binned covariance smoothing requires equispaced grid axes");
  validate_bandwidth(g, h);
  if (!b || !b->has_cov) fail(kConfig, "InvalidArgument", "binned data lacks the covariance path");
  if (!b->grid.same_shape(g)) fail(kConfig, "InvalidArgument", "binned data does not conform to the grid");
  if (b->n_pair == 0)
    fail(kNumeric, "NoPairs", "covariance smoothing needs at least one sample with two observations");
  if (!mean) fail(kConfig, "InvalidArgument", "mean surface does not conform to the grid");
  validate_plan(plan, g, h);
  return g;
}
}  // namespace

extern "C" {

int dfpca_covariance(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid, const double* h,
                     const double* mean, const dfpca_plan* plan, dfpca_surface** out) {
  return guarded(ctx, [&] {
    Grid g = validate_covariance(b, grid, h, mean, plan, out);
    run_covariance(ctx, b, g, h, mean, out);
  });
}

int dfpca_nccl_unique_id(void* id) {
  if (!id) return kConfig;
  try {
    nccl_unique_id(id);
    return 0;
  } catch (const Failure& e) {
    return e.cls;
  }
}

int dfpca_nccl_selftest(dfpca_context* ctx, int64_t* mismatches) {
  return guarded(ctx, [&] {
    const i64 bad = nccl_selftest(ctx);
    if (mismatches) *mismatches = bad;
  });
}

int dfpca_nccl_init(dfpca_context* ctx, int world, int rank, const void* id) {
  return guarded(ctx, [&] {
    if (world < 1 || rank < 0 || rank >= world || !id) fail(kConfig, "InvalidArgument", "bad rank / world / id");
    ctx->transport.reset();
    if (world > 1) ctx->transport = make_nccl_transport(world, rank, id);
  });
}

int dfpca_covariance_sharded(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid, const double* h,
                             const double* mean, const dfpca_plan* plan, dfpca_surface** out) {
  return guarded(ctx, [&] {
    Grid g = validate_covariance(b, grid, h, mean, plan, out);
    if (!ctx->transport) {
      run_covariance(ctx, b, g, h, mean, out);  // one rank: the whole covariance
      return;
    }
    run_covariance_sharded(ctx, *ctx->transport, b, g, h, mean, out);
  });
}

int dfpca_covariance_emulated(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid, const double* h,
                              const double* mean, const dfpca_plan* plan, int world, dfpca_surface** out) {
  return guarded(ctx, [&] {
    Grid g = validate_covariance(b, grid, h, mean, plan, out);
    if (world < 1) fail(kConfig, "InvalidArgument", "world must be >= 1");
    run_covariance_emulated(ctx, world, b, g, h, mean, out, nullptr);
  });
}

int dfpca_fpca_emulated(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid, const double* h,
                        const double* mean, int world, int64_t q, int64_t L_max, uint64_t seed, double* eigenvalues,
                        double* eigenfunctions, double* fve, double* total_variance, int64_t* n_components,
                        int* ranks_agree) {
  return guarded(ctx, [&] {
    dfpca_surface* cov = nullptr;
    Grid g = validate_covariance(b, grid, h, mean, nullptr, &cov);
    if (world < 1) fail(kConfig, "InvalidArgument", "world must be >= 1");
    if (L_max < 0) fail(kConfig, "InvalidArgument", "L_max must be >= 0");
    std::vector<EigOut> eig(static_cast<std::size_t>(world));
    for (auto& e : eig) {
      e.q = q;
      e.L = L_max;
      e.seed = seed;
    }
    run_covariance_emulated(ctx, world, b, g, h, mean, &cov, &eig);
    std::unique_ptr<dfpca_surface> keep(cov);
    bool agree = true;
    for (const EigOut& e : eig) {
      agree = agree && e.n == eig[0].n && e.total == eig[0].total;
      agree = agree && std::memcmp(e.values.data(), eig[0].values.data(), sizeof(double) * e.values.size()) == 0;
      agree = agree && std::memcmp(e.functions.data(), eig[0].functions.data(),
                                   sizeof(double) * e.functions.size()) == 0;
    }
    if (ranks_agree) *ranks_agree = agree ? 1 : 0;
    const EigOut& e0 = eig[0];
    for (i64 l = 0; l < L_max; ++l) {
      if (eigenvalues) eigenvalues[l] = e0.values[static_cast<std::size_t>(l)];
      if (fve) fve[l] = e0.fve[static_cast<std::size_t>(l)];
    }
    if (eigenfunctions) std::memcpy(eigenfunctions, e0.functions.data(), sizeof(double) * e0.functions.size());
    if (total_variance) *total_variance = e0.total;
    if (n_components) *n_components = e0.n;
  });
}

int dfpca_covariance_slab_dryrun(dfpca_context* ctx, const dfpca_binned* b, const dfpca_grid* grid,
                                 const double* h, const double* mean, const dfpca_plan* plan, int world, int rank,
                                 dfpca_surface** out) {
  return guarded(ctx, [&] {
    Grid g = validate_covariance(b, grid, h, mean, plan, out);
    if (world < 1 || rank < 0 || rank >= world) fail(kConfig, "InvalidArgument", "bad rank / world");
    run_covariance_dryrun(ctx, world, rank, b, g, h, mean, out);
  });
}

int dfpca_estimate_sigma2(dfpca_context* ctx, const dfpca_grid* grid, const double* diag_plus_noise,
                          const dfpca_surface* cov, const double* mean, double* sigma2) {
  return guarded(ctx, [&] {
    if (!diag_plus_noise || !cov || !mean || !sigma2)
      fail(kConfig, "InvalidArgument", "estimate_sigma2 got surfaces of the wrong kind");
    Grid g = make_grid(grid);
    run_estimate_sigma2(ctx, g, diag_plus_noise, cov, mean, sigma2);
  });
}

int dfpca_scores(dfpca_context* ctx, const dfpca_grid* grid, int64_t n_samples, const int64_t* obs_offsets,
                 const double* coords, const double* values, const double* mean, int64_t L,
                 const double* eigenvalues, const double* eigenfunctions, double sigma2, int method, double* scores,
                 int32_t* sparse_warning) {
  return guarded(ctx, [&] {
    Grid g = make_grid(grid);
    if (n_samples < 0 || !obs_offsets || L < 0 || (method != 0 && method != 1) || (n_samples > 0 && L > 0 && !scores))
      fail(kConfig, "InvalidArgument", "invalid score request");
    if (!mean || (L > 0 && (!eigenvalues || !eigenfunctions)))
      fail(kConfig, "InvalidArgument", "score request lacks the model surfaces");
    for (i64 i = 0; i < n_samples; ++i)
      if (obs_offsets[i + 1] < obs_offsets[i] || obs_offsets[0] != 0)
        fail(kConfig, "InvalidArgument", "observation offsets must be nondecreasing from 0");
    i64 bad = -1;
    try {
      run_scores(ctx, g, n_samples, obs_offsets, coords, values, mean, L, eigenvalues, eigenfunctions, sigma2,
                 method, scores, sparse_warning, &bad);
    } catch (Failure& f) {
      f.sample = bad;
      throw;
    }
  });
}

int dfpca_reconstruct(dfpca_context* ctx, const dfpca_grid* grid, const double* mean, int64_t L,
                      const double* eigenfunctions, int64_t n, const double* scores, double* out) {
  return guarded(ctx, [&] {
    Grid g = make_grid(grid);
    if (!mean || L < 0 || n < 0 || (L > 0 && (!eigenfunctions || (n > 0 && !scores))) || (n > 0 && !out))
      fail(kConfig, "InvalidArgument", "invalid reconstruction request");
    run_reconstruct(ctx, g, mean, L, eigenfunctions, n, scores, out);
  });
}

int dfpca_dataset_upload(dfpca_context* ctx, int dim, int64_t n_samples, const int64_t* obs_offsets,
                         const double* coords, const double* values, dfpca_dataset** out) {
  return guarded(ctx, [&] {
    if (!out || dim < 1 || dim > DFPCA_MAX_DIM || n_samples < 0 || !obs_offsets)
      fail(kConfig, "InvalidArgument", "invalid dataset");
    for (i64 i = 0; i < n_samples; ++i)
      if (obs_offsets[i + 1] < obs_offsets[i] || obs_offsets[0] != 0)
        fail(kConfig, "InvalidArgument", "observation offsets must be nondecreasing from 0");
    if (obs_offsets[n_samples] > 0 && (!coords || !values)) fail(kConfig, "InvalidArgument", "null observations");
    *out = upload_dataset(ctx, dim, n_samples, obs_offsets, coords, values);
  });
}

int dfpca_dataset_free(dfpca_dataset* ds) {
  delete ds;
  return 0;
}

int dfpca_cv_units(int64_t n_samples, const int64_t* obs_offsets, int target, int64_t max_units, uint64_t seed,
                   int64_t* units, int64_t capacity, int64_t* count) {
  if (n_samples < 0 || !obs_offsets || !count || (target < 0 || target > 2) || max_units < 1) return kConfig;
  try {
    const std::vector<i64> u = cv_units(n_samples, obs_offsets, target, max_units, seed);
    *count = static_cast<int64_t>(u.size() / 3);
    if (units)
      for (std::size_t k = 0; k < u.size() && static_cast<int64_t>(k / 3) < capacity; ++k) units[k] = u[k];
    return 0;
  } catch (const Failure& f) {
    return f.cls;
  }
}

int dfpca_cv_objective(dfpca_context* ctx, const dfpca_dataset* ds, const dfpca_grid* grid, int target,
                       int64_t n_units, const int64_t* units, const double* h, double* score, int64_t* used_units) {
  return guarded(ctx, [&] {
    if (!ds || !score || (target < 0 || target > 2) || n_units < 1 || !units)
      fail(kConfig, "InvalidArgument", "invalid cross-validation request");
    Grid g = make_grid(grid);
    if (g.d != ds->dim) fail(kConfig, "InvalidBandwidth", "bandwidth dimension mismatch");
    validate_bandwidth(g, h);  // h.validate(extents_) (bandwidth.hpp:75)
    *score = run_cv_objective(ctx, ds, target, n_units, units, h, used_units);
  });
}

int dfpca_surface_rows(const dfpca_surface* s, int64_t* row0, int64_t* rows) {
  if (!s) return kConfig;
  const bool cov = s->kind == DFPCA_SURFACE_COVARIANCE;
  if (row0) *row0 = cov ? s->row0 : 0;
  if (rows) *rows = cov ? (s->rows >= 0 ? s->rows : s->grid.G) : 1;
  return 0;
}

int dfpca_shard_bounds(int64_t n1, int64_t nodes_per_plane, int64_t radius, int world, int64_t* bounds) {
  if (n1 < 1 || nodes_per_plane < 1 || radius < 0 || world < 1 || !bounds) return kConfig;
  const ShardPlan p = make_shard_plan(n1, nodes_per_plane, radius, world);
  for (int r = 0; r <= world; ++r) bounds[r] = p.bounds[static_cast<std::size_t>(r)];
  return 0;
}

int dfpca_shard_blocks(int64_t n1, int64_t nodes_per_plane, int64_t radius, int world, int phase, int64_t* out,
                       int64_t capacity, int64_t* count) {
  if (n1 < 1 || nodes_per_plane < 1 || radius < 0 || world < 1 || (phase != 0 && phase != 1) || !count)
    return kConfig;
  const ShardPlan p = make_shard_plan(n1, nodes_per_plane, radius, world);
  const std::vector<ShardBlock> bl = shard_blocks(p, phase);
  *count = static_cast<int64_t>(bl.size());
  for (std::size_t i = 0; i < bl.size() && static_cast<int64_t>(i) < capacity && out; ++i) {
    int64_t* o = out + 7 * i;
    o[0] = bl[i].src;
    o[1] = bl[i].dst;
    o[2] = bl[i].r0;
    o[3] = bl[i].r1;
    o[4] = bl[i].c0;
    o[5] = bl[i].c1;
    o[6] = bl[i].transpose ? 1 : 0;
  }
  return 0;
}

int dfpca_pair_grids(dfpca_context* ctx, const dfpca_binned* b, double* pw, double* pv) {
  return guarded(ctx, [&] {
    if (!b || !b->has_cov) fail(kConfig, "InvalidArgument", "binned data lacks the covariance path");
    const i64 G = b->grid.G;
    DevBuf<double> dpw(static_cast<std::size_t>(G * G)), dpv(static_cast<std::size_t>(G * G));
    if (b->n_pair == 0) {
      DFPCA_CUDA(cudaMemsetAsync(dpw.get(), 0, dpw.bytes(), ctx->stream));
      DFPCA_CUDA(cudaMemsetAsync(dpv.get(), 0, dpv.bytes(), ctx->stream));
    } else {
      build_pair_grids(ctx, b, dpw.get(), dpv.get());
    }
    if (pw) DFPCA_CUDA(cudaMemcpyAsync(pw, dpw.get(), dpw.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
    if (pv) DFPCA_CUDA(cudaMemcpyAsync(pv, dpv.get(), dpv.bytes(), cudaMemcpyDeviceToHost, ctx->stream));
    DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int dfpca_surface_info(const dfpca_surface* s, int* kind, int64_t* n_values) {
  if (!s) return kConfig;
  if (kind) *kind = s->kind;
  if (n_values) *n_values = s->n;
  return 0;
}

int dfpca_surface_download(dfpca_context* ctx, const dfpca_surface* s, double* out) {
  return guarded(ctx, [&] {
    if (!s || !out) fail(kConfig, "InvalidArgument", "null surface or output");
    ctx->begin_stage("download");
    copy_d2h(ctx, out, s->values.get(), static_cast<i64>(sizeof(double)) * s->n);
    ctx->end_stage();
  });
}

int dfpca_surface_gather(dfpca_context* ctx, const dfpca_surface* s, int64_t n, const int64_t* index, double* out) {
  return guarded(ctx, [&] {
    if (!s || n < 0 || (n > 0 && (!index || !out))) fail(kConfig, "InvalidArgument", "null surface, index or output");
    const i64 lo = s->rows >= 0 && s->kind == DFPCA_SURFACE_COVARIANCE ? s->row0 * s->grid.G : 0;
    for (i64 i = 0; i < n; ++i)
      if (index[i] < lo || index[i] >= lo + s->n)
        fail(kConfig, "InvalidArgument", "surface index " + std::to_string(index[i]) + " outside the surface");
    if (n == 0) return;
    DevBuf<i64> idx(static_cast<std::size_t>(n));
    DevBuf<double> vals(static_cast<std::size_t>(n));
    DFPCA_CUDA(cudaMemcpyAsync(idx.get(), index, sizeof(i64) * n, cudaMemcpyHostToDevice, ctx->stream));
    gather_values(ctx, s->values.get(), lo, idx.get(), n, vals.get());
    DFPCA_CUDA(cudaMemcpyAsync(out, vals.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int dfpca_surface_upload(dfpca_context* ctx, const dfpca_grid* grid, int kind, const double* values,
                         int64_t n_values, dfpca_surface** out) {
  return guarded(ctx, [&] {
    if (!out) fail(kConfig, "InvalidArgument", "null output handle");
    *out = nullptr;
    Grid g = make_grid(grid);
    const i64 want = kind == DFPCA_SURFACE_COVARIANCE ? g.G * g.G : g.G;
    if (n_values != want) fail(kConfig, "InvalidArgument", "surface has wrong length");
    auto s = std::make_unique<dfpca_surface>();
    s->grid = g;
    s->kind = kind;
    s->n = n_values;
    s->values.alloc(static_cast<std::size_t>(n_values));
    copy_h2d(ctx, s->values.get(), values, static_cast<i64>(sizeof(double)) * n_values);
    DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = s.release();
  });
}

int dfpca_surface_free(dfpca_surface* s) {
  delete s;
  return 0;
}

int dfpca_dense_eig(dfpca_context* ctx, const dfpca_surface* cov, const dfpca_grid* grid, int64_t L_max,
                    double* eigenvalues, double* eigenfunctions, double* fve, double* total_variance,
                    int64_t* n_components) {
  return guarded(ctx, [&] {
    if (!cov) fail(kConfig, "InvalidArgument", "null covariance surface");
    if (L_max < 0) fail(kConfig, "InvalidArgument", "L_max must be >= 0");
    Grid g = make_grid(grid);
    run_dense_eig(ctx, cov, g, L_max, eigenvalues, eigenfunctions, fve, total_variance, n_components);
  });
}

int dfpca_randomized_eig(dfpca_context* ctx, const dfpca_surface* cov, const dfpca_grid* grid, int64_t q,
                         int64_t L_max, uint64_t seed, double* eigenvalues, double* eigenfunctions,
                         double* fve, double* total_variance, int64_t* n_components) {
  return guarded(ctx, [&] {
    if (!cov) fail(kConfig, "InvalidArgument", "null covariance surface");
    Grid g = make_grid(grid);
    run_randomized_eig(ctx, cov, g, q, L_max, seed, eigenvalues, eigenfunctions, fve, total_variance,
                       n_components);
  });
}

int dfpca_eig_residuals(dfpca_context* ctx, const dfpca_surface* cov, const dfpca_grid* grid, int64_t L,
                        const double* eigenvalues, const double* eigenfunctions, double* residuals) {
  return guarded(ctx, [&] {
    if (!cov) fail(kConfig, "InvalidArgument", "null covariance surface");
    Grid g = make_grid(grid);
    run_eig_residuals(ctx, cov, g, L, eigenvalues, eigenfunctions, residuals);
  });
}

int dfpca_read_long_format(dfpca_context* ctx, const char* path, dfpca_table** out) {
  return guarded(ctx, [&] {
    if (!path || !out) fail(kConfig, "InvalidArgument", "null path or output");
    *out = read_long_format_file(ctx, path);
  });
}

int dfpca_parse_long_format(dfpca_context* ctx, const char* name, const char* bytes, int64_t n_bytes,
                            dfpca_table** out) {
  return guarded(ctx, [&] {
    if (!out || n_bytes < 0 || (n_bytes > 0 && !bytes)) fail(kConfig, "InvalidArgument", "invalid byte buffer");
    *out = parse_long_format_bytes(ctx, name, bytes, n_bytes);
  });
}

int dfpca_table_info(const dfpca_table* t, int* dim, int64_t* n_samples, int64_t* n_obs, int64_t* id_bytes) {
  if (!t) return kConfig;
  table_shape(t, dim, n_samples, n_obs, id_bytes);
  return 0;
}

int dfpca_table_copy(dfpca_context* ctx, const dfpca_table* t, int64_t* obs_offsets, double* coords, double* values,
                     int64_t* id_offsets, char* id_chars) {
  return guarded(ctx, [&] {
    if (!t) fail(kConfig, "InvalidArgument", "null table");
    table_copy(ctx, t, obs_offsets, coords, values, id_offsets, id_chars);
  });
}

int dfpca_linear_bin_table(dfpca_context* ctx, const dfpca_table* t, const dfpca_grid* grid, int mean_path,
                           int covariance_path, dfpca_binned** out) {
  return guarded(ctx, [&] {
    if (!out || !t) fail(kConfig, "InvalidArgument", "null table or output handle");
    *out = nullptr;
    Grid g = make_grid(grid);
    *out = bin_table(ctx, t, g, mean_path != 0, covariance_path != 0);
  });
}

int dfpca_table_free(dfpca_table* t) {
  table_delete(t);
  return 0;
}

}  // extern "C"
