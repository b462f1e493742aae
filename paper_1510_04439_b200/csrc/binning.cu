// K1: linear binning (reference dfpca::linear_bin, binning.hpp:82-183).
//
// Bit-exactness plan.  The reference accumulates every bin sequentially in
// (sample i, observation j, corner c) order with separate multiplies and adds
// (binning.hpp:110-181).  Floating-point addition is not associative, so an
// atomicAdd scatter cannot reproduce it.  Instead:
//   1. locate: one thread per observation replays locate_cell
//      (surface.hpp:42-66) and the corner-mass products (binning.hpp:135-145)
//      with __dmul_rn/__dsub_rn/__ddiv_rn (no contraction), and counts its
//      nonzero corners (a zero-mass corner adds +-0.0, a bitwise no-op);
//   2. an exclusive scan turns counts into record offsets in (i, j, c) order;
//   3. emit: records keyed (bin * n_samples + sample) for the grids and
//      (band index) for the self-pair bands;
//   4. a stable LSD radix sort (CUB) groups records by key while keeping the
//      (i, j, c) order inside every key;
//   5. segmented sequential sums, one thread per bin / (bin, sample) /
//      band entry, in exactly the reference order.
// The result is bitwise identical to the reference for every BinnedData field.
//
// The observations are processed in sample-aligned chunks: chunk c + 1 is
// copied to the device (its own stream) while chunk c is binned.  The grid
// and band sums continue from the values the previous chunks left (carry-in),
// so every bin still sees exactly the reference's sequence of additions.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "geometry.cuh"

namespace dfpca_gpu {
namespace {

__device__ inline i64 sample_of(const i64* offsets, i64 n_samples, i64 obs) {
  // Largest i with offsets[i] <= obs (samples may be empty).
  i64 lo = 0, hi = n_samples;  // invariant offsets[lo] <= obs < offsets[hi]
  while (hi - lo > 1) {
    const i64 mid = (lo + hi) / 2;
    if (offsets[mid] <= obs)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// Pass 1: hull check, per-observation record counts.
// Observations [o0, o1) of one chunk; counts are chunk-local (index o - o0).
template <int D>
__global__ void k_bin_count(DevGrid g, const i64* __restrict__ offsets, i64 n_samples,
                            const double* __restrict__ coords, const double* __restrict__ values,
                            i64 o0, i64 o1, const i64* __restrict__ pair_slot, int want_grid_records,
                            unsigned* __restrict__ grid_count, unsigned* __restrict__ band_count,
                            unsigned long long* __restrict__ first_bad) {
  pdl_wait();
  for (i64 o = o0 + blockIdx.x * (i64)blockDim.x + threadIdx.x; o < o1;
       o += (i64)gridDim.x * blockDim.x) {
    const double* x = coords + o * (D > 0 ? D : g.d);
    const i64 lo = o - o0;
    if (!hull_contains_dev<D>(g, x)) {
      atomicMin(first_bad, static_cast<unsigned long long>(o));
      grid_count[lo] = 0;
      if (band_count) band_count[lo] = 0;
      continue;
    }
    ObsGeom geo;
    corner_geometry<D>(g, x, geo);
    const double y = values[o];
    const bool keep_all = !isfinite(y);  // a zero-mass corner times a non-finite y is NaN
    unsigned nz = 0;
    constexpr int kd = D;
    const int d = kd > 0 ? kd : g.d;
    const int corners = 1 << d;
    #pragma unroll
    for (int c = 0; c < corners; ++c) nz += (geo.mass[c] != 0.0 || keep_all) ? 1u : 0u;
    grid_count[lo] = want_grid_records ? nz : 0u;
    unsigned nb = 0;
    if (band_count) {
      const i64 i = sample_of(offsets, n_samples, o);
      if (pair_slot[i] >= 0) {
        unsigned nzb = 0;
        #pragma unroll
        for (int c = 0; c < corners; ++c) nzb += geo.mass[c] != 0.0 ? 1u : 0u;
        nb = nzb * nzb;
      }
      band_count[lo] = nb;
    }
  }
}

// Pass 2: emit records at their scanned offsets, in (i, j, c) order.  Grid
// keys are bin * key_samples + (i - i0), i0 the chunk's first sample.
template <int D>
__global__ void k_bin_emit(DevGrid g, const i64* __restrict__ offsets, i64 n_samples,
                           const double* __restrict__ coords, const double* __restrict__ values,
                           i64 o0, i64 o1, i64 i0, i64 key_samples, const i64* __restrict__ pair_slot,
                           const double* __restrict__ pair_weight, i64 codes,
                           const unsigned* __restrict__ grid_off, const unsigned* __restrict__ band_off,
                           unsigned long long* __restrict__ gkey, unsigned* __restrict__ gval,
                           double* __restrict__ gmass, unsigned* __restrict__ gobs,
                           unsigned long long* __restrict__ bkey, unsigned* __restrict__ bval,
                           double* __restrict__ bmm, unsigned* __restrict__ bobs) {
  pdl_wait();
  for (i64 o = o0 + blockIdx.x * (i64)blockDim.x + threadIdx.x; o < o1;
       o += (i64)gridDim.x * blockDim.x) {
    const double* x = coords + o * (D > 0 ? D : g.d);
    if (!hull_contains_dev<D>(g, x)) continue;
    ObsGeom geo;
    corner_geometry<D>(g, x, geo);
    const double y = values[o];
    const bool keep_all = !isfinite(y);
    const i64 i = sample_of(offsets, n_samples, o);
    constexpr int kd = D;
    const int d = kd > 0 ? kd : g.d;
    const int corners = 1 << d;
    if (gkey) {
      unsigned r = grid_off[o - o0];
      #pragma unroll
      for (int c = 0; c < corners; ++c) {
        if (!(geo.mass[c] != 0.0 || keep_all)) continue;
        gkey[r] = static_cast<unsigned long long>(geo.flat[c]) * key_samples + (i - i0);
        gval[r] = r;
        gmass[r] = geo.mass[c];
        gobs[r] = static_cast<unsigned>(o);
        ++r;
      }
    }
    if (bkey && pair_slot[i] >= 0) {
      const double pw = pair_weight[pair_slot[i]];
      unsigned r = band_off[o - o0];
      #pragma unroll
      for (int c1 = 0; c1 < corners; ++c1) {
        if (geo.mass[c1] == 0.0) continue;
        #pragma unroll
        for (int c2 = 0; c2 < corners; ++c2) {
          if (geo.mass[c2] == 0.0) continue;
          i64 code = 0;
          for (int k = 0; k < d; ++k) {
            const int off = static_cast<int>((c2 >> k) & 1) - static_cast<int>((c1 >> k) & 1);
            code = code * 3 + (off + 1);
          }
          bkey[r] = static_cast<unsigned long long>(geo.flat[c1]) * codes + code;
          bval[r] = r;
          bmm[r] = __dmul_rn(__dmul_rn(pw, geo.mass[c1]), geo.mass[c2]);
          bobs[r] = static_cast<unsigned>(o);
          ++r;
        }
      }
    }
  }
}

constexpr int kFoldWarps = 8;  // warps per block of the ordered-fold kernels (256 threads)

// Aggregate (mean-path) grids: one thread per bin, sequential over its sorted
// records = (i, j, c) order (binning.hpp:148-155).
__global__ void k_bin_aggregate(i64 G, i64 key_samples, i64 i0, const unsigned long long* __restrict__ key,
                                const unsigned* __restrict__ val, i64 n_rec,
                                const double* __restrict__ rmass, const unsigned* __restrict__ robs,
                                const double* __restrict__ values,
                                const double* __restrict__ mean_w, double* __restrict__ mass,
                                double* __restrict__ wvalue, double* __restrict__ wsquare) {
  pdl_wait();
  // One warp per bin: the lanes gather and form the per-record terms of 32
  // consecutive records in parallel and stage them in shared memory; lanes
  // 0, 1, 2 then fold mass, wvalue, wsquare (one sum each) in record order.
  __shared__ double terms[kFoldWarps][3][33];
  const int lane = threadIdx.x & 31;
  double(&t)[3][33] = terms[threadIdx.x >> 5];
  const i64 warps = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  for (i64 f = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5; f < G; f += warps) {
    const unsigned long long target = static_cast<unsigned long long>(f) * key_samples;
    i64 lo = 0, hi = n_rec;  // lower_bound of target
    while (lo < hi) {
      const i64 mid = (lo + hi) / 2;
      if (key[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    const unsigned long long end_key = target + key_samples;
    if (lo >= n_rec || key[lo] >= end_key) continue;  // no records in this chunk
    double* const dst = lane == 0 ? mass : lane == 1 ? wvalue : wsquare;
    double acc = lane < 3 ? dst[f] : 0.0;  // carry-in from earlier chunks
    for (i64 r0 = lo;; r0 += 32) {
      const i64 r = r0 + lane;
      const bool in = r < n_rec && key[r] < end_key;
      double wm = 0.0, wmy = 0.0, wmyy = 0.0;
      if (in) {
        const unsigned rec = val[r];
        const i64 i = i0 + static_cast<i64>(key[r] - target);
        const double y = values[robs[rec]];
        wm = __dmul_rn(mean_w[i], rmass[rec]);
        wmy = __dmul_rn(wm, y);
        wmyy = __dmul_rn(wmy, y);
      }
      const unsigned m = __ballot_sync(0xffffffffu, in);
      const int cnt = __popc(m);  // records of this bin are a prefix of the 32
      t[0][lane] = wm;
      t[1][lane] = wmy;
      t[2][lane] = wmyy;
      __syncwarp();
      if (lane < 3)
        for (int q = 0; q < cnt; ++q) acc = __dadd_rn(acc, t[lane][q]);
      __syncwarp();
      if (cnt < 32) break;
    }
    if (lane < 3) dst[f] = acc;
  }
}

// Per-sample grids: one thread per distinct (bin, sample) key, sequential over
// its records = (j, c) order (binning.hpp:157-162).
__global__ void k_bin_per_sample(i64 G, i64 key_samples, i64 i0, const unsigned long long* __restrict__ key,
                                 const unsigned* __restrict__ val, i64 n_rec,
                                 const double* __restrict__ rmass,
                                 const unsigned* __restrict__ robs,
                                 const double* __restrict__ values, const i64* __restrict__ pair_slot,
                                 double* __restrict__ ps_mass, double* __restrict__ ps_value) {
  pdl_wait();
  for (i64 r0 = blockIdx.x * (i64)blockDim.x + threadIdx.x; r0 < n_rec;
       r0 += (i64)gridDim.x * blockDim.x) {
    const unsigned long long k = key[r0];
    if (r0 > 0 && key[r0 - 1] == k) continue;  // not a segment head
    const i64 f = static_cast<i64>(k / key_samples);
    const i64 i = i0 + static_cast<i64>(k % key_samples);
    const i64 slot = pair_slot[i];
    if (slot < 0) continue;
    double m = 0.0, v = 0.0;
    for (i64 r = r0; r < n_rec && key[r] == k; ++r) {
      const unsigned rec = val[r];
      const double cm = rmass[rec];
      m = __dadd_rn(m, cm);
      v = __dadd_rn(v, __dmul_rn(cm, values[robs[rec]]));
    }
    ps_mass[slot * G + f] = m;
    ps_value[slot * G + f] = v;
  }
}

// Self-pair bands: one thread per distinct band index (binning.hpp:163-178).
__global__ void k_bin_band(const unsigned long long* __restrict__ key, const unsigned* __restrict__ val,
                           i64 n_rec, i64 n_keys, const double* __restrict__ bmm,
                           const unsigned* __restrict__ robs, const double* __restrict__ values,
                           double* __restrict__ diag_mass, double* __restrict__ diag_value) {
  pdl_wait();
  // One warp per band index, records folded in order as in k_bin_aggregate
  // (lane 0 the mass sum, lane 1 the value sum).
  __shared__ double terms[kFoldWarps][2][33];
  const int lane = threadIdx.x & 31;
  double(&t)[2][33] = terms[threadIdx.x >> 5];
  const i64 warps = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  for (i64 k = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5; k < n_keys; k += warps) {
    i64 lo = 0, hi = n_rec;
    while (lo < hi) {
      const i64 mid = (lo + hi) / 2;
      if (key[mid] < static_cast<unsigned long long>(k)) lo = mid + 1;
      else hi = mid;
    }
    if (lo >= n_rec || key[lo] != static_cast<unsigned long long>(k)) continue;
    double* const dst = lane == 0 ? diag_mass : diag_value;
    double acc = lane < 2 ? dst[k] : 0.0;  // carry-in from earlier chunks
    for (i64 r0 = lo;; r0 += 32) {
      const i64 r = r0 + lane;
      const bool in = r < n_rec && key[r] == static_cast<unsigned long long>(k);
      double mm = 0.0, mv = 0.0;
      if (in) {
        const unsigned rec = val[r];
        const double y = values[robs[rec]];
        mm = bmm[rec];
        mv = __dmul_rn(__dmul_rn(mm, y), y);
      }
      const int cnt = __popc(__ballot_sync(0xffffffffu, in));
      t[0][lane] = mm;
      t[1][lane] = mv;
      __syncwarp();
      if (lane < 2)
        for (int q = 0; q < cnt; ++q) acc = __dadd_rn(acc, t[lane][q]);
      __syncwarp();
      if (cnt < 32) break;
    }
    if (lane < 2) dst[k] = acc;
  }
}

// identical_mass flag: any per-sample mass grid differing from slot 0.
__global__ void k_mass_identical(const double* __restrict__ ps_mass, i64 n_pair, i64 G,
                                 int* __restrict__ differs) {
  pdl_wait();
  const i64 total = (n_pair - 1) * G;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 f = e % G;
    const double a = ps_mass[G + e], b = ps_mass[f];
    if (__double_as_longlong(a) != __double_as_longlong(b)) {
      *differs = 1;
      return;
    }
  }
}

// Shared-design probe: mass grid constant, band diagonal-only and constant.
__global__ void k_shared_design(const double* __restrict__ m, const double* __restrict__ dm, i64 G, i64 codes,
                                i64 center, int* __restrict__ bad) {
  pdl_wait();
  const double m0 = m[0], d0 = dm[center];
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < G * codes; e += (i64)gridDim.x * blockDim.x) {
    const i64 u = e / codes, c = e - u * codes;
    const bool ok = c == center
                        ? (__double_as_longlong(dm[e]) == __double_as_longlong(d0) &&
                           __double_as_longlong(m[u]) == __double_as_longlong(m0))
                        : dm[e] == 0.0;
    if (!ok) {
      *bad = 1;
      return;
    }
  }
}

int key_bits(unsigned long long max_key) {
  int b = 1;
  while (b < 64 && (max_key >> b) != 0) ++b;
  return b;
}

}  // namespace

DevGrid upload_grid_axes(dfpca_context* ctx, const Grid& g, DevBuf<double>& storage);

// coords / values are host arrays, or device arrays when device_inputs (a
// table read on the GPU, longfmt.cu): then nothing crosses PCIe.
dfpca_binned* run_linear_bin(dfpca_context* ctx, const Grid& grid, i64 n_samples,
                             const i64* obs_offsets, const double* coords, const double* values,
                             bool mean_path, bool cov_path, bool device_inputs) {
  if (n_samples < 0) fail(kConfig, "InvalidArgument", "negative sample count");
  const int d = grid.d;
  const i64 G = grid.G;
  const i64 n_obs = n_samples > 0 ? obs_offsets[n_samples] : 0;
  for (i64 i = 0; i < n_samples; ++i)
    if (obs_offsets[i + 1] < obs_offsets[i] || obs_offsets[0] != 0)
      fail(kConfig, "InvalidArgument", "observation offsets must be nondecreasing from 0");
  if (n_obs * (1ll << (2 * d)) >= (1ll << 32))
    fail(kConfig, "InvalidArgument", "too many observations for one binning call");

  auto out = std::make_unique<dfpca_binned>();
  out->grid = grid;
  out->n_samples = n_samples;
  out->has_mean = mean_path;
  out->has_cov = cov_path;
  out->codes = 1;
  for (int k = 0; k < d; ++k) out->codes *= 3;
  out->sample_sizes.resize(static_cast<std::size_t>(n_samples));

  // Host bookkeeping: sample sizes, 1/N_i, pair slots and weights (binning.hpp:118-127).
  std::vector<double> mean_w(static_cast<std::size_t>(std::max<i64>(n_samples, 1)), 0.0);
  std::vector<i64> slot(static_cast<std::size_t>(std::max<i64>(n_samples, 1)), -1);
  for (i64 i = 0; i < n_samples; ++i) {
    const i64 n = obs_offsets[i + 1] - obs_offsets[i];
    out->sample_sizes[static_cast<std::size_t>(i)] = n;
    mean_w[static_cast<std::size_t>(i)] = n > 0 ? 1.0 / static_cast<double>(n) : 0.0;
    if (cov_path && n >= 2) {
      slot[static_cast<std::size_t>(i)] = out->n_pair;
      out->sample_index.push_back(i);
      out->pair_weight_h.push_back(1.0 / (static_cast<double>(n) * static_cast<double>(n - 1)));
      ++out->n_pair;
    }
  }

  // the per-observation kernels with d as a template constant
  auto const k_bin_count_d = d == 1 ? &k_bin_count<1> : d == 2 ? &k_bin_count<2> : d == 3 ? &k_bin_count<3>
                                                                                        : &k_bin_count<0>;
  auto const k_bin_emit_d = d == 1 ? &k_bin_emit<1> : d == 2 ? &k_bin_emit<2> : d == 3 ? &k_bin_emit<3>
                                                                                     : &k_bin_emit<0>;
  ctx->begin_stage("binning");
  cudaStream_t st = ctx->stream;
  DevBuf<double> axes_store;
  DevGrid dg = upload_grid_axes(ctx, grid, axes_store);

  DevBuf<i64> d_off(static_cast<std::size_t>(n_samples + 1));
  DevBuf<double> d_coords_buf(static_cast<std::size_t>(device_inputs ? 0 : std::max<i64>(n_obs * d, 1)));
  DevBuf<double> d_values_buf(static_cast<std::size_t>(device_inputs ? 0 : std::max<i64>(n_obs, 1)));
  struct Ptr {
    const double* p;
    const double* get() const { return p; }
  };
  const Ptr d_coords{device_inputs ? coords : d_coords_buf.get()};
  const Ptr d_values{device_inputs ? values : d_values_buf.get()};
  DevBuf<double> d_meanw(mean_w.size());
  DevBuf<i64> d_slot(slot.size());
  DFPCA_CUDA(cudaMemcpyAsync(d_off.get(), obs_offsets, sizeof(i64) * (n_samples + 1),
                             cudaMemcpyHostToDevice, st));
  // Pageable observations are staged through pinned slots by host threads
  // before the binning starts (the chunked overlap below needs pinned memory
  // for the copies to be asynchronous).
  const i64 coord_bytes = static_cast<i64>(sizeof(double)) * n_obs * d;
  const bool staged = !device_inputs && n_obs > 0 && copy_is_staged(coords, coord_bytes);
  if (staged) {
    copy_h2d(ctx, d_coords_buf.get(), coords, coord_bytes);
    copy_h2d(ctx, d_values_buf.get(), values, static_cast<i64>(sizeof(double)) * n_obs);
  }
  DFPCA_CUDA(cudaMemcpyAsync(d_meanw.get(), mean_w.data(), sizeof(double) * mean_w.size(),
                             cudaMemcpyHostToDevice, st));
  DFPCA_CUDA(cudaMemcpyAsync(d_slot.get(), slot.data(), sizeof(i64) * slot.size(),
                             cudaMemcpyHostToDevice, st));

  if (mean_path) {
    out->mass.alloc(G);
    out->wvalue.alloc(G);
    out->wsquare.alloc(G);
    DFPCA_CUDA(cudaMemsetAsync(out->mass.get(), 0, out->mass.bytes(), st));
    DFPCA_CUDA(cudaMemsetAsync(out->wvalue.get(), 0, out->wvalue.bytes(), st));
    DFPCA_CUDA(cudaMemsetAsync(out->wsquare.get(), 0, out->wsquare.bytes(), st));
  }
  if (cov_path) {
    out->diag_mass.alloc(G * out->codes);
    out->diag_value.alloc(G * out->codes);
    DFPCA_CUDA(cudaMemsetAsync(out->diag_mass.get(), 0, out->diag_mass.bytes(), st));
    DFPCA_CUDA(cudaMemsetAsync(out->diag_value.get(), 0, out->diag_value.bytes(), st));
    if (out->n_pair > 0) {
      out->ps_mass.alloc(static_cast<std::size_t>(out->n_pair * G));
      out->ps_value.alloc(static_cast<std::size_t>(out->n_pair * G));
      out->pair_weight.alloc(static_cast<std::size_t>(out->n_pair));
      DFPCA_CUDA(cudaMemsetAsync(out->ps_mass.get(), 0, out->ps_mass.bytes(), st));
      DFPCA_CUDA(cudaMemsetAsync(out->ps_value.get(), 0, out->ps_value.bytes(), st));
      DFPCA_CUDA(cudaMemcpyAsync(out->pair_weight.get(), out->pair_weight_h.data(),
                                 sizeof(double) * out->n_pair, cudaMemcpyHostToDevice, st));
    }
  }

  if (n_obs > 0) {
    const bool want_grid = mean_path || (cov_path && out->n_pair > 0);
    const bool want_band = cov_path && out->n_pair > 0;
    // Sample-aligned chunks of about kChunkObs observations; every chunk's
    // copy is queued at once on the copy stream, the binning of chunk c waits
    // only for chunk c.  Each chunk costs a host round trip and a pass over
    // the bins, so chunks stay large: measured on the cfg-3 input (8.2 M
    // observations, 197 MB) 6.2 ms unchunked or in 1 M chunks, 5.1 ms in 4.
    i64 kChunkObs = std::max<i64>(i64{1} << 21, n_obs / 4);
    if (const char* e = std::getenv("DFPCA_BIN_CHUNK_OBS")) kChunkObs = std::max<i64>(1, std::atoll(e));
    std::vector<i64> cut{0};  // sample boundaries
    for (i64 i = 1; i <= n_samples; ++i)
      if (i == n_samples || obs_offsets[i] - obs_offsets[cut.back()] >= kChunkObs) cut.push_back(i);
    const std::size_t n_chunks = cut.size() - 1;
    cudaStream_t cs = ctx->copy_stream();
    std::vector<cudaEvent_t> arrived(n_chunks);
    struct Events {
      std::vector<cudaEvent_t>& e;
      ~Events() {
        for (auto x : e)
          if (x) cudaEventDestroy(x);
      }
    } events_guard{arrived};
    DFPCA_CUDA(cudaEventRecord(ctx->fence(), st));  // the allocations above are ordered before the copies
    DFPCA_CUDA(cudaStreamWaitEvent(cs, ctx->fence(), 0));
    for (std::size_t c = 0; c < n_chunks; ++c) {
      const i64 o0 = obs_offsets[cut[c]], o1 = obs_offsets[cut[c + 1]];
      if (o1 > o0 && !device_inputs && !staged) {
        DFPCA_CUDA(cudaMemcpyAsync(d_coords_buf.get() + o0 * d, coords + o0 * d, sizeof(double) * (o1 - o0) * d,
                                   cudaMemcpyHostToDevice, cs));
        DFPCA_CUDA(cudaMemcpyAsync(d_values_buf.get() + o0, values + o0, sizeof(double) * (o1 - o0),
                                   cudaMemcpyHostToDevice, cs));
      }
      arrived[c] = nullptr;
      DFPCA_CUDA(cudaEventCreateWithFlags(&arrived[c], cudaEventDisableTiming));
      DFPCA_CUDA(cudaEventRecord(arrived[c], cs));
    }
    // whatever happens below, the context stream waits for every copy before
    // the observation buffers are released (stream-ordered frees on st)
    struct CopiesDone {
      cudaStream_t st;
      cudaEvent_t last;
      ~CopiesDone() { cudaStreamWaitEvent(st, last, 0); }
    } copies_done{st, arrived.back()};
    // Per-chunk counts and record offsets on a second compute stream, queued
    // for every chunk up front: chunk c's counting runs as soon as it has
    // arrived, beside the sorting and summing of chunk c - 1 on `st`; the host
    // waits only for the totals of the chunk it is about to emit.
    cudaStream_t as = ctx->aux_stream();
    struct Counts {
      DevBuf<unsigned> gcount, bcount, goff, boff;
      DevBuf<unsigned char> tmp;
      cudaEvent_t done = nullptr;
    };
    std::vector<Counts> cnt(n_chunks);
    DevBuf<unsigned long long> bad(1);
    const unsigned long long none = ~0ull;
    DFPCA_CUDA(cudaMemcpyAsync(bad.get(), &none, sizeof(none), cudaMemcpyHostToDevice, st));
    for (std::size_t c = 0; c < n_chunks; ++c) {
      const i64 nc = obs_offsets[cut[c + 1]] - obs_offsets[cut[c]];
      Counts& k = cnt[c];
      k.gcount.alloc(static_cast<std::size_t>(nc + 1));
      k.bcount.alloc(static_cast<std::size_t>(nc + 1));
      k.goff.alloc(static_cast<std::size_t>(nc + 1));
      k.boff.alloc(static_cast<std::size_t>(nc + 1));
      std::size_t tb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb, k.gcount.get(), k.goff.get(), nc + 1, as);
      k.tmp.alloc(std::max<std::size_t>(tb, 1));
      DFPCA_CUDA(cudaEventCreateWithFlags(&k.done, cudaEventDisableTiming));
    }
    // host slots: [first bad, grid total, band total] per chunk
    unsigned long long* slots = ctx->pinned_u64(3 * n_chunks);
    struct CountsDone {
      cudaStream_t st;
      std::vector<Counts>& cnt;
      ~CountsDone() {
        for (auto& k : cnt)
          if (k.done) {
            cudaStreamWaitEvent(st, k.done, 0);  // before the buffers are freed on st
            cudaEventDestroy(k.done);
          }
      }
    } counts_done{st, cnt};
    DFPCA_CUDA(cudaEventRecord(ctx->fence(), st));  // allocations and the bad-flag reset
    DFPCA_CUDA(cudaStreamWaitEvent(as, ctx->fence(), 0));
    auto aux_launch = [&](const char* what, cudaError_t e) {
      cuda_check(e == cudaSuccess ? cudaGetLastError() : e, what);
      ++ctx->launches;
    };
    for (std::size_t c = 0; c < n_chunks; ++c) {
      const i64 o0 = obs_offsets[cut[c]], o1 = obs_offsets[cut[c + 1]], nc = o1 - o0;
      Counts& k = cnt[c];
      DFPCA_CUDA(cudaStreamWaitEvent(as, arrived[c], 0));
      if (nc > 0) {
        DFPCA_CUDA(cudaMemsetAsync(k.gcount.get() + nc, 0, sizeof(unsigned), as));
        DFPCA_CUDA(cudaMemsetAsync(k.bcount.get() + nc, 0, sizeof(unsigned), as));
        k_bin_count_d<<<grid_for(nc, 256), 256, 0, as>>>(dg, d_off.get(), n_samples, d_coords.get(), d_values.get(), o0,
                                                       o1, d_slot.get(), want_grid ? 1 : 0, k.gcount.get(),
                                                       want_band ? k.bcount.get() : nullptr, bad.get());
        aux_launch("k_bin_count", cudaSuccess);
        std::size_t tb = k.tmp.size();
        aux_launch("scan", cub::DeviceScan::ExclusiveSum(k.tmp.get(), tb, k.gcount.get(), k.goff.get(), nc + 1, as));
        if (want_band)
          aux_launch("scan", cub::DeviceScan::ExclusiveSum(k.tmp.get(), tb, k.bcount.get(), k.boff.get(), nc + 1, as));
        DFPCA_CUDA(cudaMemcpyAsync(slots + 3 * c + 1, k.goff.get() + nc, sizeof(unsigned), cudaMemcpyDeviceToHost, as));
        DFPCA_CUDA(cudaMemcpyAsync(slots + 3 * c + 2, k.boff.get() + nc, sizeof(unsigned), cudaMemcpyDeviceToHost, as));
      }
      DFPCA_CUDA(cudaMemcpyAsync(slots + 3 * c, bad.get(), sizeof(unsigned long long), cudaMemcpyDeviceToHost, as));
      DFPCA_CUDA(cudaEventRecord(k.done, as));
    }
    for (std::size_t c = 0; c < n_chunks; ++c) {
      const i64 i0 = cut[c], i1 = cut[c + 1];
      const i64 o0 = obs_offsets[i0], o1 = obs_offsets[i1], nc = o1 - o0;
      Counts& k = cnt[c];
      DFPCA_CUDA(cudaEventSynchronize(k.done));
      const unsigned long long first_bad = slots[3 * c];
      if (first_bad != none) {
        const i64 o = static_cast<i64>(first_bad);
        const i64 i = std::upper_bound(obs_offsets, obs_offsets + n_samples + 1, o) - obs_offsets - 1;
        fail_at(kConfig, "ObservationOutsideGrid",
                "sample " + std::to_string(i) + " observation " + std::to_string(o - obs_offsets[i]) +
                    " lies outside the grid hull",
                i, o - obs_offsets[i]);
      }
      if (nc == 0) continue;
      DFPCA_CUDA(cudaStreamWaitEvent(st, k.done, 0));
      unsigned totals[2] = {static_cast<unsigned>(slots[3 * c + 1] & 0xffffffffull),
                            static_cast<unsigned>(slots[3 * c + 2] & 0xffffffffull)};
      const DevBuf<unsigned>& goff = k.goff;
      const DevBuf<unsigned>& boff = k.boff;
      const i64 n_grec = want_grid ? totals[0] : 0;
      const i64 n_brec = want_band ? totals[1] : 0;
      const i64 key_samples = i1 - i0;

      DevBuf<unsigned long long> gkey(n_grec + 1), gkey2(n_grec + 1), bkey(n_brec + 1), bkey2(n_brec + 1);
      DevBuf<unsigned> gval(n_grec + 1), gval2(n_grec + 1), bval(n_brec + 1), bval2(n_brec + 1);
      DevBuf<double> gmass(n_grec + 1), bmm(n_brec + 1);
      DevBuf<unsigned> gobs(n_grec + 1), bobs(n_brec + 1);
      DFPCA_LAUNCH(ctx, k_bin_emit_d, grid_for(nc, 256), 256, 0, dg, d_off.get(), n_samples, d_coords.get(),
                   d_values.get(), o0, o1, i0, key_samples, d_slot.get(), out->pair_weight.get(), out->codes,
                   goff.get(), boff.get(), n_grec > 0 ? gkey.get() : nullptr, gval.get(), gmass.get(), gobs.get(),
                   n_brec > 0 ? bkey.get() : nullptr, bval.get(), bmm.get(), bobs.get());

      if (n_grec > 0) {
        const int bits = key_bits(static_cast<unsigned long long>(G) * key_samples);
        std::size_t sb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, sb, gkey.get(), gkey2.get(), gval.get(), gval2.get(), n_grec, 0,
                                        bits, st);
        unsigned char* stmp = ctx->scratch_bytes(sb);
        cub::DeviceRadixSort::SortPairs(stmp, sb, gkey.get(), gkey2.get(), gval.get(), gval2.get(), n_grec, 0,
                                        bits, st);
        ctx->launches += (bits + 7) / 8 + 1;
        if (mean_path)
          DFPCA_LAUNCH(ctx, k_bin_aggregate, grid_for(G * 32, 256), 256, 0, G, key_samples, i0, gkey2.get(),
                       gval2.get(), n_grec, gmass.get(), gobs.get(), d_values.get(), d_meanw.get(), out->mass.get(),
                       out->wvalue.get(), out->wsquare.get());
        if (cov_path && out->n_pair > 0)
          DFPCA_LAUNCH(ctx, k_bin_per_sample, grid_for(n_grec, 256), 256, 0, G, key_samples, i0, gkey2.get(),
                       gval2.get(), n_grec, gmass.get(), gobs.get(), d_values.get(), d_slot.get(),
                       out->ps_mass.get(), out->ps_value.get());
      }
      if (n_brec > 0) {
        const int bits = key_bits(static_cast<unsigned long long>(G) * out->codes);
        std::size_t sb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, sb, bkey.get(), bkey2.get(), bval.get(), bval2.get(), n_brec, 0,
                                        bits, st);
        unsigned char* stmp = ctx->scratch_bytes(sb);
        cub::DeviceRadixSort::SortPairs(stmp, sb, bkey.get(), bkey2.get(), bval.get(), bval2.get(), n_brec, 0,
                                        bits, st);
        ctx->launches += (bits + 7) / 8 + 1;
        DFPCA_LAUNCH(ctx, k_bin_band, grid_for(G * out->codes * 32, 256), 256, 0, bkey2.get(), bval2.get(), n_brec,
                     G * out->codes, bmm.get(), bobs.get(), d_values.get(), out->diag_mass.get(),
                     out->diag_value.get());
      }
    }
  }

  if (cov_path && out->n_pair > 1) {
    DevBuf<int> differs(1);
    DFPCA_CUDA(cudaMemsetAsync(differs.get(), 0, sizeof(int), st));
    DFPCA_LAUNCH(ctx, k_mass_identical, grid_for((out->n_pair - 1) * G, 256), 256, 0,
                 out->ps_mass.get(), out->n_pair, G, differs.get());
    int h_differs = 1;
    DFPCA_CUDA(cudaMemcpyAsync(&h_differs, differs.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    DFPCA_CUDA(cudaStreamSynchronize(st));
    out->identical_mass = h_differs == 0;
  } else {
    out->identical_mass = cov_path && out->n_pair == 1;
  }
  detect_shared_design(ctx, out.get());
  ctx->end_stage();
  DFPCA_CUDA(cudaStreamSynchronize(st));
  return out.release();
}

void detect_shared_design(dfpca_context* ctx, dfpca_binned* b) {
  b->shared_const = false;
  if (!b->has_cov || !b->identical_mass || b->n_pair < 1) return;
  const i64 G = b->grid.G;
  const i64 center = (b->codes - 1) / 2;  // code digits o_k + 1 = 1 on every axis
  cudaStream_t st = ctx->stream;
  DevBuf<int> bad(1);
  DFPCA_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), st));
  DFPCA_LAUNCH(ctx, k_shared_design, grid_for(G * b->codes, 256), 256, 0, b->ps_mass.get(), b->diag_mass.get(), G,
               b->codes, center, bad.get());
  int h_bad = 1;
  double m0 = 0.0, dm0 = 0.0;
  DFPCA_CUDA(cudaMemcpyAsync(&h_bad, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaMemcpyAsync(&m0, b->ps_mass.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaMemcpyAsync(&dm0, b->diag_mass.get() + center, sizeof(double), cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
  b->shared_const = h_bad == 0 && m0 > 0.0 && std::isfinite(m0) && std::isfinite(dm0);
  b->shared_m0 = m0;
  b->shared_dm0 = dm0;
}

}  // namespace dfpca_gpu
