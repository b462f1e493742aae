// SURVEY.md 8(f) rank 1 on the device: pooled noise variance, per-sample
// component scores (conditional expectation / integration) and curve
// reconstruction (reference scores.hpp:82-300).
//
//  * estimate_sigma2 (scores.hpp:82-108): one ordered pass over the in-mask
//    nodes (a single thread: the reference's running sum, no reassociation),
//    reading the covariance diagonal straight from the device-resident surface
//    (gathered from the ranks' slabs when sharded).
//  * integration_scores (scores.hpp:204-262): one warp per sample replays the
//    tent gridding observation by observation (the 2^d corner lanes add to
//    distinct nodes, __syncwarp between observations keeps every node's sum in
//    the reference's (j, c) order), then one thread per (sample, component)
//    forms the Riemann sum over nodes in ascending order with separate
//    rounded operations -- bit-identical to the reference.
//  * pace_scores (scores.hpp:157-194): one CTA per sample: interpolated design
//    (interp_multilinear, surface.hpp:77-105, replayed exactly), the
//    observation covariance Phi diag(lambda) Phi^T + noise I, Eigen's pivoted
//    LDLT (the same left-looking algorithm as the local-fit solve, rows
//    updated in parallel, every entry in Eigen's order), the solve and the
//    dot products.  Summation orders are the plain sequential ones; Eigen's
//    own product kernels vectorize and are version dependent, so parity is
//    to tolerance.
//  * reconstruct_on_grid (scores.hpp:280-300): elementwise.
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"
#include "geometry.cuh"
#include "shard_exec.hpp"

namespace dfpca_gpu {

DevGrid upload_grid_axes(dfpca_context* ctx, const Grid& g, DevBuf<double>& storage);

namespace {

constexpr double kSigmaFloorRel = 1e-6;  // detail::kSigmaFloorRel (scores.hpp:113)
constexpr int kPaceMaxObs = 160;         // one CTA's shared-memory design

__device__ inline double nan_d() { return __longlong_as_double(0x7ff8000000000000ll); }

// interp_multilinear (surface.hpp:77-105) of one surface at x (inside the hull)
__device__ inline double interp_dev(const DevGrid& g, const double* __restrict__ values, const double* x) {
  ObsGeom geo;
  corner_geometry(g, x, geo);
  double acc = 0.0, wsum = 0.0;
  const int corners = 1 << g.d;
  for (int c = 0; c < corners; ++c) {
    const double w = geo.mass[c];
    if (w == 0.0) continue;
    const double v = values[geo.flat[c]];
    if (isnan(v)) continue;
    acc = __dadd_rn(acc, __dmul_rn(w, v));
    wsum = __dadd_rn(wsum, w);
  }
  return wsum <= 0.0 ? nan_d() : __ddiv_rn(acc, wsum);
}

// ---- estimate_sigma2 ----
__global__ void k_cov_diagonal(const double* __restrict__ slab, i64 G, i64 row0, i64 rows, double* __restrict__ diag) {
  pdl_wait();
  for (i64 r = blockIdx.x * (i64)blockDim.x + threadIdx.x; r < rows; r += (i64)gridDim.x * blockDim.x)
    diag[row0 + r] = slab[r * G + row0 + r];
}

__global__ void k_sigma2(const double* __restrict__ dpn, const double* __restrict__ gdiag,
                         const double* __restrict__ mean, const std::uint8_t* __restrict__ mask, i64 G,
                         double* __restrict__ out) {
  pdl_wait();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0;
  i64 count = 0;
  for (i64 f = 0; f < G; ++f) {
    if (mask && !mask[f]) continue;
    const double b0 = dpn[f], gd = gdiag[f], mu = mean[f];
    if (isnan(b0) || isnan(gd) || isnan(mu)) continue;
    acc = __dadd_rn(acc, __dsub_rn(__dsub_rn(b0, gd), __dmul_rn(mu, mu)));
    ++count;
  }
  const double s = count == 0 ? 0.0 : __ddiv_rn(acc, static_cast<double>(count));
  out[0] = count == 0 ? 0.0 : (s > 0.0 ? s : 0.0);
}

// ---- integration scores ----
// One warp per sample: lanes 0..2^d-1 own the corners of the current
// observation; hull violations are reported (first sample, observation).
__global__ void k_tent_grid(DevGrid g, const i64* __restrict__ offsets, i64 n_samples,
                            const double* __restrict__ coords, const double* __restrict__ values,
                            double* __restrict__ mass, double* __restrict__ wval,
                            unsigned long long* __restrict__ bad) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const i64 warps = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  const int corners = 1 << g.d;
  const i64 G = g.strides[0] * g.shape[0];
  for (i64 i = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5; i < n_samples; i += warps) {
    double* m = mass + i * G;
    double* v = wval + i * G;
    for (i64 j = offsets[i]; j < offsets[i + 1]; ++j) {
      const double* x = coords + j * g.d;
      if (!hull_contains_dev(g, x)) {
        if (lane == 0) atomicMin(bad, static_cast<unsigned long long>(j));
        break;
      }
      if (lane < corners) {
        ObsGeom geo;
        corner_geometry(g, x, geo);
        const double w = geo.mass[lane];
        if (w != 0.0) {
          const i64 f = geo.flat[lane];
          m[f] = __dadd_rn(m[f], w);
          v[f] = __dadd_rn(v[f], __dmul_rn(w, values[j]));
        }
      }
      __syncwarp();
    }
  }
}

__global__ void k_integration_scores(const double* __restrict__ mass, const double* __restrict__ wval,
                                     const double* __restrict__ mean, const double* __restrict__ phi,
                                     const std::uint8_t* __restrict__ mask, i64 G, i64 n, i64 L, double cv,
                                     double* __restrict__ out) {
  pdl_wait();
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < n * L; e += (i64)gridDim.x * blockDim.x) {
    const i64 i = e / L, l = e % L;
    const double* m = mass + i * G;
    const double* v = wval + i * G;
    const double* p = phi + l * G;
    double acc = 0.0;
    for (i64 f = 0; f < G; ++f) {
      if ((mask && !mask[f]) || m[f] <= 0.0) continue;
      const double mu = mean[f];
      if (isnan(mu)) continue;
      const double c = __dsub_rn(__ddiv_rn(v[f], m[f]), mu);
      const double pf = p[f];
      if (!isnan(pf)) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(c, pf), cv));
    }
    out[e] = acc;
  }
}

// ---- PACE ----
// One CTA per sample.  Shared memory: design rows phi [N][L], centered y [N],
// the N x N observation covariance (column-major, as Eigen) and work vectors.
struct PaceArgs {
  DevGrid g;
  const i64* offsets;
  const double* coords;
  const double* values;
  const double* mean;
  const double* phi;  // [L][G]
  const double* lambda;
  i64 L, n_samples;
  double noise;
  double* out;        // [n][L]
  int* status;        // per sample: 0 ok, 1 singular, 2 outside hull
};

// BIG = false: samples with at most kPaceMaxObs observations, everything in
// shared memory (the others are left to the BIG launch).  BIG = true: one CTA
// per listed sample, the same steps on a per-CTA global-memory workspace of
// cap * (L + 2) + cap^2 doubles and 3 cap ints (any observation count).
template <bool BIG>
__global__ void k_pace(PaceArgs a, const i64* big_list, double* ws, int* iws, i64 cap) {
  pdl_wait();
  extern __shared__ double sm[];
  const i64 i = BIG ? big_list[blockIdx.x] : static_cast<i64>(blockIdx.x);
  if (i >= a.n_samples) return;
  const i64 j0 = a.offsets[i], nobs = a.offsets[i + 1] - j0;
  if (!BIG && nobs > kPaceMaxObs) return;
  const i64 L = a.L;
  double *ph, *yc, *S, *temp;
  int *used_idx, *trans, *ok_flag;
  if constexpr (BIG) {
    double* w = ws + static_cast<i64>(blockIdx.x) * (cap * (L + 2) + cap * cap);
    ph = w;                 // [cap][L]
    yc = ph + cap * L;      // [cap]
    temp = yc + cap;        // [cap]
    S = temp + cap;         // [N][N] column-major
    int* iw = iws + static_cast<i64>(blockIdx.x) * 3 * cap;
    used_idx = iw;
    trans = iw + cap;
    ok_flag = iw + 2 * cap;
  } else {
    __shared__ int used_sh[kPaceMaxObs], trans_sh[kPaceMaxObs], ok_sh[kPaceMaxObs];
    __shared__ double temp_sh[kPaceMaxObs];
    ph = sm;                          // [kPaceMaxObs][L]
    yc = ph + kPaceMaxObs * L;        // [kPaceMaxObs]
    S = yc + kPaceMaxObs;             // [N][N] column-major
    temp = temp_sh;
    used_idx = used_sh;
    trans = trans_sh;
    ok_flag = ok_sh;
  }
  __shared__ int n_used, bad;
  if (threadIdx.x == 0) {
    n_used = 0;
    bad = 0;
  }
  __syncthreads();
  // design, in observation order (one thread per observation, then a stable
  // compaction of the usable ones)
  for (i64 j = threadIdx.x; j < nobs; j += blockDim.x) {
    const double* x = a.coords + (j0 + j) * a.g.d;
    int ok = 1;
    if (!hull_contains_dev(a.g, x)) {
      ok = 0;
      atomicExch(&bad, 1);
    }
    double mu = ok ? interp_dev(a.g, a.mean, x) : nan_d();
    if (isnan(mu)) ok = 0;
    for (i64 l = 0; l < L && ok; ++l) {
      const double p = interp_dev(a.g, a.phi + l * (a.g.strides[0] * a.g.shape[0]), x);
      if (isnan(p)) ok = 0;
      ph[j * L + l] = p;
    }
    yc[j] = ok ? __dsub_rn(a.values[j0 + j], mu) : 0.0;
    ok_flag[j] = ok;
  }
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) a.status[i] = 2;
    return;
  }
  if (threadIdx.x == 0) {
    int u = 0;
    for (i64 j = 0; j < nobs; ++j)
      if (ok_flag[j]) used_idx[u++] = static_cast<int>(j);
    n_used = u;
  }
  __syncthreads();
  const int N = n_used;
  double* out = a.out + i * L;
  if (N == 0) {
    for (i64 l = threadIdx.x; l < L; l += blockDim.x) out[l] = 0.0;
    if (threadIdx.x == 0) a.status[i] = 0;
    return;
  }
  // compact rows in place (used_idx ascending, so a forward copy is safe)
  if (threadIdx.x == 0)
    for (int r = 0; r < N; ++r) {
      const int src = used_idx[r];
      if (src != r) {
        for (i64 l = 0; l < L; ++l) ph[r * L + l] = ph[src * L + l];
        yc[r] = yc[src];
      }
    }
  __syncthreads();
  // Sigma_y(r, c) = sum_k (phi(r,k) lambda_k) phi(c,k), k ascending, + noise on the diagonal
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
    const int r = e % N, c = e / N;
    double s = 0.0;
    for (i64 k = 0; k < L; ++k) s = __dadd_rn(s, __dmul_rn(__dmul_rn(ph[r * L + k], a.lambda[k]), ph[c * L + k]));
    if (r == c) s = __dadd_rn(s, a.noise);
    S[c * N + r] = s;
  }
  __syncthreads();
  // Eigen ldlt_inplace<Lower>::unblocked with diagonal pivoting
  __shared__ int ret_sh, fzp_sh, piv_sh;
  if (threadIdx.x == 0) {
    ret_sh = 1;
    fzp_sh = 0;
  }
  __syncthreads();
#define A_(r, c) S[(c) * N + (r)]
  for (int k = 0; k < N; ++k) {
    if (threadIdx.x == 0) {
      int piv = k;
      double best = fabs(A_(k, k));
      for (int q = k + 1; q < N; ++q)
        if (fabs(A_(q, q)) > best) {
          best = fabs(A_(q, q));
          piv = q;
        }
      trans[k] = piv;
      piv_sh = piv;
    }
    __syncthreads();
    const int piv = piv_sh;
    if (piv != k) {
      // swap rows k <-> piv of the factored columns, column k <-> piv below piv,
      // the diagonal, and the mirrored strip between them (Eigen's order)
      for (int j = threadIdx.x; j < k; j += blockDim.x) {
        const double t = A_(k, j);
        A_(k, j) = A_(piv, j);
        A_(piv, j) = t;
      }
      for (int q = piv + 1 + threadIdx.x; q < N; q += blockDim.x) {
        const double t = A_(q, k);
        A_(q, k) = A_(q, piv);
        A_(q, piv) = t;
      }
      if (threadIdx.x == 0) {
        const double t = A_(k, k);
        A_(k, k) = A_(piv, piv);
        A_(piv, piv) = t;
      }
      for (int q = k + 1 + threadIdx.x; q < piv; q += blockDim.x) {
        const double t = A_(q, k);
        A_(q, k) = A_(piv, q);
        A_(piv, q) = t;
      }
    }
    __syncthreads();
    if (k > 0) {
      for (int j = threadIdx.x; j < k; j += blockDim.x) temp[j] = __dmul_rn(A_(j, j), A_(k, j));
      __syncthreads();
      // rows k..N-1 of column k: each entry's dot product in ascending j
      for (int q = k + threadIdx.x; q < N; q += blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < k; ++j) s = __dadd_rn(s, __dmul_rn(A_(q, j), temp[j]));
        A_(q, k) = __dsub_rn(A_(q, k), s);
      }
      __syncthreads();
    }
    const double akk = A_(k, k);
    const bool valid = fabs(akk) > 0.0;
    if (k == 0 && !valid) {
      if (threadIdx.x == 0) ret_sh = 0;
      __syncthreads();
      break;
    }
    if (valid) {
      for (int q = k + 1 + threadIdx.x; q < N; q += blockDim.x) A_(q, k) = __ddiv_rn(A_(q, k), akk);
    } else if (threadIdx.x == 0) {
      for (int q = k + 1; q < N; ++q)
        if (A_(q, k) != 0.0) ret_sh = 0;
    }
    if (threadIdx.x == 0) {
      if (fzp_sh && valid) ret_sh = 0;
      else if (!valid) fzp_sh = 1;
    }
    __syncthreads();
  }
  // info() == Success and min D > 0, else SingularCovariance
  __shared__ int singular;
  if (threadIdx.x == 0) {
    double dmin = 1.0 / 0.0;
    for (int q = 0; q < N; ++q) dmin = A_(q, q) < dmin ? A_(q, q) : dmin;
    singular = (!ret_sh || !(dmin > 0.0)) ? 1 : 0;
    a.status[i] = singular;
  }
  __syncthreads();
  if (singular) return;
  // w = P^T L^-T D^-1 L^-1 P y (LDLT::solve), sequential like Eigen's triangular solves
  if (threadIdx.x == 0) {
    double* x = temp;
    for (int q = 0; q < N; ++q) x[q] = yc[q];
    for (int k = 0; k < N; ++k) {
      const double t = x[k];
      x[k] = x[trans[k]];
      x[trans[k]] = t;
    }
    for (int j = 0; j < N; ++j)
      for (int q = j + 1; q < N; ++q) x[q] = __dsub_rn(x[q], __dmul_rn(A_(q, j), x[j]));
    for (int q = 0; q < N; ++q) x[q] = fabs(A_(q, q)) > 2.2250738585072014e-308 ? __ddiv_rn(x[q], A_(q, q)) : 0.0;
    for (int j = N - 1; j >= 0; --j)
      for (int q = 0; q < j; ++q) x[q] = __dsub_rn(x[q], __dmul_rn(A_(j, q), x[j]));
    for (int k = N - 1; k >= 0; --k) {
      const double t = x[k];
      x[k] = x[trans[k]];
      x[trans[k]] = t;
    }
  }
#undef A_
  __syncthreads();
  for (i64 l = threadIdx.x; l < L; l += blockDim.x) {
    double dot = 0.0;
    for (int q = 0; q < N; ++q) dot = __dadd_rn(dot, __dmul_rn(ph[q * L + l], temp[q]));
    out[l] = __dmul_rn(a.lambda[l], dot);
  }
}

// ---- reconstruct_on_grid ----
__global__ void k_reconstruct(const double* __restrict__ mean, const double* __restrict__ phi, i64 G, i64 L,
                              const double* __restrict__ scores, i64 n, double* __restrict__ out) {
  pdl_wait();
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < n * G; e += (i64)gridDim.x * blockDim.x) {
    const i64 i = e / G, f = e % G;
    const double mu = mean[f];
    double x = mu;
    if (!isnan(mu))
      for (i64 l = 0; l < L; ++l) {
        const double p = phi[l * G + f];
        if (isnan(p)) {
          x = nan_d();
          break;
        }
        x = __dadd_rn(x, __dmul_rn(scores[i * L + l], p));
      }
    out[e] = isnan(mu) ? nan_d() : x;
  }
}

}  // namespace

void run_estimate_sigma2(dfpca_context* ctx, const Grid& grid, const double* diag_plus_noise,
                         const dfpca_surface* cov, const double* mean, double* sigma2) {
  const i64 G = grid.G;
  cudaStream_t st = ctx->stream;
  if (cov->kind != DFPCA_SURFACE_COVARIANCE)
    fail(kConfig, "InvalidArgument", "estimate_sigma2 got surfaces of the wrong kind");
  const i64 rows = cov->rows >= 0 ? cov->rows : G;
  Transport* tr = ctx->transport && ctx->transport->world() > 1 ? ctx->transport.get() : nullptr;
  if (cov->n != rows * G || (rows != G && !tr))
    fail(kConfig, "InvalidArgument", "estimate_sigma2 surfaces must share one grid");
  ctx->begin_stage("sigma2");
  DevBuf<double> dpn(G), mu(G), gdiag(G), res(1);
  DFPCA_CUDA(cudaMemcpyAsync(dpn.get(), diag_plus_noise, sizeof(double) * G, cudaMemcpyHostToDevice, st));
  DFPCA_CUDA(cudaMemcpyAsync(mu.get(), mean, sizeof(double) * G, cudaMemcpyHostToDevice, st));
  DFPCA_CUDA(cudaMemsetAsync(gdiag.get(), 0, sizeof(double) * G, st));
  if (rows > 0)
    DFPCA_LAUNCH(ctx, k_cov_diagonal, grid_for(rows, 256), 256, 0, cov->values.get(), G, cov->row0, rows,
                 gdiag.get());
  if (tr) {  // every rank holds the diagonal of its rows; zeros elsewhere add exactly
    DevBuf<double> all(static_cast<std::size_t>(tr->world() * G));
    tr->all_gather(ctx, gdiag.get(), all.get(), G);
    std::vector<double> h(static_cast<std::size_t>(tr->world() * G)), d(static_cast<std::size_t>(G), 0.0);
    DFPCA_CUDA(cudaMemcpyAsync(h.data(), all.get(), sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
    DFPCA_CUDA(cudaStreamSynchronize(st));
    // pick each node's owner value (exactly one rank holds it)
    for (int r = 0; r < tr->world(); ++r)
      for (i64 f = 0; f < G; ++f)
        if (h[static_cast<std::size_t>(r * G + f)] != 0.0 || std::isnan(h[static_cast<std::size_t>(r * G + f)]))
          d[static_cast<std::size_t>(f)] = h[static_cast<std::size_t>(r * G + f)];
    DFPCA_CUDA(cudaMemcpyAsync(gdiag.get(), d.data(), sizeof(double) * G, cudaMemcpyHostToDevice, st));
  }
  DevBuf<std::uint8_t> mask;
  if (grid.has_mask) {
    mask.alloc(G);
    DFPCA_CUDA(cudaMemcpyAsync(mask.get(), grid.mask.data(), G, cudaMemcpyHostToDevice, st));
  }
  DFPCA_LAUNCH(ctx, k_sigma2, 1, 32, 0, dpn.get(), gdiag.get(), mu.get(), grid.has_mask ? mask.get() : nullptr, G,
               res.get());
  DFPCA_CUDA(cudaMemcpyAsync(sigma2, res.get(), sizeof(double), cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
  ctx->end_stage();
}

void run_scores(dfpca_context* ctx, const Grid& grid, i64 n, const i64* offsets, const double* coords,
                const double* values, const double* mean, i64 L, const double* eigenvalues,
                const double* eigenfunctions, double sigma2, int method, double* scores, int* sparse_warning,
                i64* bad_sample) {
  const i64 G = grid.G;
  const int d = grid.d;
  cudaStream_t st = ctx->stream;
  *bad_sample = -1;
  // integration_scores' sparse-sample warning (pace_scores leaves it unset)
  for (i64 i = 0; i < n; ++i)
    if (sparse_warning) sparse_warning[i] = method == 1 && (offsets[i + 1] - offsets[i]) * 4 < G ? 1 : 0;
  if (L == 0 || n == 0) return;
  const i64 n_obs = offsets[n];
  ctx->begin_stage("scores");
  DevBuf<double> axes;
  const DevGrid dg = upload_grid_axes(ctx, grid, axes);
  DevBuf<i64> d_off(static_cast<std::size_t>(n + 1));
  DevBuf<double> d_coords(static_cast<std::size_t>(std::max<i64>(1, n_obs * d)));
  DevBuf<double> d_values(static_cast<std::size_t>(std::max<i64>(1, n_obs)));
  DevBuf<double> d_mean(G), d_phi(static_cast<std::size_t>(L * G)), d_out(static_cast<std::size_t>(n * L));
  DFPCA_CUDA(cudaMemcpyAsync(d_off.get(), offsets, sizeof(i64) * (n + 1), cudaMemcpyHostToDevice, st));
  if (n_obs > 0) {
    DFPCA_CUDA(cudaMemcpyAsync(d_coords.get(), coords, sizeof(double) * n_obs * d, cudaMemcpyHostToDevice, st));
    DFPCA_CUDA(cudaMemcpyAsync(d_values.get(), values, sizeof(double) * n_obs, cudaMemcpyHostToDevice, st));
  }
  DFPCA_CUDA(cudaMemcpyAsync(d_mean.get(), mean, sizeof(double) * G, cudaMemcpyHostToDevice, st));
  DFPCA_CUDA(cudaMemcpyAsync(d_phi.get(), eigenfunctions, sizeof(double) * L * G, cudaMemcpyHostToDevice, st));
  if (method == 1) {
    DevBuf<double> mass(static_cast<std::size_t>(n * G)), wval(static_cast<std::size_t>(n * G));
    DevBuf<unsigned long long> bad(1);
    DFPCA_CUDA(cudaMemsetAsync(mass.get(), 0, mass.bytes(), st));
    DFPCA_CUDA(cudaMemsetAsync(wval.get(), 0, wval.bytes(), st));
    DFPCA_CUDA(cudaMemsetAsync(bad.get(), 0xff, sizeof(unsigned long long), st));
    DFPCA_LAUNCH(ctx, k_tent_grid, grid_for(n * 32, 256, 148ll * 64), 256, 0, dg, d_off.get(), n, d_coords.get(),
                 d_values.get(), mass.get(), wval.get(), bad.get());
    unsigned long long hb = ~0ull;
    DFPCA_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(hb), cudaMemcpyDeviceToHost, st));
    DFPCA_CUDA(cudaStreamSynchronize(st));
    if (hb != ~0ull) {
      const i64 j = static_cast<i64>(hb);
      *bad_sample = static_cast<i64>(std::upper_bound(offsets, offsets + n + 1, j) - offsets) - 1;
      fail(kConfig, "OutOfDomain", "observation outside the grid hull cannot be scored");
    }
    DevBuf<std::uint8_t> mask;
    if (grid.has_mask) {
      mask.alloc(G);
      DFPCA_CUDA(cudaMemcpyAsync(mask.get(), grid.mask.data(), G, cudaMemcpyHostToDevice, st));
    }
    DFPCA_LAUNCH(ctx, k_integration_scores, grid_for(n * L, 128, 148ll * 64), 128, 0, mass.get(), wval.get(),
                 d_mean.get(), d_phi.get(), grid.has_mask ? mask.get() : nullptr, G, n, L, grid.cell_volume(),
                 d_out.get());
  } else {
    // samples up to kPaceMaxObs observations: one shared-memory CTA each;
    // larger ones: one CTA each on a global-memory workspace, in batches
    i64 max_small = 0, max_big = 0;
    std::vector<i64> big;
    for (i64 i = 0; i < n; ++i) {
      const i64 c = offsets[i + 1] - offsets[i];
      if (c > kPaceMaxObs) {
        big.push_back(i);
        max_big = std::max(max_big, c);
      } else {
        max_small = std::max(max_small, c);
      }
    }
    DevBuf<double> lam(static_cast<std::size_t>(L));
    DFPCA_CUDA(cudaMemcpyAsync(lam.get(), eigenvalues, sizeof(double) * L, cudaMemcpyHostToDevice, st));
    DevBuf<int> status(static_cast<std::size_t>(n));
    PaceArgs a{};
    a.g = dg;
    a.offsets = d_off.get();
    a.coords = d_coords.get();
    a.values = d_values.get();
    a.mean = d_mean.get();
    a.phi = d_phi.get();
    a.lambda = lam.get();
    a.L = L;
    a.n_samples = n;
    a.noise = std::max(sigma2, kSigmaFloorRel * eigenvalues[0]);
    a.out = d_out.get();
    a.status = status.get();
    const std::size_t smem = sizeof(double) * (kPaceMaxObs * (L + 1) + max_small * max_small);
    if (smem > 200 * 1024)
      fail(kConfig, "InvalidArgument", "too many components x observations for the on-chip PACE design");
    allow_smem(k_pace<false>, smem);
    DFPCA_LAUNCH(ctx, k_pace<false>, static_cast<unsigned>(n), 128, smem, a, nullptr, nullptr, nullptr, i64{0});
    if (!big.empty()) {
      const i64 per = max_big * (L + 2) + max_big * max_big;  // doubles per CTA
      const i64 batch = std::max<i64>(1, std::min<i64>(static_cast<i64>(big.size()), (i64{1} << 28) / per));
      DevBuf<double> ws(static_cast<std::size_t>(batch * per));
      DevBuf<int> iws(static_cast<std::size_t>(batch * 3 * max_big));
      DevBuf<i64> list(big.size());
      DFPCA_CUDA(cudaMemcpyAsync(list.get(), big.data(), sizeof(i64) * big.size(), cudaMemcpyHostToDevice, st));
      for (i64 b0 = 0; b0 < static_cast<i64>(big.size()); b0 += batch) {
        const i64 nb = std::min<i64>(batch, static_cast<i64>(big.size()) - b0);
        DFPCA_LAUNCH(ctx, k_pace<true>, static_cast<unsigned>(nb), 256, 0, a, list.get() + b0, ws.get(), iws.get(),
                     max_big);
      }
    }
    std::vector<int> hs(static_cast<std::size_t>(n));
    DFPCA_CUDA(cudaMemcpyAsync(hs.data(), status.get(), sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    DFPCA_CUDA(cudaStreamSynchronize(st));
    for (i64 i = 0; i < n; ++i) {
      if (hs[static_cast<std::size_t>(i)] == 2) {
        *bad_sample = i;
        fail(kConfig, "OutOfDomain", "coordinate outside the grid hull");
      }
      if (hs[static_cast<std::size_t>(i)] == 1) {
        *bad_sample = i;
        fail(kNumeric, "SingularCovariance",
             "observation covariance is numerically singular even after the noise floor");
      }
    }
  }
  DFPCA_CUDA(cudaMemcpyAsync(scores, d_out.get(), sizeof(double) * n * L, cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
  ctx->end_stage();
}

void run_reconstruct(dfpca_context* ctx, const Grid& grid, const double* mean, i64 L, const double* eigenfunctions,
                     i64 n, const double* scores, double* out) {
  const i64 G = grid.G;
  cudaStream_t st = ctx->stream;
  ctx->begin_stage("reconstruct");
  DevBuf<double> d_mean(G), d_phi(static_cast<std::size_t>(std::max<i64>(1, L * G))),
      d_s(static_cast<std::size_t>(std::max<i64>(1, n * L))), d_out(static_cast<std::size_t>(std::max<i64>(1, n * G)));
  DFPCA_CUDA(cudaMemcpyAsync(d_mean.get(), mean, sizeof(double) * G, cudaMemcpyHostToDevice, st));
  if (L > 0) {
    DFPCA_CUDA(cudaMemcpyAsync(d_phi.get(), eigenfunctions, sizeof(double) * L * G, cudaMemcpyHostToDevice, st));
    DFPCA_CUDA(cudaMemcpyAsync(d_s.get(), scores, sizeof(double) * n * L, cudaMemcpyHostToDevice, st));
  }
  if (n > 0)
    DFPCA_LAUNCH(ctx, k_reconstruct, grid_for(n * G, 256, 148ll * 32), 256, 0, d_mean.get(), d_phi.get(), G, L,
                 d_s.get(), n, d_out.get());
  DFPCA_CUDA(cudaMemcpyAsync(out, d_out.get(), sizeof(double) * n * G, cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
  ctx->end_stage();
}

}  // namespace dfpca_gpu
