// the leave-one-observation-out CV objective of the
// bandwidth search (reference bandwidth.hpp:56-163, CvObjective) on the GPU.
//
// Every evaluation unit (an observation for the mean / squares targets, an
// ordered raw pair for the covariance target) needs one direct local-linear
// fit over the whole dataset at its own location (smoother.hpp:376-407,
// gather_mean_equations / gather_pair_equations :83-160) with the ridge pinned
// at 0 and the first diagonal entry of the inverse (local_fit.hpp:63-100).
// Units are independent, so the evaluation is a batch:
//   * mean / squares: CTA = 32 units x one chunk of observations, the chunk
//     staged in shared memory tile by tile and shared by the 32 units; every
//     thread accumulates its unit's moment sums over a strided part of the
//     tile; partial sums per (chunk, unit) are added in chunk order;
//   * covariance: thread = (unit, sample): the sample's in-window observations
//     for s and t, then every ordered pair j != l (the reference's loops);
//   * one thread per unit then assembles the normal equations, replays
//     Eigen's pivoted LDLT with the pinned ridge, solves for b0 and for
//     (A^-1)_00, and forms the unit's squared leave-one-out residual.
// The host adds the residuals in unit order (the reference's running sum).
// Moment sums are reassociated (partial sums), so the bar is a relative
// tolerance on the score, not bits.
#include <algorithm>
#include <cmath>
#include <random>
#include <string>
#include <vector>

#include "common.cuh"
#include "solve.cuh"

namespace dfpca_gpu {
namespace {

constexpr int kUnitsPerCta = 32;
constexpr int kGroups = 8;  // warps per CTA, each a strided share of the tile
constexpr int kObsTile = 256;
constexpr int kPairMaxObs = 64;  // covariance target: observations per sample

__device__ inline double kernel_eval_dev(const double* u, const double* h, int dim) {
  double k = 1.0;
  for (int a = 0; a < dim; ++a) {
    const double z = __ddiv_rn(u[a], h[a]);
    const double t = __dsub_rn(1.0, __dmul_rn(z, z));
    if (!(t > 0.0)) return 0.0;
    k = __dmul_rn(k, __ddiv_rn(__dmul_rn(0.75, t), h[a]));
  }
  return k;
}

// accumulate_moments (local_fit.hpp:102-115) for a p-variate covariate u
template <int P>
__device__ __forceinline__ void accumulate(const double (&u)[P], double w, double wy, double (&S)[1 + P + P * (P + 1) / 2],
                                           double (&T)[1 + P]) {
  S[0] += w;
  T[0] += wy;
  int q = 1 + P;
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const double wu = w * u[k];
    S[1 + k] += wu;
    T[1 + k] += wy * u[k];
#pragma unroll
    for (int l = k; l < P; ++l) S[q++] += wu * u[l];
  }
}

struct CvData {
  int dim;
  const i64* offsets;
  const double* coords;  // n_obs * dim
  const double* values;
  const double* obs_w;   // 1 / N_i of the observation's sample
  i64 n_samples, n_obs;
};

// ---- mean / squares target ----
template <int D>
__global__ void __launch_bounds__(kUnitsPerCta * kGroups)
    k_cv_mean_partials(CvData data, const double* __restrict__ tgt, int n_units, const double* __restrict__ hh,
                       int squares, i64 chunk_len, double* __restrict__ partial) {
  pdl_wait();
  constexpr int NM = 1 + D + D * (D + 1) / 2, NL = 1 + D;
  __shared__ double sx[kObsTile][D];
  __shared__ double sy[kObsTile], sw[kObsTile];
  __shared__ double red[kGroups][kUnitsPerCta][NM + NL];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int unit = blockIdx.x * kUnitsPerCta + lane;
  const bool live = unit < n_units;
  double h[D], t[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    h[k] = hh[k];
    t[k] = live ? tgt[static_cast<i64>(unit) * D + k] : 0.0;
  }
  double S[NM], T[NL];
#pragma unroll
  for (int i = 0; i < NM; ++i) S[i] = 0.0;
#pragma unroll
  for (int i = 0; i < NL; ++i) T[i] = 0.0;
  const i64 o0 = static_cast<i64>(blockIdx.y) * chunk_len;
  const i64 o1 = o0 + chunk_len < data.n_obs ? o0 + chunk_len : data.n_obs;
  for (i64 b = o0; b < o1; b += kObsTile) {
    const int cnt = static_cast<int>(o1 - b < kObsTile ? o1 - b : kObsTile);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
#pragma unroll
      for (int k = 0; k < D; ++k) sx[e][k] = data.coords[(b + e) * D + k];
      const double y = data.values[b + e];
      sy[e] = squares ? y * y : y;
      sw[e] = data.obs_w[b + e];
    }
    __syncthreads();
    if (!live) continue;
    for (int e = grp; e < cnt; e += kGroups) {
      double u[D];
#pragma unroll
      for (int k = 0; k < D; ++k) u[k] = t[k] - sx[e][k];
      const double kw = kernel_eval_dev(u, h, D);
      if (kw == 0.0) continue;
      const double w = sw[e] * kw;
      accumulate<D>(u, w, w * sy[e], S, T);
    }
  }
  if (live) {
#pragma unroll
    for (int i = 0; i < NM; ++i) red[grp][lane][i] = S[i];
#pragma unroll
    for (int i = 0; i < NL; ++i) red[grp][lane][NM + i] = T[i];
  }
  __syncthreads();
  if (grp == 0 && live) {
    double* out = partial + (static_cast<i64>(blockIdx.y) * n_units + unit) * (NM + NL);
    for (int i = 0; i < NM + NL; ++i) {
      double s = 0.0;
      for (int g = 0; g < kGroups; ++g) s += red[g][lane][i];
      out[i] = s;
    }
  }
}

// ---- covariance target: thread = (unit, sample) ----
template <int D>
__global__ void __launch_bounds__(kUnitsPerCta * kGroups)
    k_cv_pair_partials(CvData data, const double* __restrict__ tgt, int n_units, const double* __restrict__ hh,
                       i64 chunk_len, double* __restrict__ partial) {
  pdl_wait();
  constexpr int P = 2 * D;
  constexpr int NM = 1 + P + P * (P + 1) / 2, NL = 1 + P;
  extern __shared__ double red_dyn[];  // [kGroups][kUnitsPerCta][NM + NL]
  auto red = reinterpret_cast<double (*)[kUnitsPerCta][NM + NL]>(red_dyn);
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int unit = blockIdx.x * kUnitsPerCta + lane;
  const bool live = unit < n_units;
  double h[D], ts[D], tt[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    h[k] = hh[k];
    ts[k] = live ? tgt[static_cast<i64>(unit) * P + k] : 0.0;
    tt[k] = live ? tgt[static_cast<i64>(unit) * P + D + k] : 0.0;
  }
  double S[NM], T[NL];
#pragma unroll
  for (int i = 0; i < NM; ++i) S[i] = 0.0;
#pragma unroll
  for (int i = 0; i < NL; ++i) T[i] = 0.0;
  const i64 s0 = static_cast<i64>(blockIdx.y) * chunk_len;
  const i64 s1 = s0 + chunk_len < data.n_samples ? s0 + chunk_len : data.n_samples;
  for (i64 i = s0 + grp; live && i < s1; i += kGroups) {
    const i64 b = data.offsets[i], n = data.offsets[i + 1] - b;
    if (n < 2) continue;
    const double pw = 1.0 / (static_cast<double>(n) * static_cast<double>(n - 1));
    int in_s[kPairMaxObs], in_t[kPairMaxObs];
    double kw_s[kPairMaxObs], kw_t[kPairMaxObs];
    int ns = 0, nt = 0;
    for (i64 j = 0; j < n; ++j) {
      const double* x = data.coords + (b + j) * D;
      double u[D];
#pragma unroll
      for (int k = 0; k < D; ++k) u[k] = ts[k] - x[k];
      const double ks = kernel_eval_dev(u, h, D);
      if (ks != 0.0) {
        in_s[ns] = static_cast<int>(j);
        kw_s[ns++] = ks;
      }
#pragma unroll
      for (int k = 0; k < D; ++k) u[k] = tt[k] - x[k];
      const double kt = kernel_eval_dev(u, h, D);
      if (kt != 0.0) {
        in_t[nt] = static_cast<int>(j);
        kw_t[nt++] = kt;
      }
    }
    for (int a = 0; a < ns; ++a) {
      const i64 j = in_s[a];
      const double* xj = data.coords + (b + j) * D;
      const double yj = data.values[b + j];
      for (int c = 0; c < nt; ++c) {
        const i64 l = in_t[c];
        if (l == j) continue;  // raw products exclude the diagonal
        const double* xl = data.coords + (b + l) * D;
        double u[P];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          u[k] = ts[k] - xj[k];
          u[D + k] = tt[k] - xl[k];
        }
        const double w = pw * kw_s[a] * kw_t[c];
        accumulate<P>(u, w, w * yj * data.values[b + l], S, T);
      }
    }
  }
  if (live) {
#pragma unroll
    for (int i = 0; i < NM; ++i) red[grp][lane][i] = S[i];
#pragma unroll
    for (int i = 0; i < NL; ++i) red[grp][lane][NM + i] = T[i];
  }
  __syncthreads();
  if (grp == 0 && live) {
    double* out = partial + (static_cast<i64>(blockIdx.y) * n_units + unit) * (NM + NL);
    for (int i = 0; i < NM + NL; ++i) {
      double s = 0.0;
      for (int g = 0; g < kGroups; ++g) s += red[g][lane][i];
      out[i] = s;
    }
  }
}

// ---- per unit: chunk sums, solve_local(fixed_ridge = 0, want_inv00), term ----
// local_fit.hpp:63-100 with the ridge pinned; Eigen's pivoted LDLT replayed
// (solve.cuh) for b0 and (A^-1)_00 = solve(e1)(0).
template <int N>
__device__ inline int cv_solve(const double* S, const double* T, double& b0, double& inv00) {
  constexpr int p = N - 1;
  const double s0 = S[0];
  if (!(s0 > 0.0)) return kFitEmpty;
  double A[N][N];
  A[0][0] = S[0];
  double rhs[N];
  rhs[0] = T[0];
  for (int k = 0; k < p; ++k) {
    A[0][k + 1] = A[k + 1][0] = S[1 + k];
    rhs[k + 1] = T[1 + k];
    for (int l = k; l < p; ++l) A[k + 1][l + 1] = A[l + 1][k + 1] = S[quad_index(p, k, l)];
  }
  int trans[N];
  double invD[N];
  for (int k = 0; k < N; ++k) {
    trans[k] = k;
    invD[k] = 0.0;
  }
  bool ret = true, fzp = false, broke = false;
  ldlt_steps<N>(A, trans, invD, ret, fzp, broke, std::make_integer_sequence<int, N>{});
  bool ok = ret;
  if (ok) {
    double dmax = 0.0, dmin = 1.0 / 0.0, dsmin = 1.0 / 0.0;
    for (int i = 0; i < N; ++i) {
      const double a = fabs(A[i][i]);
      dmax = a > dmax ? a : dmax;
      dmin = a < dmin ? a : dmin;
      dsmin = A[i][i] < dsmin ? A[i][i] : dsmin;
    }
    ok = dmax > 0.0 && dsmin > 0.0 && dmin > 1e-8 * dmax;
  }
  if (ok) {
    double x[2][N];
    for (int i = 0; i < N; ++i) {
      x[0][i] = rhs[i];
      x[1][i] = i == 0 ? 1.0 : 0.0;
    }
    for (int v = 0; v < 2; ++v) {
      for (int k = 0; k < N; ++k) {
        const double tmp = x[v][k];
        x[v][k] = x[v][trans[k]];
        x[v][trans[k]] = tmp;
      }
      for (int j = 0; j < N; ++j)
        for (int i = j + 1; i < N; ++i) x[v][i] -= A[i][j] * x[v][j];
      for (int i = 0; i < N; ++i) x[v][i] = fabs(A[i][i]) > 2.2250738585072014e-308 ? x[v][i] * invD[i] : 0.0;
      for (int j = N - 1; j >= 0; --j)
        for (int i = 0; i < j; ++i) x[v][i] -= A[j][i] * x[v][j];
      for (int k = N - 1; k >= 0; --k) {
        const double tmp = x[v][k];
        x[v][k] = x[v][trans[k]];
        x[v][trans[k]] = tmp;
      }
    }
    bool finite = true;
    for (int i = 0; i < N; ++i) finite = finite && isfinite(x[0][i]);
    if (finite) {
      b0 = x[0][0];
      inv00 = x[1][0];
      return kFitOk;
    }
  }
  b0 = T[0] / s0;
  inv00 = 1.0 / s0;
  return kFitLocalConstant;
}

struct UnitInfo {
  double y;       // response of the unit (y, y^2 or y_j y_l)
  double weight;  // 1 / N_i or 1 / (N_i (N_i - 1))
};

template <int N>
__global__ void k_cv_finish(const double* __restrict__ partial, int n_chunks, int n_units,
                            const UnitInfo* __restrict__ info, double kernel0, double* __restrict__ term,
                            int* __restrict__ flag) {
  pdl_wait();
  constexpr int p = N - 1, NM = 1 + p + p * (p + 1) / 2, NL = 1 + p;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n_units) return;
  double S[NM], T[NL];
  for (int i = 0; i < NM; ++i) S[i] = 0.0;
  for (int i = 0; i < NL; ++i) T[i] = 0.0;
  for (int c = 0; c < n_chunks; ++c) {
    const double* pp = partial + (static_cast<i64>(c) * n_units + u) * (NM + NL);
    for (int i = 0; i < NM; ++i) S[i] += pp[i];
    for (int i = 0; i < NL; ++i) T[i] += pp[NM + i];
  }
  double b0 = 0.0, inv00 = 0.0;
  const int st = cv_solve<N>(S, T, b0, inv00);
  // CvObjective::operator() (bandwidth.hpp:91-113)
  if (st == kFitEmpty) {
    flag[u] = 1;
    term[u] = 0.0;
    return;
  }
  const double self = info[u].weight * kernel0 * inv00;
  const double denom = 1.0 - self;
  if (denom < 1e-6) {
    flag[u] = 2;
    term[u] = 0.0;
    return;
  }
  const double r = (info[u].y - b0) / (denom > 1e-8 ? denom : 1e-8);
  flag[u] = 0;
  term[u] = r * r;
}

}  // namespace


dfpca_dataset* upload_dataset(dfpca_context* ctx, int dim, i64 n, const i64* offsets, const double* coords,
                              const double* values) {
  auto ds = std::make_unique<dfpca_dataset>();
  ds->dim = dim;
  ds->n_samples = n;
  ds->n_obs = offsets[n];
  ds->offsets_h.assign(offsets, offsets + n + 1);
  ds->coords_h.assign(coords, coords + ds->n_obs * dim);
  ds->values_h.assign(values, values + ds->n_obs);
  std::vector<double> w(static_cast<std::size_t>(std::max<i64>(1, ds->n_obs)));
  for (i64 i = 0; i < n; ++i) {
    const i64 cnt = offsets[i + 1] - offsets[i];
    for (i64 j = offsets[i]; j < offsets[i + 1]; ++j) w[static_cast<std::size_t>(j)] = 1.0 / static_cast<double>(cnt);
  }
  cudaStream_t st = ctx->stream;
  ds->offsets.alloc(static_cast<std::size_t>(n + 1));
  ds->coords.alloc(static_cast<std::size_t>(std::max<i64>(1, ds->n_obs * dim)));
  ds->values.alloc(static_cast<std::size_t>(std::max<i64>(1, ds->n_obs)));
  ds->obs_w.alloc(static_cast<std::size_t>(std::max<i64>(1, ds->n_obs)));
  DFPCA_CUDA(cudaMemcpyAsync(ds->offsets.get(), offsets, sizeof(i64) * (n + 1), cudaMemcpyHostToDevice, st));
  if (ds->n_obs > 0) {
    DFPCA_CUDA(cudaMemcpyAsync(ds->coords.get(), coords, sizeof(double) * ds->n_obs * dim, cudaMemcpyHostToDevice, st));
    DFPCA_CUDA(cudaMemcpyAsync(ds->values.get(), values, sizeof(double) * ds->n_obs, cudaMemcpyHostToDevice, st));
    DFPCA_CUDA(cudaMemcpyAsync(ds->obs_w.get(), w.data(), sizeof(double) * ds->n_obs, cudaMemcpyHostToDevice, st));
  }
  DFPCA_CUDA(cudaStreamSynchronize(st));
  return ds.release();
}

// CvObjective::enumerate_units (bandwidth.hpp:118-140): every observation
// (mean, squares) or ordered pair j != l (covariance), then a seeded partial
// Fisher-Yates keeps max_units of them (RandomStream, rng.hpp).
std::vector<i64> cv_units(i64 n_samples, const i64* offsets, int target, i64 max_units, std::uint64_t seed) {
  std::vector<i64> units;  // (sample, j, l) triples
  for (i64 i = 0; i < n_samples; ++i) {
    const i64 n = offsets[i + 1] - offsets[i];
    if (target == 1) {
      if (n < 2) continue;
      for (i64 j = 0; j < n; ++j)
        for (i64 l = 0; l < n; ++l)
          if (l != j) units.insert(units.end(), {i, j, l});
    } else {
      for (i64 j = 0; j < n; ++j) units.insert(units.end(), {i, j, 0});
    }
  }
  const i64 total = static_cast<i64>(units.size() / 3);
  if (total == 0) fail(kConfig, "InvalidArgument", "cross-validation needs at least one evaluation unit");
  if (total > max_units) {
    auto splitmix = [](std::uint64_t x) {
      x += 0x9e3779b97f4a7c15ULL;
      x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
      x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
      return x ^ (x >> 31);
    };
    std::mt19937_64 eng(splitmix(seed));
    for (i64 j = 0; j < max_units; ++j) {
      const double uni = (static_cast<double>(eng() >> 11) + 0.5) * 0x1.0p-53;
      const i64 pick = j + static_cast<i64>(uni * static_cast<double>(total - j));
      const i64 q = std::min(pick, total - 1);
      for (int c = 0; c < 3; ++c) std::swap(units[static_cast<std::size_t>(3 * j + c)], units[static_cast<std::size_t>(3 * q + c)]);
    }
    units.resize(static_cast<std::size_t>(3 * max_units));
  }
  return units;
}

template <int D>
static void cv_launch(dfpca_context* ctx, const dfpca_dataset* ds, int target, int n_units, const double* d_tgt,
                      const double* d_h, double* d_partial, int n_chunks, i64 chunk_len) {
  const CvData data{ds->dim, ds->offsets.get(), ds->coords.get(), ds->values.get(), ds->obs_w.get(), ds->n_samples,
                    ds->n_obs};
  const dim3 grid(static_cast<unsigned>((n_units + kUnitsPerCta - 1) / kUnitsPerCta), static_cast<unsigned>(n_chunks));
  if (target == 1) {
    constexpr int P = 2 * D;
    const std::size_t smem = sizeof(double) * kGroups * kUnitsPerCta * ((1 + P + P * (P + 1) / 2) + (1 + P));
    allow_smem(k_cv_pair_partials<D>, smem);
    DFPCA_LAUNCH(ctx, k_cv_pair_partials<D>, grid, kUnitsPerCta * kGroups, smem, data, d_tgt, n_units, d_h,
                 chunk_len, d_partial);
  } else {
    DFPCA_LAUNCH(ctx, k_cv_mean_partials<D>, grid, kUnitsPerCta * kGroups, 0, data, d_tgt, n_units, d_h,
                 target == 2 ? 1 : 0, chunk_len, d_partial);
  }
}

template <int N>
static void cv_finish_launch(dfpca_context* ctx, const double* d_partial, int n_chunks, int n_units,
                             const UnitInfo* d_info, double kernel0, double* d_term, int* d_flag) {
  DFPCA_LAUNCH(ctx, k_cv_finish<N>, static_cast<unsigned>((n_units + 127) / 128), 128, 0, d_partial, n_chunks,
               n_units, d_info, kernel0, d_term, d_flag);
}

// CvObjective::operator() (bandwidth.hpp:74-115) over the given units.
double run_cv_objective(dfpca_context* ctx, const dfpca_dataset* ds, int target, i64 n_units_l, const i64* units,
                        const double* h, i64* used_out) {
  const int d = ds->dim;
  const int n_units = static_cast<int>(n_units_l);
  const int p = target == 1 ? 2 * d : d;
  cudaStream_t st = ctx->stream;
  ctx->begin_stage("cv");
  // unit targets, responses and weights (host, from the dataset copy)
  std::vector<double> tgt(static_cast<std::size_t>(n_units) * p);
  std::vector<UnitInfo> info(static_cast<std::size_t>(n_units));
  for (int u = 0; u < n_units; ++u) {
    const i64 i = units[3 * u], j = units[3 * u + 1], l = units[3 * u + 2];
    const i64 b = ds->offsets_h[static_cast<std::size_t>(i)];
    const i64 n = ds->offsets_h[static_cast<std::size_t>(i) + 1] - b;
    if (i < 0 || i >= ds->n_samples || j < 0 || j >= n || (target == 1 && (l < 0 || l >= n || l == j)))
      fail(kConfig, "InvalidArgument", "cross-validation unit out of range");
    for (int k = 0; k < d; ++k) tgt[static_cast<std::size_t>(u) * p + k] = ds->coords_h[static_cast<std::size_t>((b + j) * d + k)];
    const double yj = ds->values_h[static_cast<std::size_t>(b + j)];
    if (target == 1) {
      for (int k = 0; k < d; ++k)
        tgt[static_cast<std::size_t>(u) * p + d + k] = ds->coords_h[static_cast<std::size_t>((b + l) * d + k)];
      info[static_cast<std::size_t>(u)] = {yj * ds->values_h[static_cast<std::size_t>(b + l)],
                                           1.0 / (static_cast<double>(n) * (static_cast<double>(n) - 1.0))};
    } else {
      info[static_cast<std::size_t>(u)] = {target == 2 ? yj * yj : yj, 1.0 / static_cast<double>(n)};
    }
  }
  if (target == 1)
    for (i64 i = 0; i < ds->n_samples; ++i)
      if (ds->offsets_h[static_cast<std::size_t>(i) + 1] - ds->offsets_h[static_cast<std::size_t>(i)] > kPairMaxObs)
        fail(kConfig, "InvalidArgument",
             "covariance-target cross-validation on the GPU takes up to " + std::to_string(kPairMaxObs) +
                 " observations per sample");
  double k0 = 1.0;
  for (int k = 0; k < d; ++k) k0 *= kernel_axis_value(0.0, h[k]);
  const double kernel0 = target == 1 ? k0 * k0 : k0;
  // chunks: enough CTAs to cover the SMs a few times
  const i64 items = target == 1 ? ds->n_samples : ds->n_obs;
  const int unit_ctas = (n_units + kUnitsPerCta - 1) / kUnitsPerCta;
  int n_chunks = static_cast<int>(std::max<i64>(1, std::min<i64>(items / 64 + 1, (4 * ctx->sm_count + unit_ctas - 1) / unit_ctas)));
  const i64 chunk_len = (items + n_chunks - 1) / n_chunks;
  n_chunks = static_cast<int>(std::max<i64>(1, (items + chunk_len - 1) / std::max<i64>(chunk_len, 1)));
  const int nmnl = (1 + p + p * (p + 1) / 2) + (1 + p);
  DevBuf<double> d_tgt(tgt.size()), d_h(static_cast<std::size_t>(d)),
      d_partial(static_cast<std::size_t>(n_chunks) * n_units * nmnl), d_term(static_cast<std::size_t>(n_units));
  DevBuf<UnitInfo> d_info(info.size());
  DevBuf<int> d_flag(static_cast<std::size_t>(n_units));
  DFPCA_CUDA(cudaMemcpyAsync(d_tgt.get(), tgt.data(), sizeof(double) * tgt.size(), cudaMemcpyHostToDevice, st));
  DFPCA_CUDA(cudaMemcpyAsync(d_h.get(), h, sizeof(double) * d, cudaMemcpyHostToDevice, st));
  DFPCA_CUDA(cudaMemcpyAsync(d_info.get(), info.data(), sizeof(UnitInfo) * info.size(), cudaMemcpyHostToDevice, st));
  DFPCA_CUDA(cudaMemsetAsync(d_partial.get(), 0, d_partial.bytes(), st));
  switch (d) {
    case 1: cv_launch<1>(ctx, ds, target, n_units, d_tgt.get(), d_h.get(), d_partial.get(), n_chunks, chunk_len); break;
    case 2: cv_launch<2>(ctx, ds, target, n_units, d_tgt.get(), d_h.get(), d_partial.get(), n_chunks, chunk_len); break;
    default: cv_launch<3>(ctx, ds, target, n_units, d_tgt.get(), d_h.get(), d_partial.get(), n_chunks, chunk_len); break;
  }
  switch (p + 1) {
    case 2: cv_finish_launch<2>(ctx, d_partial.get(), n_chunks, n_units, d_info.get(), kernel0, d_term.get(), d_flag.get()); break;
    case 3: cv_finish_launch<3>(ctx, d_partial.get(), n_chunks, n_units, d_info.get(), kernel0, d_term.get(), d_flag.get()); break;
    case 4: cv_finish_launch<4>(ctx, d_partial.get(), n_chunks, n_units, d_info.get(), kernel0, d_term.get(), d_flag.get()); break;
    case 5: cv_finish_launch<5>(ctx, d_partial.get(), n_chunks, n_units, d_info.get(), kernel0, d_term.get(), d_flag.get()); break;
    default: cv_finish_launch<7>(ctx, d_partial.get(), n_chunks, n_units, d_info.get(), kernel0, d_term.get(), d_flag.get()); break;
  }
  std::vector<double> term(static_cast<std::size_t>(n_units));
  std::vector<int> flag(static_cast<std::size_t>(n_units));
  DFPCA_CUDA(cudaMemcpyAsync(term.data(), d_term.get(), sizeof(double) * n_units, cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaMemcpyAsync(flag.data(), d_flag.get(), sizeof(int) * n_units, cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
  ctx->end_stage();
  double acc = 0.0;
  i64 used = 0;
  for (int u = 0; u < n_units; ++u)
    if (flag[static_cast<std::size_t>(u)] == 0) {
      acc += term[static_cast<std::size_t>(u)];
      ++used;
    }
  if (used_out) *used_out = used;
  if (used == 0)
    fail(kNumeric, "BandwidthTooSmall",
         "no cross-validation unit has neighbors at bandwidth " + std::to_string(h[0]) +
             "; every window degenerates to its own observation");
  return acc / static_cast<double>(used);
}

}  // namespace dfpca_gpu
