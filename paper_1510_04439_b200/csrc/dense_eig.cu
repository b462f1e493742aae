// dense_eig (eigensolve.hpp:205-228) on the device without a library
// eigensolver.  The reference decomposes the whole M x M matrix (LAPACK
// dsyevd through Eigen) and keeps the leading L_max pairs above the
// 1e-12 lambda_1 cut; this computes exactly those pairs and the sum of all
// eigenvalues above the cut (the reference's total variance).
//
//   1. Householder tridiagonalization T = Q^T A Q (dsytd2's reflectors:
//      x = A[k][k+1..], beta = -sign(alpha) ||x||, tau = (beta - alpha) /
//      beta, v = x / (alpha - beta), p = tau A22 v, K = tau / 2 p^T v,
//      w = p - K v, A22 -= v w^T + w v^T) in ONE cooperative kernel with one
//      grid barrier per column: after the barrier every CTA forms w_k, the
//      updated row k + 1 and from it v_{k+1} in shared memory (redundantly,
//      in the same operation order, so all CTAs hold identical values), then
//      one pass over the trailing rows both applies the rank-2 update and
//      takes the dot products with v_{k+1} (p_{k+1}): the trailing matrix is
//      read and written once per column.  Entry (i, j) subtracts
//      (v_i w_j) + (w_i v_j), the (j, i) entry's terms in swapped order, so
//      A22 stays exactly symmetric.
//   2. Eigenvalues of T by 32-point multisection of Sturm counts, one warp
//      per eigenvalue: the leading L_max, then whichever side of the cut is
//      smaller (the sum above the cut is the trace minus the sum below).
//   3. Eigenvectors of T by inverse iteration (LU with partial pivoting,
//      three solves; one warp per eigenvalue, all in parallel), then
//      Gram-Schmidt (two passes) inside clusters of gaps below 1e-3 ||T||
//      (LAPACK dstein's ORTOL).
//   4. Back-transformation x = H_0 ... H_{M-3} y, one CTA per vector.
//   5. The reference's finalization (eig.cu finish_eigensystem).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace dfpca_gpu {
namespace {

constexpr int kTrdThreads = 1024;
constexpr int kTrdWarps = kTrdThreads / 32;
constexpr double kEps = 2.220446049250313e-16;

__device__ inline double dw_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}

// Deterministic block sum (fixed mapping of terms to threads): every CTA
// that sums the same values gets the same result.  One barrier: the callers
// rotate three `red` buffers, so a buffer is rewritten only after two more
// barriers, when every thread has read it.
__device__ inline double trd_block_sum(double v, double* red) {
  v = dw_sum(v);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (lane == 0) red[wib] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < kTrdWarps; ++w) t += red[w];
  return t;
}

struct Reflector {
  double tau, beta, scale;
};

__device__ inline Reflector make_reflector(double alpha, double sigma) {
  Reflector r{0.0, alpha, 0.0};
  if (sigma != 0.0) {
    r.beta = -copysign(sqrt(fma(alpha, alpha, sigma)), alpha);
    r.tau = (r.beta - alpha) / r.beta;
    r.scale = 1.0 / (alpha - r.beta);
  }
  return r;
}

// One pass over the trailing rows c0 .. c0 + mn - 1 (columns c0 ..): with
// kUpdate the rank-2 update by the previous step's v, w (indexed from c0 - 1),
// and in every case p = tau A v_new and this CTA's share of p^T v_new.  CTA b
// owns a contiguous block of rows; when the block has fewer rows than warps
// each row is split into column segments (summed in a fixed order), so every
// warp streams about the same number of bytes.
template <bool kUpdate>
__device__ inline void trd_rows(double* __restrict__ A, int n, int c0, int mn, const double* sv_old,
                                const double* sw, const double* snv, double tau, double* __restrict__ pn,
                                double* __restrict__ partn, double* red, double* segsum) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int Rb = (mn + gridDim.x - 1) / gridDim.x;
  const int rb0 = blockIdx.x * Rb;
  const int rows = max(0, min(Rb, mn - rb0));
  const int S = max(1, kTrdWarps / max(Rb, 1));
  const int Lseg = ((mn + S - 1) / S + 31) / 32 * 32;
  constexpr int U = 8;  // loads in flight per lane
  double contrib = 0.0;
  auto row_seg = [&](int r, int cb, int ce) {
    double* ri = A + static_cast<i64>(c0 + r) * n + c0;
    double vi = 0.0, wi = 0.0;
    if (kUpdate) {
      vi = sv_old[1 + r];
      wi = sw[1 + r];
    }
    double acc = 0.0;
    int j = cb + lane;
    for (; j + 32 * (U - 1) < ce; j += 32 * U) {
      double a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) a[u] = ri[j + 32 * u];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int jj = j + 32 * u;
        double nv = a[u];
        if (kUpdate) {
          nv = nv - (__dmul_rn(vi, sw[1 + jj]) + __dmul_rn(wi, sv_old[1 + jj]));
          ri[jj] = nv;
        }
        acc = fma(nv, snv[jj], acc);
      }
    }
    for (; j < ce; j += 32) {
      double nv = ri[j];
      if (kUpdate) {
        nv = nv - (__dmul_rn(vi, sw[1 + j]) + __dmul_rn(wi, sv_old[1 + j]));
        ri[j] = nv;
      }
      acc = fma(nv, snv[j], acc);
    }
    return dw_sum(acc);
  };
  if (S == 1) {
    for (int rr = wib; rr < rows; rr += kTrdWarps) {
      const int r = rb0 + rr;
      const double pr = tau * row_seg(r, 0, mn);
      if (lane == 0) {
        pn[r] = pr;
        contrib = fma(pr, snv[r], contrib);
      }
    }
  } else {
    const int rr = wib / S, seg = wib % S;
    double part = 0.0;
    if (rr < rows) part = row_seg(rb0 + rr, seg * Lseg, min(mn, (seg + 1) * Lseg));
    if (lane == 0) segsum[wib] = part;
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < rows) {
      double t = 0.0;
      for (int q = 0; q < S; ++q) t += segsum[threadIdx.x * S + q];
      const int r = rb0 + threadIdx.x;
      const double pr = tau * t;
      pn[r] = pr;
      contrib = pr * snv[r];
    }
  }
  const double pv = trd_block_sum(contrib, red);
  if (threadIdx.x == 0) partn[blockIdx.x] = pv;
}

constexpr int kTrdMaxPer = 4;  // row elements per thread prefetched into registers (n <= 4096 in one round trip)

// A (n x n, row-major, symmetric) is overwritten.  Outputs d[n], e[n-1],
// tau[n-2], V[n-2][n] (row k holds v_k at columns k+1.., v_k[0] = 1).
// Scratch: p[2][n], part[2][gridDim].
__global__ void __launch_bounds__(kTrdThreads, 1)
    k_trd(double* __restrict__ A, int n, double* __restrict__ d, double* __restrict__ e, double* __restrict__ taus,
          double* __restrict__ V, double* __restrict__ p, double* __restrict__ part) {
  pdl_wait();
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sh[];  // v [n], w [n], next row [n], v_next [n]
  double* sv = sh;
  double* sw = sh + n;
  double* srow = sh + 2 * n;
  double* snv = sh + 3 * n;
  __shared__ double red[3][kTrdWarps];  // K, sigma, p^T v sums (rotated: one barrier each)
  __shared__ double segsum[kTrdWarps];
  const bool rec = blockIdx.x == 0;

  // step 0's reflector from row 0, and p_0 = tau_0 A[1..][1..] v_0
  Reflector R;
  {
    const int m = n - 1;
    const double* row0 = A + 1;
    double s = 0.0;
    for (int j = 1 + threadIdx.x; j < m; j += kTrdThreads) s = fma(row0[j], row0[j], s);
    R = make_reflector(row0[0], trd_block_sum(s, red[1]));
    for (int j = threadIdx.x; j < m; j += kTrdThreads) sv[j] = j == 0 ? 1.0 : row0[j] * R.scale;
    __syncthreads();
    if (rec) {
      if (threadIdx.x == 0) {
        d[0] = A[0];
        e[0] = R.beta;
        taus[0] = R.tau;
      }
      for (int j = threadIdx.x; j < m; j += kTrdThreads) V[1 + j] = sv[j];
    }
    trd_rows<false>(A, n, 1, m, nullptr, nullptr, sv, R.tau, p + 1, part, red[2], segsum);
  }
  grid.sync();

  for (int k = 0; k + 2 < n; ++k) {
    const int m = n - k - 1;  // v_k, w_k, p_k over indices k + 1 .. n - 1
    const double* pk = p + (k & 1) * n + k + 1;
    const double* rk1 = A + static_cast<i64>(k + 1) * n + k + 1;
    // everything this step reads from global memory, in one round trip
    double preg[kTrdMaxPer], rreg[kTrdMaxPer];
#pragma unroll
    for (int q = 0; q < kTrdMaxPer; ++q) {
      const int j = threadIdx.x + q * kTrdThreads;
      if (j < m) {
        preg[q] = pk[j];
        rreg[q] = rk1[j];
      }
    }
    const double p0 = pk[0];
    const double t = static_cast<int>(threadIdx.x) < static_cast<int>(gridDim.x)
                         ? part[(k & 1) * gridDim.x + threadIdx.x]
                         : 0.0;
    // K_k (same order in every CTA), w_k, the updated row k + 1 over columns
    // k + 1 .. (index 0 = the diagonal) and its norm beyond the subdiagonal
    const double K = 0.5 * R.tau * trd_block_sum(t, red[0]);
    const double w0 = p0 - K * sv[0];
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kTrdMaxPer; ++q) {
      const int j = threadIdx.x + q * kTrdThreads;
      if (j < m) {
        const double vj = sv[j], wj = preg[q] - K * vj;
        sw[j] = wj;
        const double r = rreg[q] - (wj + __dmul_rn(w0, vj));  // v_k[0] = 1
        srow[j] = r;
        if (j >= 2) s = fma(r, r, s);
      }
    }
    for (int j = threadIdx.x + kTrdMaxPer * kTrdThreads; j < m; j += kTrdThreads) {  // n > 4096
      const double vj = sv[j], wj = pk[j] - K * vj;
      sw[j] = wj;
      const double r = rk1[j] - (wj + __dmul_rn(w0, vj));
      srow[j] = r;
      s = fma(r, r, s);
    }
    const double sig = trd_block_sum(s, red[1]);
    if (k + 3 == n) {  // the last 2 x 2 block
      if (rec && threadIdx.x == 0) {
        d[n - 2] = srow[0];
        e[n - 2] = srow[1];
        const double* rl = A + static_cast<i64>(n - 1) * n + n - 1;
        d[n - 1] = rl[0] - (__dmul_rn(sv[1], sw[1]) + __dmul_rn(sw[1], sv[1]));
      }
      break;
    }
    const int mn = m - 1;  // v_{k+1} over indices k + 2 .. n - 1
    const Reflector Rn = make_reflector(srow[1], sig);
    for (int j = threadIdx.x; j < mn; j += kTrdThreads) snv[j] = j == 0 ? 1.0 : srow[1 + j] * Rn.scale;
    __syncthreads();
    if (rec) {
      if (threadIdx.x == 0) {
        d[k + 1] = srow[0];
        e[k + 1] = Rn.beta;
        taus[k + 1] = Rn.tau;
      }
      double* vk = V + static_cast<i64>(k + 1) * n + k + 2;
      for (int j = threadIdx.x; j < mn; j += kTrdThreads) vk[j] = snv[j];
    }
    trd_rows<true>(A, n, k + 2, mn, sv, sw, snv, Rn.tau, p + ((k + 1) & 1) * n + k + 2,
                   part + ((k + 1) & 1) * gridDim.x, red[2], segsum);
    double* tmp = sv;
    sv = snv;
    snv = tmp;
    R = Rn;
    grid.sync();
  }
}

__device__ inline double dfast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  return r * fma(-x, r, 2.0);
}

// Number of eigenvalues of T below x (Sturm sequence, dlaneg's pivmin rule).
__host__ __device__ inline int sturm_count(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                           double x, double pivmin) {
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  int c = q < 0.0;
  for (int i = 1; i < n; ++i) {
#ifdef __CUDA_ARCH__
    q = (d[i] - x) - e2[i - 1] * dfast_rcp(q);
#else
    q = (d[i] - x) - e2[i - 1] / q;
#endif
    if (fabs(q) < pivmin) q = -pivmin;
    c += q < 0.0;
  }
  return c;
}

// lam[j] = the eigenvalue of ascending index a0 + j (j < count), one warp
// each: 32-point multisection of [gl, gu] to the dstebz tolerance.
__global__ void k_bisect(const double* __restrict__ d, const double* __restrict__ e2, int n, int a0, int count,
                         double gl, double gu, double pivmin, double* __restrict__ lam) {
  pdl_wait();
  const int j = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (j >= count) return;
  const int idx = a0 + j;
  double lo = gl, hi = gu;  // count(lo) <= idx < count(hi)
  for (int it = 0; it < 80; ++it) {
    const double tol = 2.0 * kEps * fmax(fabs(lo), fabs(hi)) + pivmin;
    if (hi - lo <= tol) break;
    const double x = lo + (hi - lo) * ((lane + 1) / 33.0);
    const int c = sturm_count(d, e2, n, x, pivmin);
    const int nb = __popc(__ballot_sync(0xffffffffu, c <= idx));  // counts grow with x: lanes < nb
    const double nlo = __shfl_sync(0xffffffffu, x, (nb + 31) & 31);
    const double nhi = __shfl_sync(0xffffffffu, x, nb & 31);
    if (nb > 0) lo = nlo;
    if (nb < 32) hi = nhi;
  }
  if (lane == 0) lam[j] = 0.5 * (lo + hi);
}

// Eigenvector of T for the shift shift[c], one warp per eigenvalue (all in
// parallel): LU of T - shift I with partial pivoting (dgttrf) and three
// solves (dgttrs) by lane 0 with the recurrences carried in registers, from
// a fixed start vector, normalised by the warp.  Y [count][n]; work per
// warp 4 n doubles + n ints.
__device__ inline double lu_rcp(double x) {
  return fabs(x) > 1e-290 ? dfast_rcp(x) : 1.0 / x;
}

__global__ void k_tri_invit(const double* __restrict__ d, const double* __restrict__ e, int n,
                            const double* __restrict__ shift, int count, double tnorm, double* __restrict__ Y,
                            double* __restrict__ work, int* __restrict__ iwork) {
  pdl_wait();
  const int c = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (c >= count) return;
  double* du = work + static_cast<i64>(c) * 4 * n;
  double* du2 = du + n;
  double* dl = du2 + n;
  double* rdd = dl + n;
  double* x = Y + static_cast<i64>(c) * n;
  int* piv = iwork + static_cast<i64>(c) * n;
  const double tiny = kEps * fmax(tnorm, 1e-300);
  const double lm = shift[c];
  if (lane == 0) {
    double cd = d[0] - lm, cu = n > 1 ? e[0] : 0.0;
    for (int i = 0; i + 1 < n; ++i) {
      const double l = e[i], nd = d[i + 1] - lm, nu = i + 2 < n ? e[i + 1] : 0.0;
      double dd;
      if (fabs(cd) >= fabs(l)) {
        const double f = cd != 0.0 ? l * lu_rcp(cd) : 0.0;
        dl[i] = f;
        dd = cd;
        du[i] = cu;
        du2[i] = 0.0;
        piv[i] = i;
        cd = nd - f * cu;
        cu = nu;
      } else {
        const double f = cd * lu_rcp(l);
        dl[i] = f;
        dd = l;
        du[i] = nd;
        du2[i] = nu;
        piv[i] = i + 1;
        cd = cu - f * nd;
        cu = -f * nu;
      }
      if (fabs(dd) < tiny) dd = dd < 0.0 ? -tiny : tiny;
      rdd[i] = 1.0 / dd;
    }
    if (fabs(cd) < tiny) cd = cd < 0.0 ? -tiny : tiny;
    rdd[n - 1] = 1.0 / cd;
  }
  for (int i = lane; i < n; i += 32) x[i] = 1.0 + 0.25 * sin(0.7 * (i + 1) + 1.3 * (c + 1));
  __syncwarp();
  for (int it = 0; it < 3; ++it) {
    if (lane == 0) {
      double xi = x[0];
      for (int i = 0; i + 1 < n; ++i) {
        const double nx = x[i + 1], f = dl[i];
        if (piv[i] == i) {
          x[i] = xi;
          xi = nx - f * xi;
        } else {
          x[i] = nx;
          xi = xi - f * nx;
        }
      }
      double x1 = xi * rdd[n - 1];
      x[n - 1] = x1;
      double x2 = x1;
      x1 = (x[n - 2] - du[n - 2] * x2) * rdd[n - 2];
      x[n - 2] = x1;
      for (int i = n - 3; i >= 0; --i) {
        const double v = (x[i] - du[i] * x1 - du2[i] * x2) * rdd[i];
        x[i] = v;
        x2 = x1;
        x1 = v;
      }
    }
    __syncwarp();
    double s2 = 0.0;
    for (int i = lane; i < n; i += 32) s2 = fma(x[i], x[i], s2);
    const double inv = 1.0 / sqrt(dw_sum(s2));
    for (int i = lane; i < n; i += 32) x[i] *= inv;
    __syncwarp();
  }
}

// Orthonormalises each cluster's vectors in order (two Gram-Schmidt passes
// against the earlier members), one warp per cluster.
__global__ void k_cluster_mgs(int n, const int* __restrict__ cl_start, int n_clusters, double* __restrict__ Y) {
  pdl_wait();
  const int cl = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (cl >= n_clusters) return;
  const int c0 = cl_start[cl], c1 = cl_start[cl + 1];
  for (int c = c0 + 1; c < c1; ++c) {
    double* x = Y + static_cast<i64>(c) * n;
    for (int pass = 0; pass < 2; ++pass) {
      for (int c2 = c0; c2 < c; ++c2) {
        const double* u = Y + static_cast<i64>(c2) * n;
        double s = 0.0;
        for (int i = lane; i < n; i += 32) s = fma(x[i], u[i], s);
        s = dw_sum(s);
        for (int i = lane; i < n; i += 32) x[i] -= s * u[i];
        __syncwarp();
      }
      double s2 = 0.0;
      for (int i = lane; i < n; i += 32) s2 = fma(x[i], x[i], s2);
      const double inv = 1.0 / sqrt(dw_sum(s2));
      for (int i = lane; i < n; i += 32) x[i] *= inv;
      __syncwarp();
    }
  }
}

// X[c] = H_0 ... H_{n-3} Y[c] (H_k = I - tau_k v_k v_k^T on indices k + 1 ..),
// one CTA per vector, held in shared memory; the next reflector streams into
// a second shared buffer (cp.async) while the current one is applied, so the
// per-reflector chain is two barriers and no global-memory latency.  The
// partial sums alternate between two reduction buffers, so a fast warp's
// next partial cannot overwrite one still being read.
constexpr int kBtThreads = 512;
__device__ __forceinline__ void bt_cp8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src));
}
__global__ void __launch_bounds__(kBtThreads) k_back_transform(const double* __restrict__ V,
                                                               const double* __restrict__ taus, int n,
                                                               const double* __restrict__ Y, double* __restrict__ X) {
  pdl_wait();
  extern __shared__ double bsm[];  // x [n], tau [n], v buffers [2][n]
  double* xs = bsm;
  double* ts = bsm + n;
  double* ub[2] = {bsm + 2 * n, bsm + 3 * n};
  __shared__ double red[2][kBtThreads / 32];
  const int c = blockIdx.x, lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < n; i += kBtThreads) {
    xs[i] = Y[static_cast<i64>(c) * n + i];
    ts[i] = i + 2 < n ? taus[i] : 0.0;
  }
  auto issue = [&](int k, double* dst) {
    const double* u = V + static_cast<i64>(k) * n + k + 1;
    for (int j = threadIdx.x; j < n - k - 1; j += kBtThreads) bt_cp8(dst + j, u + j);
  };
  int k = n - 3, b = 0, par = 0;
  if (k >= 0) issue(k, ub[0]);
  asm volatile("cp.async.commit_group;\n" ::);
  for (; k >= 0; --k) {
    // v_k has landed and every thread is past the previous reflector's update
    // (so its buffer, ub[b ^ 1], may be refilled with v_{k-1})
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    if (k >= 1) issue(k - 1, ub[b ^ 1]);
    asm volatile("cp.async.commit_group;\n" ::);
    const int m = n - k - 1;
    const double* u = ub[b];  // u[0] = 1 (stored)
    double* xx = xs + k + 1;
    double s = 0.0;
    for (int j = threadIdx.x; j < m; j += kBtThreads) s = fma(u[j], xx[j], s);
    s = dw_sum(s);
    if (lane == 0) red[par][wib] = s;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kBtThreads / 32; ++w) t += red[par][w];
    t *= ts[k];
    for (int j = threadIdx.x; j < m; j += kBtThreads) xx[j] -= t * u[j];
    b ^= 1;
    par ^= 1;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kBtThreads) X[static_cast<i64>(c) * n + i] = xs[i];
}

}  // namespace

std::size_t dense_trd_smem(i64 M) { return sizeof(double) * 4 * static_cast<std::size_t>(M); }

// The leading `count` eigenpairs of the symmetric M x M matrix `sigma`
// (device, row-major): eigenvalues descending into lam_out, eigenvectors as
// rows of vecs [count][M] (device), and the sum of all eigenvalues above
// cut_rel * max(0, lambda_1) into above_cut.  Returns false when M is
// outside the kernels' range (3 <= M, 4 M doubles of shared memory, a
// cooperative grid) or T is not finite; the caller uses the library
// eigensolver then.
bool dense_top_eigenpairs(dfpca_context* ctx, const double* sigma, i64 M, int count, double cut_rel,
                          std::vector<double>& lam_out, double* vecs, double& above_cut) {
  const std::size_t shm = dense_trd_smem(M);
  if (M < 3 || shm > 220 * 1024 || count < 1 || count > M) return false;
  allow_smem(k_trd, shm);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trd, kTrdThreads, shm) != cudaSuccess || per_sm < 1)
    return false;
  cudaStream_t st = ctx->stream;
  const int n = static_cast<int>(M);
  const int blocks = ctx->sm_count;
  DevBuf<double> A(static_cast<std::size_t>(M * M)), V(static_cast<std::size_t>(M * M)), d(M), e(M), taus(M),
      p(static_cast<std::size_t>(2 * M)), part(static_cast<std::size_t>(2 * blocks));
  DFPCA_CUDA(cudaMemcpyAsync(A.get(), sigma, sizeof(double) * M * M, cudaMemcpyDeviceToDevice, st));
  {
    double* a = A.get();
    double *dp = d.get(), *ep = e.get(), *tp = taus.get(), *vp = V.get(), *pp = p.get(), *qp = part.get();
    int nn = n;
    void* args[] = {&a, &nn, &dp, &ep, &tp, &vp, &pp, &qp};
    const int slot = ctx->profile ? ctx->kernel_begin("k_trd") : -1;
    const cudaError_t le = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_trd), dim3(blocks),
                                                       dim3(kTrdThreads), args, shm, st);
    if (le == cudaErrorCooperativeLaunchTooLarge) {  // SMs taken (e.g. by MPS limits): the library path
      cudaGetLastError();
      return false;
    }
    DFPCA_CUDA(le);
    if (slot >= 0) ctx->kernel_end(slot);
    ++ctx->launches;
  }
  std::vector<double> hd(static_cast<std::size_t>(n)), he(static_cast<std::size_t>(n), 0.0);
  DFPCA_CUDA(cudaMemcpyAsync(hd.data(), d.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaMemcpyAsync(he.data(), e.get(), sizeof(double) * (n - 1), cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
  // Gershgorin interval, ||T||, trace, pivmin (dstebz)
  double gl = 1e300, gu = -1e300, tnorm = 0.0, emax2 = 0.0, trace = 0.0;
  std::vector<double> he2(static_cast<std::size_t>(n), 0.0);
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? std::fabs(he[i - 1]) : 0.0) + (i + 1 < n ? std::fabs(he[i]) : 0.0);
    gl = std::min(gl, hd[i] - r);
    gu = std::max(gu, hd[i] + r);
    tnorm = std::max(tnorm, std::fabs(hd[i]) + r);
    trace += hd[i];
    if (i + 1 < n) {
      he2[i] = he[i] * he[i];
      emax2 = std::max(emax2, he2[i]);
    }
  }
  if (!std::isfinite(tnorm)) return false;
  if (tnorm == 0.0) {  // the zero matrix: every eigenvalue is 0, none passes the cut
    lam_out.assign(static_cast<std::size_t>(count), 0.0);
    above_cut = 0.0;
    return true;
  }
  const double pivmin = 2.2250738585072014e-308 * std::max(1.0, emax2);
  const double pad = 2.0 * kEps * tnorm * n + 2.0 * pivmin;
  gl -= pad;
  gu += pad;
  DevBuf<double> e2(static_cast<std::size_t>(n)), lam(static_cast<std::size_t>(n));
  DFPCA_CUDA(cudaMemcpyAsync(e2.get(), he2.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
  auto bisect = [&](int a0, int cnt, std::vector<double>& out) {
    out.assign(static_cast<std::size_t>(std::max(cnt, 0)), 0.0);
    if (cnt <= 0) return;
    DFPCA_LAUNCH(ctx, k_bisect, static_cast<unsigned>((cnt * 32 + 255) / 256), 256, 0, d.get(), e2.get(), n, a0, cnt,
                 gl, gu, pivmin, lam.get());
    DFPCA_CUDA(cudaMemcpyAsync(out.data(), lam.get(), sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
    DFPCA_CUDA(cudaStreamSynchronize(st));
  };
  std::vector<double> asc;
  bisect(n - count, count, asc);
  lam_out.assign(asc.rbegin(), asc.rend());
  // the eigenvalues above the cut are the n - count(cut) largest
  const double cut = std::max(0.0, lam_out[0]) * cut_rel;
  const int below = sturm_count(hd.data(), he2.data(), n, cut, pivmin);
  const int n_above = n - below;
  above_cut = 0.0;
  if (n_above <= count) {
    for (int l = 0; l < n_above; ++l) above_cut += lam_out[static_cast<std::size_t>(l)];
  } else if (n_above - count <= below) {
    std::vector<double> rest;
    bisect(below, n_above - count, rest);
    for (int l = 0; l < count; ++l) above_cut += lam_out[static_cast<std::size_t>(l)];
    for (auto it = rest.rbegin(); it != rest.rend(); ++it) above_cut += *it;
  } else {
    std::vector<double> low;
    bisect(0, below, low);
    double s = 0.0;
    for (double v : low) s += v;
    above_cut = trace - s;
  }
  // shifts (equal eigenvalues pulled apart, dstein-style) and the clusters
  // reorthogonalised afterwards (dstein's rule: gaps below 1e-3 ||T||)
  std::vector<double> shifts(lam_out);
  std::vector<int> cls;
  for (int c = 0; c < count; ++c) {
    if (c > 0) {
      const double sep = 10.0 * kEps * std::max(std::fabs(shifts[c]), tnorm * kEps);
      if (!(shifts[c - 1] - shifts[c] > sep)) shifts[c] = shifts[c - 1] - sep;
    }
    if (c == 0 || !(lam_out[c - 1] - lam_out[c] <= 1e-3 * tnorm)) cls.push_back(c);
  }
  const int ncl = static_cast<int>(cls.size());
  cls.push_back(count);
  DFPCA_CUDA(cudaMemcpyAsync(lam.get(), shifts.data(), sizeof(double) * count, cudaMemcpyHostToDevice, st));
  DevBuf<int> dcl(cls.size());
  DFPCA_CUDA(cudaMemcpyAsync(dcl.get(), cls.data(), sizeof(int) * cls.size(), cudaMemcpyHostToDevice, st));
  DevBuf<double> work(static_cast<std::size_t>(count) * 4 * n), Y(static_cast<std::size_t>(count) * n);
  DevBuf<int> iwork(static_cast<std::size_t>(count) * n);
  DFPCA_LAUNCH(ctx, k_tri_invit, static_cast<unsigned>((count * 32 + 63) / 64), 64, 0, d.get(), e.get(), n,
               lam.get(), count, tnorm, Y.get(), work.get(), iwork.get());
  DFPCA_LAUNCH(ctx, k_cluster_mgs, static_cast<unsigned>((ncl * 32 + 63) / 64), 64, 0, n, dcl.get(), ncl, Y.get());
  const std::size_t bsm = sizeof(double) * 4 * static_cast<std::size_t>(n);
  allow_smem(k_back_transform, bsm);
  DFPCA_LAUNCH(ctx, k_back_transform, static_cast<unsigned>(count), kBtThreads, bsm, V.get(), taus.get(), n, Y.get(),
               vecs);
  return true;
}

}  // namespace dfpca_gpu
