// K6-K8: matrixization and the random-projection eigensolver
// (reference matrixize / randomized_eig / finalize_eigensystem,
// eigensolve.hpp:71-103, 121-194, 245-279), all on the device:
//   Omega   seeded M x q sketch: mt19937_64 (one CTA, parallel twist) +
//           Box-Muller, the reference's RandomStream draw order (rng.hpp:30-78);
//   Y       = Sigma Omega                      (DMMA GEMM, split-K)
//   Q       Cholesky QR twice (DMMA Gram products + fused factor/solve
//           passes); Householder QR (one reflector per launch) when the
//           sketch is too ill-conditioned for it
//   small   = Q^T (Sigma Q), symmetrized       (DMMA GEMMs)
//   eig     q <= 128: tridiagonalization + multisection + inverse iteration
//           (one CTA); larger q: cyclic parallel Jacobi
//   lifted  = Q V                               (DMMA GEMM)
//   final   Riemann MGS, norm cut, sign canonicalization (one CTA)
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <cmath>
#include <vector>

#include "gemm.cuh"
#include "shard_exec.hpp"

namespace dfpca_gpu {
namespace {

// ---------------------------------------------------------------- RNG ----
constexpr int kMtN = 312, kMtM = 156;
constexpr unsigned long long kMtA = 0xB5026F5AA96619E9ull;
constexpr unsigned long long kMtUpper = 0xFFFFFFFF80000000ull, kMtLower = 0x7FFFFFFFull;

__host__ __device__ inline unsigned long long splitmix64(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// std::mt19937_64 seeded with `seed` (or resumed from `state`), producing
// n_words tempered outputs (a multiple of 312 when the state is carried on).
// The twist runs out of place between two state buffers: the 156 words that
// depend only on the old state, one barrier, the 156 that need the first
// half's new words, and each thread tempers the word it has just written --
// two barriers per 312 outputs.
__global__ void __launch_bounds__(kMtN) k_mt19937_64(unsigned long long seed, i64 n_words,
                                                     unsigned long long* __restrict__ out,
                                                     unsigned long long* __restrict__ state, int resume) {
  pdl_wait();
  __shared__ unsigned long long buf[2][kMtN];
  if (resume) {
    buf[0][threadIdx.x] = state[threadIdx.x];
  } else if (threadIdx.x == 0) {
    buf[0][0] = seed;
    for (int i = 1; i < kMtN; ++i)
      buf[0][i] =
          6364136223846793005ull * (buf[0][i - 1] ^ (buf[0][i - 1] >> 62)) + static_cast<unsigned long long>(i);
  }
  __syncthreads();
  const int i = threadIdx.x;
  int cur = 0;
  for (i64 base = 0; base < n_words; base += kMtN) {
    const unsigned long long* a = buf[cur];
    unsigned long long* b = buf[cur ^ 1];
    if (i < kMtN - kMtM) {
      const unsigned long long x = (a[i] & kMtUpper) | (a[i + 1] & kMtLower);
      b[i] = a[i + kMtM] ^ (x >> 1) ^ ((x & 1ull) ? kMtA : 0ull);
    }
    __syncthreads();
    if (i >= kMtN - kMtM) {
      const unsigned long long nxt = i < kMtN - 1 ? a[i + 1] : b[0];
      const unsigned long long x = (a[i] & kMtUpper) | (nxt & kMtLower);
      b[i] = b[i - (kMtN - kMtM)] ^ (x >> 1) ^ ((x & 1ull) ? kMtA : 0ull);
    }
    if (base + i < n_words) {
      unsigned long long y = b[i];
      y ^= (y >> 29) & 0x5555555555555555ull;
      y ^= (y << 17) & 0x71D67FFFEDA60000ull;
      y ^= (y << 37) & 0xFFF7EEE000000000ull;
      y ^= y >> 43;
      out[base + i] = y;
    }
    __syncthreads();
    cur ^= 1;
  }
  if (state) state[i] = buf[cur][i];  // the state after the last full twist (resume point)
}

// Omega(i, j) = sd * normal #(j * M + i) (column-major fill,
// eigensolve.hpp:257-258); normals come in Box-Muller pairs cos, sin.
// Stored row-major [M][ldq] (ldq even; the padding is never read) as the
// GEMM's K-major operand.
__global__ void k_box_muller(const unsigned long long* __restrict__ words, i64 M, i64 q, i64 ldq, double sd,
                             i64 p_begin, i64 p_end, double* __restrict__ omega) {
  pdl_wait();
  const i64 total = M * q;
  for (i64 pidx = p_begin + blockIdx.x * (i64)blockDim.x + threadIdx.x; pidx < p_end;
       pidx += (i64)gridDim.x * blockDim.x) {
    const double u1 = (static_cast<double>(words[2 * pidx] >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = (static_cast<double>(words[2 * pidx + 1] >> 11) + 0.5) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    double sn, cs;
    sincos(a, &sn, &cs);
    const double vals[2] = {r * cs, r * sn};
    for (int h = 0; h < 2; ++h) {
      const i64 idx = 2 * pidx + h;
      if (idx >= total) break;
      const i64 j = idx / M, ii = idx % M;
      omega[ii * ldq + j] = sd * vals[h];
    }
  }
}

// ----------------------------------------------------------- helpers ----
__global__ void k_gather_sigma(const double* __restrict__ cov, i64 G, const i64* __restrict__ node_of_row,
                               i64 M, double* __restrict__ sig) {
  pdl_wait();
  const i64 total = M * M;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / M, c = e % M;
    sig[e] = cov[node_of_row[r] * G + node_of_row[c]];
  }
}

// out[c][r] = in[r][c] for r < rows, c < cols (row strides ld_in, ld_out).
__global__ void k_transpose(const double* __restrict__ in, i64 rows, i64 cols, i64 ld_in, double* __restrict__ out,
                            i64 ld_out) {
  pdl_wait();
  __shared__ double tile[32][33];
  const i64 tiles_c = (cols + 31) / 32;
  const i64 br = blockIdx.x / tiles_c, bc = blockIdx.x % tiles_c;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  for (int r = ty; r < 32; r += 8) {
    const i64 gr = br * 32 + r, gc = bc * 32 + tx;
    tile[r][tx] = (gr < rows && gc < cols) ? in[gr * ld_in + gc] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const i64 oc = br * 32 + tx, orow = bc * 32 + r;  // out[orow][oc] = in[oc][orow]
    if (orow < cols && oc < rows) out[orow * ld_out + oc] = tile[tx][r];
  }
}

void transpose(dfpca_context* ctx, const double* in, i64 rows, i64 cols, double* out, i64 ld_in = -1,
               i64 ld_out = -1) {
  const i64 blocks = ((rows + 31) / 32) * ((cols + 31) / 32);
  DFPCA_LAUNCH(ctx, k_transpose, static_cast<unsigned>(blocks), 256, 0, in, rows, cols, ld_in < 0 ? cols : ld_in,
               out, ld_out < 0 ? rows : ld_out);
}

__device__ inline double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[32] = v;
  }
  __syncthreads();
  return red[32];
}

// ------------------------------------------------------- Householder ----
// Columns of Y are the rows of Yt [q][M].  Reflector j: v (v_j = 1) stored in
// Yt[j][j+1..], tau[j], R(j,j) = beta.

// Make reflector for column j from the current Yt[j][j..].
__device__ void make_reflector(double* col, i64 j, i64 M, double* tau, double* red) {
  double s = 0.0;
  for (i64 i = j + 1 + threadIdx.x; i < M; i += blockDim.x) s += col[i] * col[i];
  const double sigma = block_sum(s, red);
  const double x0 = col[j];
  double t = 0.0, beta = x0, scale = 0.0;
  if (sigma > 0.0) {
    beta = sqrt(x0 * x0 + sigma);
    if (x0 >= 0.0) beta = -beta;
    t = (beta - x0) / beta;
    scale = 1.0 / (x0 - beta);
  }
  __syncthreads();
  for (i64 i = j + 1 + threadIdx.x; i < M; i += blockDim.x) col[i] = sigma > 0.0 ? col[i] * scale : 0.0;
  if (threadIdx.x == 0) {
    tau[j] = t;
    col[j] = beta;
  }
  __syncthreads();
}

// Apply reflector j to columns c = j+1.. (one CTA per column); the CTA of
// column j+1 then forms reflector j+1.  Launch with j = -1 to only form
// reflector 0.
__global__ void k_house_step(double* __restrict__ Yt, i64 M, i64 q, i64 j, double* __restrict__ tau) {
  pdl_wait();
  __shared__ double red[33];
  const i64 c = j + 1 + blockIdx.x;
  if (c >= q) return;
  double* col = Yt + c * M;
  if (j >= 0) {
    const double* v = Yt + j * M;
    double s = threadIdx.x == 0 ? col[j] : 0.0;  // v_j = 1
    for (i64 i = j + 1 + threadIdx.x; i < M; i += blockDim.x) s += v[i] * col[i];
    const double w = block_sum(s, red) * tau[j];
    for (i64 i = j + threadIdx.x; i < M; i += blockDim.x) col[i] -= w * (i == j ? 1.0 : v[i]);
    __syncthreads();
  }
  if (c == j + 1) make_reflector(col, c, M, tau, red);
}

// Q = H_0 ... H_{q-1} [I; 0], backward accumulation; Qt rows are Q columns.
__global__ void k_q_init(double* __restrict__ Qt, i64 M, i64 q) {
  pdl_wait();
  const i64 total = q * M;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / M, i = e % M;
    Qt[e] = (r == i) ? 1.0 : 0.0;
  }
}

__global__ void k_q_apply(const double* __restrict__ Yt, const double* __restrict__ tau, i64 M, i64 q,
                          i64 j, double* __restrict__ Qt) {
  pdl_wait();
  __shared__ double red[33];
  const i64 c = j + blockIdx.x;
  if (c >= q) return;
  const double* v = Yt + j * M;
  double* col = Qt + c * M;
  double s = threadIdx.x == 0 ? col[j] : 0.0;
  for (i64 i = j + 1 + threadIdx.x; i < M; i += blockDim.x) s += v[i] * col[i];
  const double w = block_sum(s, red) * tau[j];
  for (i64 i = j + threadIdx.x; i < M; i += blockDim.x) col[i] -= w * (i == j ? 1.0 : v[i]);
}

// ------------------------------------------------------------ Jacobi ----
// Cyclic Jacobi with round-robin pair ordering: each round applies n/2
// disjoint rotations at once.  A (n x n, symmetrized on entry) and V live in
// global memory (L1/L2 resident).  Outputs eigenvalues descending and V's
// columns in the same order.
__global__ void __launch_bounds__(1024) k_jacobi(double* __restrict__ Ag, double* __restrict__ Vg, int n,
                                                 double* __restrict__ evals, int* __restrict__ info,
                                                 int in_smem) {
  pdl_wait();
  extern __shared__ double sh[];
  const int np = (n + 1) & ~1;  // padded to even (index n is a dummy)
  double* cs = sh;               // [np/2] cos
  double* sn = sh + np / 2;      // [np/2] sin
  int* pp = reinterpret_cast<int*>(sh + np);
  int* qq = pp + np / 2;
  __shared__ double red[33];
  __shared__ int converged;
  const int tid = threadIdx.x, nt = blockDim.x;
  // A and V live in shared memory when they fit (q <= ~110), else in global
  double* A = in_smem ? sh + 2 * np : Ag;
  double* V = in_smem ? A + n * n : Vg;
  if (in_smem) {
    for (int e = tid; e < n * n; e += nt) A[e] = Ag[e];
    __syncthreads();
  }
  // symmetrize (eigensolve.hpp:265) and V = I
  for (int e = tid; e < n * n; e += nt) {
    const int r = e / n, c = e % n;
    if (r < c) {
      const double s = 0.5 * (A[r * n + c] + A[c * n + r]);
      A[r * n + c] = s;
      A[c * n + r] = s;
    }
    V[e] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  double fro = 0.0;
  for (int e = tid; e < n * n; e += nt) fro += A[e] * A[e];
  const double norm2 = block_sum(fro, red);
  double last_off = 0.0;
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int e = tid; e < n * n; e += nt) {
      const int r = e / n, c = e % n;
      if (r != c) off += A[e] * A[e];
    }
    off = block_sum(off, red);
    // off-diagonal Frobenius norm at 1e-14 of the matrix's: rounding keeps
    // rotated entries at ~eps |lambda|, so a tighter bound may never be met
    if (tid == 0)
      converged = !(off > 1e-28 * norm2) || norm2 == 0.0 ||
                  (sweep > 2 && !(off < 0.5 * last_off) && !(off > 1e-20 * norm2));  // stalled at rounding
    last_off = off;
    __syncthreads();
    if (converged) break;
    for (int round = 0; round < np - 1; ++round) {
      // pairing: position 0 fixed, others rotate
      for (int k = tid; k < np / 2; k += nt) {
        auto pos = [&](int x) { return x == 0 ? 0 : 1 + (x - 1 + round) % (np - 1); };
        int a = pos(k), b = pos(np - 1 - k);
        if (a > b) {
          const int t = a;
          a = b;
          b = t;
        }
        pp[k] = a;
        qq[k] = b;
        double c = 1.0, s = 0.0;
        if (b < n) {
          const double apq = A[a * n + b];
          if (apq != 0.0) {
            const double app = A[a * n + a], aqq = A[b * n + b];
            const double theta = (aqq - app) / (2.0 * apq);
            const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
          }
        }
        cs[k] = c;
        sn[k] = s;
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int e = tid; e < (np / 2) * n; e += nt) {
        const int k = e / n, col = e % n;
        const int a = pp[k], b = qq[k];
        if (b >= n || sn[k] == 0.0) continue;
        const double c = cs[k], s = sn[k];
        const double xa = A[a * n + col], xb = A[b * n + col];
        A[a * n + col] = c * xa - s * xb;
        A[b * n + col] = s * xa + c * xb;
      }
      __syncthreads();
      // columns: A <- A J, V <- V J
      for (int e = tid; e < (np / 2) * n; e += nt) {
        const int k = e / n, row = e % n;
        const int a = pp[k], b = qq[k];
        if (b >= n || sn[k] == 0.0) continue;
        const double c = cs[k], s = sn[k];
        const double xa = A[row * n + a], xb = A[row * n + b];
        A[row * n + a] = c * xa - s * xb;
        A[row * n + b] = s * xa + c * xb;
        const double va = V[row * n + a], vb = V[row * n + b];
        V[row * n + a] = c * va - s * vb;
        V[row * n + b] = s * va + c * vb;
      }
      __syncthreads();
      // the annihilated pair is exactly zero in exact arithmetic; storing the
      // zero removes the rounding floor that would otherwise stall the
      // off-diagonal norm near n * eps * |A| for q ~ 100
      for (int k = tid; k < np / 2; k += nt) {
        const int a = pp[k], b = qq[k];
        if (b < n && sn[k] != 0.0) {
          A[a * n + b] = 0.0;
          A[b * n + a] = 0.0;
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    info[0] = (converged || !(last_off > 1e-20 * norm2)) ? 0 : 1;
    for (int i = 0; i < n; ++i) evals[i] = A[i * n + i];
  }
  __syncthreads();
  // order descending (stable selection on one thread; n <= a few hundred)
  if (tid == 0) {
    for (int i = 0; i < n; ++i) {
      int best = i;
      for (int j = i + 1; j < n; ++j)
        if (evals[j] > evals[best]) best = j;
      if (best != i) {
        const double t = evals[i];
        evals[i] = evals[best];
        evals[best] = t;
        info[1 + i] = best;
      } else {
        info[1 + i] = i;
      }
    }
  }
  __syncthreads();
  // apply the same swaps to V's columns
  for (int i = 0; i < n; ++i) {
    const int b = info[1 + i];
    if (b != i)
      for (int r = tid; r < n; r += nt) {
        const double t = V[r * n + i];
        V[r * n + i] = V[r * n + b];
        V[r * n + b] = t;
      }
    __syncthreads();
  }
  if (in_smem)
    for (int e = tid; e < n * n; e += nt) Vg[e] = V[e];
}

// ----------------------------------------------------- Cholesky QR ----
// One pass of Cholesky QR on X [M][q] (row-major): G = X^T X comes from the
// DMMA Gram product; k_chol_factor (one CTA) factors G = R^T R (upper R,
// q <= 128, right-looking in shared memory, one barrier per pivot: row k is
// scaled on its way out to global memory, so the trailing update reads the
// unscaled row without a hazard), and k_row_trsm solves Xout R = X by
// forward substitution, one thread per row, R read as shared-memory
// broadcasts.  flags[0] = 1 on a non-positive pivot; flags[1] = max|G - I|
// (how far X already was from orthonormal columns).
constexpr int kCqMaxQ = 128;

// Right-looking Cholesky (upper, G = R^T R) on one CTA of 1024 threads, one
// barrier per pivot: row k is scaled on its way out to global memory, so the
// trailing update (a warp per row, lanes over columns) reads the unscaled
// row without a hazard.  Measured faster than 32-wide blocked panels and than
// a 256-thread column-oriented variant (87 vs 150 / 137 us at q = 99): the
// factorization is bound by its pivot chain, and more warps hide it better.
__global__ void __launch_bounds__(1024) k_chol_factor(const double* __restrict__ Gg, int q, double* __restrict__ Rg,
                                                      double* __restrict__ flags, double shift_scale) {
  pdl_wait();
  extern __shared__ double sm[];
  const int ld = q + 1;
  double* R = sm;
  __shared__ double red[32];
  __shared__ double shift;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double dmax = 0.0;
  for (int e = tid; e < q * q; e += blockDim.x) {
    const int r = e / q, c = e % q;
    const double g = Gg[e];
    R[r * ld + c] = g;
    Rg[e] = 0.0;
    dmax = fmax(dmax, fabs(g - (r == c ? 1.0 : 0.0)));
  }
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (lane == 0) red[warp] = dmax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < nw; ++w) m = fmax(m, red[w]);
    flags[1] = m;
    flags[0] = 0.0;
    // shifted Cholesky QR (Fukaya et al. 2020): G + s I with
    // s = 11 (M q + q (q + 1)) u ||X||_F^2 makes the factorization succeed for
    // sketches up to cond ~ 1/u; two more unshifted passes restore
    // orthogonality
    double tr = 0.0;
    for (int i = 0; i < q; ++i) tr += R[i * ld + i];
    shift = shift_scale * tr;
  }
  __syncthreads();
  if (shift_scale > 0.0)
    for (int i = tid; i < q; i += blockDim.x) R[i * ld + i] += shift;
  __syncthreads();
  for (int k = 0; k < q; ++k) {
    const double d = R[k * ld + k];
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) flags[0] = 1.0;
      return;  // uniform
    }
    const double rk = sqrt(d), inv = 1.0 / rk, dinv = 1.0 / d;
    for (int j = k + tid; j < q; j += blockDim.x) Rg[k * q + j] = j == k ? rk : R[k * ld + j] * inv;
    for (int i = k + 1 + warp; i < q; i += nw) {
      const double rki = R[k * ld + i] * dinv;
      for (int j = i + lane; j < q; j += 32) R[i * ld + j] -= rki * R[k * ld + j];
    }
    __syncthreads();
  }
}

// One warp per row: x_j = y_j / R_jj is broadcast from the lane holding it
// and every lane updates its entries l > j (column-oriented substitution:
// the dependent chain is one shuffle + one FMA per column).  R (q x q upper)
// sits in shared memory, read as conflict-free row segments.
constexpr int kTrsmWarps = 16;

__global__ void __launch_bounds__(kTrsmWarps * 32) k_row_trsm(const double* __restrict__ X, i64 M, int q, i64 ldx,
                                                              const double* __restrict__ Rg,
                                                              const double* __restrict__ flags,
                                                              double* __restrict__ Xout) {
  pdl_wait();
  if (flags[0] != 0.0) return;
  extern __shared__ double sm[];
  double* R = sm;           // [q][q]
  double* rinv = sm + q * q;  // 1 / R_jj
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < q * q; e += blockDim.x) R[e] = Rg[e];
  __syncthreads();
  for (int j = tid; j < q; j += blockDim.x) rinv[j] = 1.0 / R[j * q + j];
  __syncthreads();
  constexpr int kPer = kCqMaxQ / 32;  // entries per lane
  for (i64 row = static_cast<i64>(blockIdx.x) * kTrsmWarps + warp; row < M;
       row += static_cast<i64>(gridDim.x) * kTrsmWarps) {
    double y[kPer];
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int l = lane + 32 * t;
      y[t] = l < q ? X[row * ldx + l] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      for (int jl = 0; jl < 32; ++jl) {
        const int j = 32 * t + jl;
        if (j >= q) break;
        const double xj = __shfl_sync(0xffffffffu, y[t], jl) * rinv[j];
        if (lane == jl) y[t] = xj;
        const double* Rj = R + j * q;
#pragma unroll
        for (int u = t; u < kPer; ++u) {
          const int l = lane + 32 * u;
          if (l > j && l < q) y[u] -= xj * Rj[l];
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int l = lane + 32 * t;
      if (l < q) Xout[row * ldx + l] = y[t];
    }
  }
}

std::size_t trsm_smem(int q) { return sizeof(double) * (static_cast<std::size_t>(q) * q + q); }

// ------------------------------------------- small symmetric eigensolver ----
// Rayleigh-Ritz problem (eigensolve.hpp:264-270) on one CTA of 16 warps,
// n <= 128 (the reference runs SelfAdjointEigenSolver; any exact
// eigendecomposition gives the same Ritz pairs up to rounding):
//   symmetrize; Householder tridiagonalization (dsytd2) with the matrix in
//   registers (thread (column, row group)), the vectors in shared memory;
//   eigenvalues by Sturm-count multisection, 128 points per round (4 per
//   lane, independent chains), one warp per eigenvalue -- only the
//   candidates: a Ritz value at or below the cut enters no sum and is never
//   read (the cut's count comes from one more Sturm count);
//   eigenvectors of the candidates (eigenvalue > 1e-12 max(0, lambda_max),
//   the only ones finalize_eigensystem reads) by inverse iteration on the
//   tridiagonal (dgttrf/dgttrs with precomputed pivot reciprocals), one warp
//   per cluster with reorthogonalization inside clusters (gaps below
//   kClusterGap |T|), then back-transformed by the reflectors.
// Outputs: evals descending [n]; V [n][n] row-major, column c = eigenvector
// of evals[c] for the leading min(candidates, max_vec) (zero otherwise);
// info[0] = candidate count, info[1] = vectors computed; Vt [n][n] scratch
// (the tridiagonal eigenvectors as rows: coalesced reorthogonalization).
constexpr int kEigMaxN = 128;
// Cluster rule of the inverse iteration.  Vectors computed independently
// for eigenvalues a gap g apart are orthogonal to ~u |T| / g (the shifts are
// exact to ~u |T|), so with g >= 1e-7 |T| the loss is <= 2.2e-9 -- far inside
// the 1e-6 rad subspace bound and removed by the finalization's Gram-Schmidt
// -- and only closer eigenvalues are iterated together with
// reorthogonalization.  (LAPACK dstein groups gaps below 1e-3 |T|: at wide
// bandwidths that put the whole decaying tail of the Ritz spectrum, 20+
// members, into one sequential cluster.)
constexpr double kClusterGap = 1e-7;
#ifndef DFPCA_EIG_VEC_MARGIN
#define DFPCA_EIG_VEC_MARGIN 4
#endif
constexpr int kEigThreads = 512;
constexpr int kEigGroups = kEigThreads / kEigMaxN;  // row groups per column
constexpr int kEigWarps = kEigThreads / 32;
constexpr int kEigIIWarps = 8;  // warps with an inverse-iteration workspace

__device__ inline double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 1/x: the MUFU estimate refined by one Newton step (relative error well
// below 1e-12; a Sturm count only needs the signs of the pivots).
__device__ inline double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r * fma(-x, r, 2.0);
}

// Counts of eigenvalues of T (d, e2 = e^2) below each of 4 points (LAPACK
// dlaneg-style recurrences, run side by side).
__device__ inline void sturm_count4(const double* d, const double* e2, int n, const double x[4], double pivmin,
                                    int c[4]) {
  double qv[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    qv[r] = d[0] - x[r];
    if (fabs(qv[r]) < pivmin) qv[r] = -pivmin;
    c[r] = qv[r] < 0.0;
  }
  for (int i = 1; i < n; ++i) {
    const double di = d[i], ei = e2[i - 1];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      qv[r] = (di - x[r]) - ei * fast_rcp(qv[r]);
      if (fabs(qv[r]) < pivmin) qv[r] = -pivmin;
      c[r] += qv[r] < 0.0;
    }
  }
}

struct TriWork {  // one warp's inverse-iteration workspace
  double dd[kEigMaxN], rdd[kEigMaxN], du[kEigMaxN], du2[kEigMaxN], dl[kEigMaxN], x[kEigMaxN];
  int piv[kEigMaxN];
};

// Acceptance of a Cholesky QR from its per-pass flags (k_chol_factor: flags[2p]
// = breakdown, flags[2p + 1] = max |G - I| of pass p): every factorization
// succeeded and the last pass started within 0.1 of orthonormal columns (so
// it restored orthogonality to rounding).  The host applies the same rule.
__host__ __device__ inline bool qr_accepted(const double* flags, int passes) {
  bool ok = true;
  for (int p = 0; p < passes; ++p) ok = ok && flags[2 * p] == 0.0;
  return ok && flags[2 * (passes - 1) + 1] < 0.1;
}

__global__ void __launch_bounds__(kEigThreads) k_tri_eig(const double* __restrict__ Bg, int n,
                                                          double* __restrict__ evals_out, double* __restrict__ V,
                                                          int* __restrict__ info, int max_vec,
                                                          double* __restrict__ Vt,
                                                          const double* __restrict__ qr_flags, int qr_passes) {
  pdl_wait();
  // a Cholesky QR the host will reject (qr_accepted) makes this call moot:
  // skip it rather than spend the eigensolve on a basis about to be redone
  if (qr_flags && !qr_accepted(qr_flags, qr_passes)) return;
  extern __shared__ double sm[];
  double* Hv = sm;                    // [n][kEigMaxN] reflector vectors (row k: v of H_k)
  double* d = Hv + n * kEigMaxN;      // diagonal
  double* e = d + kEigMaxN;           // off-diagonal
  double* e2 = e + kEigMaxN;          // e^2
  double* tau = e2 + kEigMaxN;        // reflector scalars
  double* vb = tau + kEigMaxN;        // v of the current step
  double* wb = vb + kEigMaxN;         // w of the current step
  double* pp = wb + kEigMaxN;         // [kEigGroups][kEigMaxN] p partials
  double* lam = pp + kEigGroups * kEigMaxN;  // ascending eigenvalues
  double* xk = lam + kEigMaxN;        // column k of the current step
  TriWork* work = reinterpret_cast<TriWork*>(xk + kEigMaxN);
  double* btx = reinterpret_cast<double*>(work + kEigIIWarps);  // [kEigWarps][kEigMaxN] back-transform rows
  __shared__ int n_cand, n_vec, n_neg, n_clusters, cl_start[kEigMaxN + 1];
  __shared__ double tnorm_s, pivmin_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col = tid & (kEigMaxN - 1), grp = tid / kEigMaxN;  // thread (column, row group)

  // symmetrized on load (eigensolve.hpp:265)
  // ---- tridiagonalization: A = Q T Q^T, Q = H_0 ... H_{n-3};
  // H_k = I - tau_k v v^T on indices k+1..n-1 (v_{k+1} = 1), v kept in Hv[k].
  // The matrix lives in registers: thread (col, grp) holds A[j][col] for the
  // rows j = grp + kEigGroups r, so the p products and the rank-2 updates are
  // kRpt independent FMA chains per thread (FP64 latency is long; this is
  // what hides it); shared memory carries only the vectors.  Four barriers
  // per step.
  constexpr int kRpt = kEigMaxN / kEigGroups;
  double a[kRpt];
#pragma unroll
  for (int r = 0; r < kRpt; ++r) {
    const int j = grp + kEigGroups * r;
    a[r] = (j < n && col < n) ? 0.5 * (Bg[j * n + col] + Bg[col * n + j]) : 0.0;
  }
  __shared__ double ksum[kEigWarps], tau_s, kk_s;
  for (int k = 0; k + 2 < n; ++k) {
    const int m0 = k + 1;  // first trailing index
    // 1. column k (= row k) to shared memory
    if (col == k) {
#pragma unroll
      for (int r = 0; r < kRpt; ++r) {
        const int j = grp + kEigGroups * r;
        if (j >= k && j < n) xk[j] = a[r];
      }
    }
    __syncthreads();
    // 2. the reflector (warp 0)
    if (warp == 0) {
      double s = 0.0;
      for (int j = m0 + 1 + lane; j < n; j += 32) s += xk[j] * xk[j];
      const double sig = warp_sum(s);
      const double alpha = xk[m0];
      double t = 0.0, beta = alpha, scale = 0.0;
      if (sig > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + sig), alpha);
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      for (int j = m0 + lane; j < n; j += 32) {
        const double v = j == m0 ? 1.0 : xk[j] * scale;
        vb[j] = v;
        Hv[k * kEigMaxN + j] = v;
      }
      if (lane == 0) {
        tau[k] = t;
        tau_s = t;
        e[k] = beta;
        d[k] = xk[k];
      }
    }
    __syncthreads();
    const double t = tau_s;
    if (t == 0.0) continue;  // uniform: nothing to annihilate
    // 3. p partials (A22 v over this thread's rows) and v^T A22 v per warp
    double ps = 0.0;
    if (col >= m0 && col < n) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int r = 0; r < kRpt; r += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = grp + kEigGroups * (r + u);
          const double term = (j >= m0 && j < n) ? a[r + u] * vb[j] : 0.0;
          if (u == 0) s0 += term;
          else if (u == 1) s1 += term;
          else if (u == 2) s2 += term;
          else s3 += term;
        }
      }
      ps = (s0 + s1) + (s2 + s3);
      pp[grp * kEigMaxN + col] = ps;
    }
    const double qv = warp_sum(col >= m0 && col < n ? ps * vb[col] : 0.0);
    if (lane == 0) ksum[warp] = qv;
    __syncthreads();
    // 4. p = t A22 v; K = t/2 p^T v = t^2/2 v^T A22 v
    if (grp == 0 && col >= m0 && col < n) {
      double s = 0.0;
#pragma unroll
      for (int g = 0; g < kEigGroups; ++g) s += pp[g * kEigMaxN + col];
      wb[col] = t * s;
    }
    if (tid == 0) {
      double q = 0.0;
      for (int w = 0; w < kEigWarps; ++w) q += ksum[w];
      kk_s = 0.5 * t * t * q;
    }
    __syncthreads();
    // 5. A22 -= v w^T + w v^T, w = p - K v
    if (col >= m0 && col < n) {
      const double K = kk_s;
      const double vc = vb[col], wc = wb[col] - K * vc;
#pragma unroll
      for (int r = 0; r < kRpt; ++r) {
        const int j = grp + kEigGroups * r;
        if (j >= m0 && j < n) {
          const double vj = vb[j];
          a[r] -= vj * wc + (wb[j] - K * vj) * vc;
        }
      }
    }
  }
  // the last 2 x 2 block
  if (col == n - 2 || col == n - 1) {
#pragma unroll
    for (int r = 0; r < kRpt; ++r) {
      const int j = grp + kEigGroups * r;
      if (j == col) d[col] = a[r];
      if (col == n - 2 && j == n - 1) e[n - 2] = a[r];
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (n == 2) tau[0] = 0.0;
    double emax = 0.0, tn = 0.0;
    for (int i = 0; i < n; ++i) {
      const double ei = i + 1 < n ? fabs(e[i]) : 0.0, em = i > 0 ? fabs(e[i - 1]) : 0.0;
      if (i + 1 < n) {
        e2[i] = e[i] * e[i];
        emax = fmax(emax, e2[i]);
      }
      tn = fmax(tn, fabs(d[i]) + ei + em);
    }
    tnorm_s = tn;
    pivmin_s = 2.2250738585072014e-308 * fmax(1.0, emax);
  }
  __syncthreads();
  const double tnorm = tnorm_s, pivmin = pivmin_s;

  // ---- eigenvalues: only the candidates are needed (eigenvalue > cut =
  // 1e-12 max(0, lambda_max): finalize_eigensystem reads nothing else, and
  // the total variance sums only them).  Warp w resolves the (w+1)-th largest
  // eigenvalue by multisection (128 points per round, 4 independent Sturm
  // chains per lane); then the cut gives the candidate count (one Sturm
  // count) and the remaining candidates are spread over the warps.
  auto resolve = [&](int j) {  // j: ascending index, lambda_j > 0 known
    double lo = 0.0, hi = tnorm + 2.0 * pivmin;
    for (int round = 0; round < 12; ++round) {
      const double width = hi - lo;
      if (!(width > 2.0 * 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin)) break;
      double x[4];
      int c[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) x[r] = lo + width * (static_cast<double>(4 * lane + r + 1) / 129.0);
      sturm_count4(d, e2, n, x, pivmin, c);
      int fr = 4;  // first of this lane's points with count > j
#pragma unroll
      for (int r = 3; r >= 0; --r)
        if (c[r] > j) fr = r;
      const unsigned above = __ballot_sync(0xffffffffu, fr < 4);
      const int fl = above ? __ffs(above) - 1 : 32;
      // index f = 4 fl + fr of the first point above: bracket [point f-1, point f]
      const int f = fl == 32 ? 128 : 4 * fl + __shfl_sync(0xffffffffu, fr, fl == 32 ? 0 : fl);
      const double nlo = f == 0 ? lo : lo + width * (static_cast<double>(f) / 129.0);
      const double nhi = f == 128 ? hi : lo + width * (static_cast<double>(f + 1) / 129.0);
      lo = nlo;
      hi = nhi;
    }
    return 0.5 * (lo + hi);
  };
  if (tid == 0) {
    double x4[4] = {0.0, 0.0, 0.0, 0.0};
    int c4[4];
    sturm_count4(d, e2, n, x4, pivmin, c4);
    n_neg = c4[0];
  }
  __syncthreads();
  const int n_pos = n - n_neg;
  if (warp < n_pos) {
    const double v = resolve(n - 1 - warp);
    if (lane == 0) lam[n - 1 - warp] = v;
  }
  __syncthreads();
  if (tid == 0) {
    const double cut = n_pos > 0 ? lam[n - 1] * 1e-12 : 0.0;
    int nc = 0;
    if (n_pos > 0) {
      double x4[4] = {cut, cut, cut, cut};
      int c4[4];
      sturm_count4(d, e2, n, x4, pivmin, c4);
      nc = n - c4[0];  // eigenvalues above the cut
      if (nc > n_pos) nc = n_pos;
    }
    n_cand = nc;
  }
  __syncthreads();
  for (int c = kEigWarps + warp; c < n_cand; c += kEigWarps) {
    const double v = resolve(n - 1 - c);
    if (lane == 0) lam[n - 1 - c] = v;
  }
  __syncthreads();

  // ---- clusters of the candidates (descending order c = n-1-j)
  // Vectors only for the leading max_vec candidates: the finalization keeps
  // at most L_max of them (the caller passes L_max plus a margin for skipped
  // ones, and asks again with max_vec = n when that was not enough).
  if (tid == 0) {
    const int nc = n_cand;
    const int nv = nc < max_vec ? nc : max_vec;
    int ncl = 0;
    for (int c = 0; c < nv; ++c) {
      if (c == 0 || !(fabs(lam[n - 1 - c] - lam[n - c]) <= kClusterGap * tnorm)) cl_start[ncl++] = c;
    }
    cl_start[ncl] = nv;
    n_clusters = ncl;
    n_vec = nv;
    // the non-candidates are never read (finalize stops at the cut): zero
    for (int c = 0; c < n; ++c) evals_out[c] = c < nc ? lam[n - 1 - c] : 0.0;
    info[0] = nc;
    info[1] = nv;
  }
  __syncthreads();
  for (int e_ = tid; e_ < n * n; e_ += blockDim.x)
    if (e_ % n >= n_vec) V[e_] = 0.0;

  // ---- inverse iteration, one warp per cluster (members in order); the
  // T-eigenvectors of a cluster stay in V's columns until the cluster is done
  if (warp < kEigIIWarps) {
    TriWork& w = work[warp];
    const double eps = 2.220446049250313e-16;
    for (int cl = warp; cl < n_clusters; cl += kEigIIWarps) {
      const int c0 = cl_start[cl], c1 = cl_start[cl + 1];
      double prev = 0.0;
      for (int c = c0; c < c1; ++c) {
        double lm = lam[n - 1 - c];
        // separate (numerically) equal members, as dstein
        if (c > c0 && !(fabs(prev - lm) > 10.0 * eps * fabs(lm))) lm = prev - 10.0 * eps * fmax(fabs(lm), tnorm * eps);
        prev = lm;
        if (lane == 0) {
          // LU with partial pivoting of T - lm I (dgttrf)
          for (int i = 0; i < n; ++i) {
            w.dd[i] = d[i] - lm;
            if (i + 1 < n) {
              w.du[i] = e[i];
              w.dl[i] = e[i];
            }
            w.du2[i] = 0.0;
            w.piv[i] = i;
          }
          for (int i = 0; i + 1 < n; ++i) {
            if (fabs(w.dd[i]) >= fabs(w.dl[i])) {
              const double f = w.dd[i] != 0.0 ? w.dl[i] / w.dd[i] : 0.0;
              w.dl[i] = f;
              w.dd[i + 1] -= f * w.du[i];
            } else {
              const double f = w.dd[i] / w.dl[i];
              w.dd[i] = w.dl[i];
              w.dl[i] = f;
              const double tmp = w.du[i];
              w.du[i] = w.dd[i + 1];
              w.dd[i + 1] = tmp - f * w.dd[i + 1];
              if (i + 2 < n) {
                w.du2[i] = w.du[i + 1];
                w.du[i + 1] = -f * w.du[i + 1];
              }
              w.piv[i] = i + 1;
            }
          }
        }
        __syncwarp();
        const double tiny = eps * fmax(tnorm, 1e-300);
        for (int i = lane; i < n; i += 32) {
          double v = w.dd[i];
          if (fabs(v) < tiny) v = copysign(tiny, v == 0.0 ? 1.0 : v);
          w.dd[i] = v;
          w.rdd[i] = 1.0 / v;
          w.x[i] = 1.0 + 0.25 * sin(0.7 * (i + 1) + 1.3 * (c + 1));  // deterministic start
        }
        __syncwarp();
        for (int it = 0; it < 3; ++it) {
          if (lane == 0) {
            // solve (T - lm I) y = x (dgttrs): L then U
            for (int i = 0; i + 1 < n; ++i) {
              if (w.piv[i] == i) {
                w.x[i + 1] -= w.dl[i] * w.x[i];
              } else {
                const double tmp = w.x[i];
                w.x[i] = w.x[i + 1];
                w.x[i + 1] = tmp - w.dl[i] * w.x[i];
              }
            }
            double x1 = w.x[n - 1] * w.rdd[n - 1], x2 = 0.0;
            w.x[n - 1] = x1;
            if (n >= 2) {
              x2 = x1;
              x1 = (w.x[n - 2] - w.du[n - 2] * x2) * w.rdd[n - 2];
              w.x[n - 2] = x1;
            }
            for (int i = n - 3; i >= 0; --i) {
              const double xi = (w.x[i] - w.du[i] * x1 - w.du2[i] * x2) * w.rdd[i];
              w.x[i] = xi;
              x2 = x1;
              x1 = xi;
            }
          }
          __syncwarp();
          for (int c2 = c0; c2 < c; ++c2) {  // orthogonalize against earlier members (rows of Vt)
            const double* u = Vt + static_cast<i64>(c2) * n;
            double s = 0.0;
            for (int i = lane; i < n; i += 32) s += w.x[i] * u[i];
            s = warp_sum(s);
            for (int i = lane; i < n; i += 32) w.x[i] -= s * u[i];
            __syncwarp();
          }
          double s2 = 0.0;
          for (int i = lane; i < n; i += 32) s2 += w.x[i] * w.x[i];
          const double inv = 1.0 / sqrt(warp_sum(s2));
          for (int i = lane; i < n; i += 32) w.x[i] *= inv;
          __syncwarp();
        }
        for (int i = lane; i < n; i += 32) Vt[static_cast<i64>(c) * n + i] = w.x[i];
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // ---- back-transform every vector: z <- H_0 ... H_{n-3} z (a warp per vector)
  {
    double* x = btx + warp * kEigMaxN;
    for (int c = warp; c < n_vec; c += kEigWarps) {
      for (int i = lane; i < n; i += 32) x[i] = Vt[static_cast<i64>(c) * n + i];
      __syncwarp();
      for (int k = n - 3; k >= 0; --k) {
        const double t = tau[k];
        if (t == 0.0) continue;
        const int m = n - k - 1;
        const double* hv = Hv + k * kEigMaxN + k + 1;  // v_i = hv[i], v_0 = 1
        double sdot = 0.0;
        for (int i = lane; i < m; i += 32) sdot += hv[i] * x[k + 1 + i];
        sdot = t * warp_sum(sdot);
        for (int i = lane; i < m; i += 32) x[k + 1 + i] -= sdot * hv[i];
        __syncwarp();
      }
      for (int i = lane; i < n; i += 32) V[i * n + c] = x[i];
      __syncwarp();
    }
  }
  __syncthreads();
}

std::size_t tri_eig_smem(int n) {
  return sizeof(double) * (static_cast<std::size_t>(n) * kEigMaxN + (8 + kEigGroups) * kEigMaxN) +
         sizeof(TriWork) * kEigIIWarps + sizeof(double) * kEigWarps * kEigMaxN;
}

// ---------------------------------------------------------- finalize ----
// Lt: [q][M] lifted vectors (descending).  Keeps up to L_max vectors with
// tilde > cut after Riemann MGS (eigensolve.hpp:161-176).
__global__ void __launch_bounds__(1024) k_finalize(const double* __restrict__ Lt, const double* __restrict__ tilde,
                                                   i64 M, int q, int L_max, double cut, double cv,
                                                   double* __restrict__ kept, int* __restrict__ kept_src,
                                                   int* __restrict__ n_kept, int gram_schmidt, int n_avail,
                                                   int* __restrict__ exhausted) {
  pdl_wait();
  __shared__ double red[33];
  __shared__ i64 first_nz;
  int nk = 0;
  if (threadIdx.x == 0) *exhausted = 0;
  for (int l = 0; l < q && nk < L_max; ++l) {
    if (!(tilde[l] > cut)) break;
    if (l >= n_avail) {  // a candidate without a computed vector: the caller recomputes them all
      if (threadIdx.x == 0) *exhausted = 1;
      break;
    }
    double* v = kept + static_cast<i64>(nk) * M;
    for (i64 i = threadIdx.x; i < M; i += blockDim.x) v[i] = Lt[static_cast<i64>(l) * M + i];
    __syncthreads();
    for (int u = 0; u < (gram_schmidt ? nk : 0); ++u) {
      const double* uv = kept + static_cast<i64>(u) * M;
      double s = 0.0;
      for (i64 i = threadIdx.x; i < M; i += blockDim.x) s += uv[i] * v[i];
      const double coef = cv * block_sum(s, red);
      for (i64 i = threadIdx.x; i < M; i += blockDim.x) v[i] -= coef * uv[i];
      __syncthreads();
    }
    double s2 = 0.0;
    for (i64 i = threadIdx.x; i < M; i += blockDim.x) s2 += v[i] * v[i];
    const double norm = sqrt(cv * block_sum(s2, red));
    if (gram_schmidt && !(norm > 1e-10)) continue;  // dense_eig normalizes unconditionally
    for (i64 i = threadIdx.x; i < M; i += blockDim.x) v[i] /= norm;
    __syncthreads();
    double s1 = 0.0;
    for (i64 i = threadIdx.x; i < M; i += blockDim.x) s1 += v[i];
    double sgn = cv * block_sum(s1, red);
    if (fabs(sgn) < 1e-12 * sqrt(cv * static_cast<double>(M))) {
      if (threadIdx.x == 0) first_nz = M;
      __syncthreads();
      for (i64 i = threadIdx.x; i < M; i += blockDim.x)
        if (v[i] != 0.0) atomicMin(reinterpret_cast<unsigned long long*>(&first_nz),
                                   static_cast<unsigned long long>(i));
      __syncthreads();
      sgn = first_nz < M ? v[first_nz] : 0.0;
    }
    if (sgn < 0.0)
      for (i64 i = threadIdx.x; i < M; i += blockDim.x) v[i] = -v[i];
    __syncthreads();
    if (threadIdx.x == 0) kept_src[nk] = l;
    ++nk;
  }
  if (threadIdx.x == 0) *n_kept = nk;
}

__global__ void k_residual_norms(const double* __restrict__ SV, const double* __restrict__ V, i64 M, i64 L,
                                 const double* __restrict__ lam, double cv, double* __restrict__ out) {
  pdl_wait();
  __shared__ double red[33];
  const i64 l = blockIdx.x;
  double s = 0.0;
  for (i64 i = threadIdx.x; i < M; i += blockDim.x) {
    const double r = cv * SV[i * L + l] - lam[l] * V[i * L + l];
    s += r * r;
  }
  const double t = block_sum(s, red);
  if (threadIdx.x == 0) out[l] = sqrt(cv * t);
}

}  // namespace

struct MatrixView {
  DevBuf<double> owned;
  const double* sigma = nullptr;
  i64 M = 0;
  std::vector<i64> node_of_row;
};

static MatrixView matrixize_dev(dfpca_context* ctx, const dfpca_surface* cov, const Grid& grid) {
  MatrixView mv;
  const i64 G = grid.G;
  for (i64 f = 0; f < G; ++f)
    if (!grid.has_mask || grid.mask[f]) mv.node_of_row.push_back(f);
  mv.M = static_cast<i64>(mv.node_of_row.size());
  if (mv.M == 0) fail(kConfig, "InvalidArgument", "no in-mask nodes to decompose");
  if (mv.M == G) {
    mv.sigma = cov->values.get();
  } else {
    DevBuf<i64> nor(static_cast<std::size_t>(mv.M));
    DFPCA_CUDA(cudaMemcpyAsync(nor.get(), mv.node_of_row.data(), sizeof(i64) * mv.M,
                               cudaMemcpyHostToDevice, ctx->stream));
    mv.owned.alloc(static_cast<std::size_t>(mv.M * mv.M));
    DFPCA_LAUNCH(ctx, k_gather_sigma, grid_for(mv.M * mv.M, 256), 256, 0, cov->values.get(), G,
                 nor.get(), mv.M, mv.owned.get());
    mv.sigma = mv.owned.get();
    DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return mv;
}

// This rank's rows of the in-mask matrix of a row-sharded covariance:
// sigma_t = (Sigma[own in-mask rows][all in-mask columns])^T, [M][m_loc],
// and every rank's row count / offset (in-mask rows are in node order, and
// the slabs are consecutive node ranges).
struct RowShard {
  i64 M = 0, m_loc = 0, m_max = 0;
  std::vector<i64> node_of_row;
  std::vector<i64> counts, offsets;
  DevBuf<double> sigma_t;
};

__global__ void k_gather_rows(const double* __restrict__ slab, i64 G, i64 row0, const i64* __restrict__ rows_nodes,
                              i64 m_loc, const i64* __restrict__ node_of_row, i64 M, double* __restrict__ out) {
  pdl_wait();
  const i64 total = m_loc * M;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / M, c = e % M;
    out[e] = slab[(rows_nodes[r] - row0) * G + node_of_row[c]];
  }
}

static RowShard shard_rows_dev(dfpca_context* ctx, Transport& tr, const dfpca_surface* cov, const Grid& grid) {
  RowShard rs;
  const i64 G = grid.G;
  for (i64 f = 0; f < G; ++f)
    if (!grid.has_mask || grid.mask[f]) rs.node_of_row.push_back(f);
  rs.M = static_cast<i64>(rs.node_of_row.size());
  if (rs.M == 0) fail(kConfig, "InvalidArgument", "no in-mask nodes to decompose");
  const i64 row0 = cov->row0, nrows = cov->rows >= 0 ? cov->rows : G;
  std::vector<i64> mine;
  for (i64 r = 0; r < rs.M; ++r) {
    const i64 f = rs.node_of_row[static_cast<std::size_t>(r)];
    if (f >= row0 && f < row0 + nrows) mine.push_back(f);
  }
  rs.m_loc = static_cast<i64>(mine.size());
  // every rank's in-mask row count (all-gathered), hence offsets and padding
  const int W = tr.world();
  DevBuf<double> cnt(1), cnts(static_cast<std::size_t>(W));
  const double c = static_cast<double>(rs.m_loc);
  DFPCA_CUDA(cudaMemcpyAsync(cnt.get(), &c, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  tr.all_gather(ctx, cnt.get(), cnts.get(), 1);
  std::vector<double> hc(static_cast<std::size_t>(W));
  DFPCA_CUDA(cudaMemcpyAsync(hc.data(), cnts.get(), sizeof(double) * W, cudaMemcpyDeviceToHost, ctx->stream));
  DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  i64 off = 0;
  for (int r = 0; r < W; ++r) {
    rs.counts.push_back(static_cast<i64>(hc[static_cast<std::size_t>(r)]));
    rs.offsets.push_back(off);
    off += rs.counts.back();
    rs.m_max = std::max(rs.m_max, rs.counts.back());
  }
  if (off != rs.M) fail(kConfig, "InvalidArgument", "covariance slabs do not cover the grid once");
  if (rs.m_loc > 0) {
    DevBuf<i64> nodes(static_cast<std::size_t>(rs.m_loc)), nor(static_cast<std::size_t>(rs.M));
    DFPCA_CUDA(cudaMemcpyAsync(nodes.get(), mine.data(), sizeof(i64) * rs.m_loc, cudaMemcpyHostToDevice,
                               ctx->stream));
    DFPCA_CUDA(cudaMemcpyAsync(nor.get(), rs.node_of_row.data(), sizeof(i64) * rs.M, cudaMemcpyHostToDevice,
                               ctx->stream));
    DevBuf<double> rows(static_cast<std::size_t>(rs.m_loc * rs.M));
    DFPCA_LAUNCH(ctx, k_gather_rows, grid_for(rs.m_loc * rs.M, 256), 256, 0, cov->values.get(), G, row0,
                 nodes.get(), rs.m_loc, nor.get(), rs.M, rows.get());
    rs.sigma_t.alloc(static_cast<std::size_t>(rs.m_loc * rs.M));
    transpose(ctx, rows.get(), rs.m_loc, rs.M, rs.sigma_t.get());
    DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return rs;
}

// finalize_eigensystem (eigensolve.hpp:146-194) on the device: candidates Lt
// [q][M] in descending order of tilde (host copy tilde_h, device tilde_d).
// Returns false (nothing written) when a kept candidate had no computed
// vector (n_avail < the candidates the finalization reached).
static bool finish_eigensystem(dfpca_context* ctx, const Grid& grid, const std::vector<i64>& node_of_row, i64 M,
                               const double* Lt, const double* tilde_d, const std::vector<double>& tilde,
                               i64 L_max, bool gram_schmidt, double* eigenvalues, double* eigenfunctions,
                               double* fve, double* total_variance, i64* n_components, i64 n_avail = -1,
                               const double* tilde_total_in = nullptr) {
  cudaStream_t st = ctx->stream;
  const i64 q = static_cast<i64>(tilde.size());
  const double cv = grid.cell_volume();
  const double cut = tilde.empty() ? 0.0 : std::max(0.0, tilde[0]) * 1e-12;
  double tilde_total = 0.0;
  for (double t : tilde)
    if (t > cut) tilde_total += t;
  if (tilde_total_in) tilde_total = *tilde_total_in;  // a partial spectrum: the caller's sum over the cut
  const double total = tilde_total * cv;

  DevBuf<double> kept(static_cast<std::size_t>(std::max<i64>(L_max, 1) * M));
  DevBuf<int> kept_src(static_cast<std::size_t>(std::max<i64>(L_max, 1))), nkept(2);
  DFPCA_LAUNCH(ctx, k_finalize, 1, 1024, 0, Lt, tilde_d, M, static_cast<int>(q), static_cast<int>(L_max), cut,
               cv, kept.get(), kept_src.get(), nkept.get(), gram_schmidt ? 1 : 0,
               static_cast<int>(n_avail < 0 ? q : n_avail), nkept.get() + 1);
  int nk2[2] = {0, 0};
  DFPCA_CUDA(cudaMemcpyAsync(nk2, nkept.get(), sizeof(nk2), cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
  if (nk2[1] != 0) return false;
  const int nk = nk2[0];
  std::vector<int> src(static_cast<std::size_t>(std::max(nk, 1)));
  std::vector<double> kv(static_cast<std::size_t>(nk) * M);
  if (nk > 0) {
    DFPCA_CUDA(cudaMemcpyAsync(src.data(), kept_src.get(), sizeof(int) * nk, cudaMemcpyDeviceToHost, st));
    DFPCA_CUDA(cudaMemcpyAsync(kv.data(), kept.get(), sizeof(double) * nk * M, cudaMemcpyDeviceToHost, st));
  }
  DFPCA_CUDA(cudaStreamSynchronize(st));
  ctx->end_stage();

  const i64 G = grid.G;
  double cum = 0.0;
  for (int l = 0; l < nk; ++l) {
    const double lam = tilde[static_cast<std::size_t>(src[l])] * cv;
    if (eigenvalues) eigenvalues[l] = lam;
    cum += lam;
    if (fve) fve[l] = total > 0.0 ? cum / total : 1.0;
    if (eigenfunctions) {
      double* surf = eigenfunctions + static_cast<i64>(l) * G;
      for (i64 f = 0; f < G; ++f) surf[f] = std::nan("");
      for (i64 r = 0; r < M; ++r) surf[node_of_row[static_cast<std::size_t>(r)]] = kv[static_cast<std::size_t>(l) * M + r];
    }
  }
  if (total_variance) *total_variance = total;
  if (n_components) *n_components = nk;
  return true;
}


void run_randomized_eig(dfpca_context* ctx, const dfpca_surface* cov, const Grid& grid, i64 q_req,
                        i64 L_max, unsigned long long seed, double* eigenvalues, double* eigenfunctions,
                        double* fve, double* total_variance, i64* n_components) {
  if (cov->kind != DFPCA_SURFACE_COVARIANCE)
    fail(kConfig, "InvalidArgument", "matrixize expects a covariance surface");
  Transport* tr = ctx->transport && ctx->transport->world() > 1 ? ctx->transport.get() : nullptr;
  const i64 cov_rows = cov->rows >= 0 ? cov->rows : grid.G;
  if (cov->n != cov_rows * grid.G || (!tr && cov_rows != grid.G))
    fail(kConfig, "InvalidArgument", "covariance surface has wrong length");
  if (q_req < L_max)
    fail(kConfig, "SketchTooSmall",
         "sketch size " + std::to_string(q_req) + " is below the requested component count " +
             std::to_string(L_max));
  cudaStream_t st = ctx->stream;
  ctx->begin_stage("eigen");
  // One device: the in-mask matrix.  Row-sharded (a slab of a sharded
  // covariance on every rank): this rank's in-mask rows, transposed into the
  // K-major operand, and the two products with Sigma are all-gathered.
  MatrixView mv = tr ? MatrixView{} : matrixize_dev(ctx, cov, grid);
  RowShard rs;
  if (tr) {
    rs = shard_rows_dev(ctx, *tr, cov, grid);
    mv.M = rs.M;
    mv.node_of_row = rs.node_of_row;
  }
  const i64 M = mv.M;
  const i64 q = std::min<i64>(q_req, M);
  // [M][q] operands are stored with an even row stride ldq so the GEMM
  // operand copies are 16-byte cp.async (the padding column is never read)
  const i64 ldq = (q + 1) & ~1ll;
  // out[M][ldq] = Sigma X for X [M][ldq]: sums split exactly as the
  // one-device product (same split-K), so every row is bit-identical
  // columns [c0, c0 + nc) of out = Sigma X (column blocks: a sharded run
  // splits exactly like the one-device run, so the rows are bit-identical)
  auto apply_sigma = [&](const double* X, double* out, i64 c0, i64 nc) {
    if (!tr) {
      gemm_tn(ctx, M, nc, M, mv.sigma, M, nullptr, X + c0, ldq, out + c0, ldq, false);
      return;
    }
    const i64 chunk = std::max<i64>(1, rs.m_max * ldq);
    DevBuf<double> loc(static_cast<std::size_t>(chunk));
    DFPCA_CUDA(cudaMemsetAsync(loc.get(), 0, sizeof(double) * chunk, st));
    if (rs.m_loc > 0)
      gemm_tn(ctx, rs.m_loc, nc, M, rs.sigma_t.get(), rs.m_loc, nullptr, X + c0, ldq, loc.get() + c0, ldq, false, 0,
              -1, gemm_splits(ctx, M, nc, M));
    DevBuf<double> all(static_cast<std::size_t>(tr->world() * chunk));
    tr->all_gather(ctx, loc.get(), all.get(), chunk);
    for (int r = 0; r < tr->world(); ++r)
      if (rs.counts[static_cast<std::size_t>(r)] > 0)
        DFPCA_CUDA(cudaMemcpy2DAsync(out + rs.offsets[static_cast<std::size_t>(r)] * ldq + c0, sizeof(double) * ldq,
                                     all.get() + static_cast<i64>(r) * chunk + c0, sizeof(double) * ldq,
                                     sizeof(double) * nc, static_cast<std::size_t>(rs.counts[static_cast<std::size_t>(r)]),
                                     cudaMemcpyDeviceToDevice, st));
  };

  // Omega and Y = Sigma Omega ([M][q]; Sigma is exactly symmetric, so
  // Sigma(k, m) is the K-major operand), pipelined by column blocks: the
  // one-CTA Mersenne Twister runs on the aux stream and stops after the
  // words of the first 64 columns (rounded up to whole twists, its state
  // saved); while it produces the rest, the first block's Box-Muller and
  // product run on the context stream.
  const i64 n_words = 2 * ((M * q + 1) / 2);
  const i64 pairs_total = (M * q + 1) / 2;
  const i64 c1 = std::min<i64>(q, 64);
  const i64 w1 = std::min<i64>(n_words, ((c1 * M + kMtN - 1) / kMtN) * kMtN);
  DevBuf<unsigned long long> words(static_cast<std::size_t>(n_words)), mt_state(kMtN);
  DevBuf<double> omega(static_cast<std::size_t>(M * ldq));
  DevBuf<double> Y(static_cast<std::size_t>(M * ldq));
  const double sd = 1.0 / std::sqrt(static_cast<double>(q));
  {
    cudaStream_t aux = ctx->aux_stream();
    cudaEvent_t ev[3];
    for (auto& e : ev) DFPCA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct Evs {
      cudaEvent_t* e;
      ~Evs() {
        for (int i = 0; i < 3; ++i) cudaEventDestroy(e[i]);
      }
    } evs{ev};
    DFPCA_CUDA(cudaEventRecord(ev[0], st));  // the buffers' stream-ordered allocations
    DFPCA_CUDA(cudaStreamWaitEvent(aux, ev[0], 0));
    {
      struct AuxLaunch {  // launches below go to the aux stream
        dfpca_context* c;
        cudaStream_t saved;
        AuxLaunch(dfpca_context* c_, cudaStream_t s) : c(c_), saved(c_->stream) { c->stream = s; }
        ~AuxLaunch() { c->stream = saved; }
      } on_aux(ctx, aux);
      DFPCA_LAUNCH(ctx, k_mt19937_64, 1, kMtN, 0, splitmix64(seed), w1, words.get(), mt_state.get(), 0);
      DFPCA_CUDA(cudaEventRecord(ev[1], aux));
      if (w1 < n_words)
        DFPCA_LAUNCH(ctx, k_mt19937_64, 1, kMtN, 0, 0ull, n_words - w1, words.get() + w1, mt_state.get(), 1);
      DFPCA_CUDA(cudaEventRecord(ev[2], aux));
    }
    DFPCA_CUDA(cudaStreamWaitEvent(st, ev[1], 0));
    // Box-Muller pairs of the first block: its columns hold c1 * M normals
    // (even: c1 = 64 when there is a second block); one block takes them all
    const i64 p_split = c1 < q ? (c1 * M) / 2 : pairs_total;
    DFPCA_LAUNCH(ctx, k_box_muller, grid_for(p_split, 256), 256, 0, words.get(), M, q, ldq, sd, 0ll, p_split,
                 omega.get());
    apply_sigma(omega.get(), Y.get(), 0, c1);
    DFPCA_CUDA(cudaStreamWaitEvent(st, ev[2], 0));
    if (c1 < q) {
      DFPCA_LAUNCH(ctx, k_box_muller, grid_for(pairs_total - p_split, 256), 256, 0, words.get(), M, q, ldq, sd,
                   p_split, pairs_total, omega.get());
      apply_sigma(omega.get(), Y.get(), c1, q - c1);
    }
  }

  // Thin Q with range(Q) = range(Y) (eigensolve.hpp:260-263; any orthonormal
  // basis of range(Y) gives the same Ritz pairs): Cholesky QR twice -- two
  // DMMA Gram products and two fused factor+solve passes -- accepted when
  // the first pass left Q1 within 0.1 of orthonormal (then the second pass
  // restores orthogonality to rounding); otherwise (nearly rank-deficient
  // sketches) Householder QR, one reflector per launch.
  // The Cholesky-QR acceptance flags are read at the stage's one host sync
  // (with the Ritz values), so nothing waits in between; a rejected sketch
  // reruns the rest from Y with shifted Cholesky QR, then Householder QR.
  // mode 0: Cholesky QR twice; 1: shifted Cholesky QR three times (sketches
  // too ill-conditioned for mode 0, cond up to ~1/u); 2: Householder QR
  auto from_Y = [&](int mode) -> bool {
    const bool cholqr = mode < 2;
    DevBuf<double> Q(static_cast<std::size_t>(M * ldq)), Qt(static_cast<std::size_t>(M * q)), flags(8);
    if (cholqr) {
      DevBuf<double> G(static_cast<std::size_t>(q * q)), R(static_cast<std::size_t>(q * q)),
          Qa(static_cast<std::size_t>(M * ldq)), Qb(static_cast<std::size_t>(M * ldq));
      const int qi = static_cast<int>(q);
      const std::size_t fsm = sizeof(double) * q * (q + 1), tsm = trsm_smem(qi);
      allow_smem(k_chol_factor, fsm);
      allow_smem(k_row_trsm, tsm);
      const unsigned ctas =
          static_cast<unsigned>(std::min<i64>((M + kTrsmWarps - 1) / kTrsmWarps, 2 * ctx->sm_count));
      const int passes = mode == 0 ? 2 : 3;
      const double shift_scale =
          11.0 * (static_cast<double>(M) * q + static_cast<double>(q) * (q + 1)) * 1.1102230246251565e-16;
      const double* src = Y.get();
      for (int ps = 0; ps < passes; ++ps) {
        double* dst = ps == passes - 1 ? Q.get() : (ps % 2 == 0 ? Qa.get() : Qb.get());
        gemm_tn(ctx, q, q, M, src, ldq, nullptr, src, ldq, G.get(), q, false);
        DFPCA_LAUNCH(ctx, k_chol_factor, 1, 1024, fsm, G.get(), qi, R.get(), flags.get() + 2 * ps,
                     mode == 1 && ps == 0 ? shift_scale : 0.0);
        DFPCA_LAUNCH(ctx, k_row_trsm, ctas, kTrsmWarps * 32, tsm, src, M, qi, ldq, R.get(), flags.get() + 2 * ps,
                     dst);
        src = dst;
      }
      transpose(ctx, Q.get(), M, q, Qt.get(), ldq, M);
    } else {
      DevBuf<double> Yt(static_cast<std::size_t>(M * q)), tau(static_cast<std::size_t>(q));
      transpose(ctx, Y.get(), M, q, Yt.get(), ldq, M);
      for (i64 j = -1; j < q - 1; ++j) {
        const i64 cols = q - (j + 1);
        DFPCA_LAUNCH(ctx, k_house_step, static_cast<unsigned>(cols), 512, 0, Yt.get(), M, q, j, tau.get());
      }
      DFPCA_LAUNCH(ctx, k_q_init, grid_for(M * q, 256), 256, 0, Qt.get(), M, q);
      for (i64 j = q - 1; j >= 0; --j)
        DFPCA_LAUNCH(ctx, k_q_apply, static_cast<unsigned>(q - j), 512, 0, Yt.get(), tau.get(), M, q, j,
                     Qt.get());
      transpose(ctx, Qt.get(), q, M, Q.get(), M, ldq);
    }

    // small = Q^T (Sigma Q)
    DevBuf<double> Z(static_cast<std::size_t>(M * ldq));
    apply_sigma(Q.get(), Z.get(), 0, q);
    DevBuf<double> small(static_cast<std::size_t>(q * q)), Vs(static_cast<std::size_t>(q * q));
    gemm_tn(ctx, q, q, M, Q.get(), ldq, nullptr, Z.get(), ldq, small.get(), q, false);

    DevBuf<double> evals(static_cast<std::size_t>(q)), Vt(static_cast<std::size_t>(q * q));
    DevBuf<int> info(static_cast<std::size_t>(q + 2));
    const bool tri = q <= kEigMaxN;
    // vectors for the leading L_max + 4 candidates (more only if the
    // finalization skips that many: then all of them, below)
    i64 max_vec = std::min<i64>(q, L_max + DFPCA_EIG_VEC_MARGIN);
    auto tri_eig = [&](i64 mv_) {
      const std::size_t tsm = tri_eig_smem(static_cast<int>(q));
      allow_smem(k_tri_eig, tsm);
      DFPCA_LAUNCH(ctx, k_tri_eig, 1, kEigThreads, tsm, small.get(), static_cast<int>(q), evals.get(), Vs.get(),
                   info.get(), static_cast<int>(mv_), Vt.get(), cholqr ? flags.get() : nullptr,
                   mode == 0 ? 2 : 3);
    };
    if (tri) {
      tri_eig(max_vec);
    } else {
      const int np = static_cast<int>((q + 1) & ~1ll);
      std::size_t jsmem = sizeof(double) * np * 2;
      const bool jac_smem = jsmem + sizeof(double) * 2 * q * q <= 200 * 1024;
      if (jac_smem) {
        jsmem += sizeof(double) * 2 * q * q;
        allow_smem(k_jacobi, jsmem);
      }
      DFPCA_LAUNCH(ctx, k_jacobi, 1, 1024, jsmem, small.get(), Vs.get(), static_cast<int>(q), evals.get(),
                   info.get(), jac_smem ? 1 : 0);
    }

    // lifted = Q V  ([M][q]) -> Lt [q][M]
    DevBuf<double> lifted(static_cast<std::size_t>(M * q)), Lt(static_cast<std::size_t>(M * q));
    gemm_tn(ctx, M, q, q, Qt.get(), M, nullptr, Vs.get(), q, lifted.get(), q, false);
    transpose(ctx, lifted.get(), M, q, Lt.get());

    std::vector<double> tilde(static_cast<std::size_t>(q));
    int jinfo = 0;
    double hf[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    DFPCA_CUDA(cudaMemcpyAsync(tilde.data(), evals.get(), sizeof(double) * q, cudaMemcpyDeviceToHost, st));
    DFPCA_CUDA(cudaMemcpyAsync(&jinfo, info.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    if (cholqr) DFPCA_CUDA(cudaMemcpyAsync(hf, flags.get(), sizeof(hf), cudaMemcpyDeviceToHost, st));
    DFPCA_CUDA(cudaStreamSynchronize(st));
    if (cholqr && !qr_accepted(hf, mode == 0 ? 2 : 3)) return false;
    if (!tri && jinfo != 0) fail(kNumeric, "EigFailure", "projected eigensolver did not converge");

    if (!finish_eigensystem(ctx, grid, mv.node_of_row, M, Lt.get(), evals.get(), tilde, L_max, true, eigenvalues,
                            eigenfunctions, fve, total_variance, n_components, tri ? max_vec : q)) {
      // more candidates were skipped than the margin covered: all vectors
      tri_eig(q);
      gemm_tn(ctx, M, q, q, Qt.get(), M, nullptr, Vs.get(), q, lifted.get(), q, false);
      transpose(ctx, lifted.get(), M, q, Lt.get());
      finish_eigensystem(ctx, grid, mv.node_of_row, M, Lt.get(), evals.get(), tilde, L_max, true, eigenvalues,
                         eigenfunctions, fve, total_variance, n_components);
    }
    return true;
  };
  if (!(q <= kCqMaxQ && (from_Y(0) || from_Y(1)))) from_Y(2);
}


// ---- dense_eig (eigensolve.hpp:205-228): cuSOLVER syevd on the device ----
namespace {
struct CusolverApi {
  using Handle = void*;
  int (*Create)(Handle*) = nullptr;
  int (*Destroy)(Handle) = nullptr;
  int (*SetStream)(Handle, cudaStream_t) = nullptr;
  int (*DsyevdBufferSize)(Handle, int, int, int, const double*, int, const double*, int*) = nullptr;
  int (*Dsyevd)(Handle, int, int, int, double*, int, double*, double*, int, int*) = nullptr;
  static constexpr int kEigModeVector = 1, kFillLower = 0;
  static CusolverApi& get() {
    static CusolverApi api;
    static bool tried = false;
    if (!tried) {
      tried = true;
      std::vector<std::string> names;
      if (const char* e = std::getenv("DFPCA_CUSOLVER_LIB")) names.push_back(e);
      names.push_back("libcusolver.so.11");
      void* h = nullptr;
      for (const auto& n : names)
        if ((h = dlopen(n.c_str(), RTLD_NOW | RTLD_GLOBAL))) break;
      if (h) {
        api.Create = reinterpret_cast<decltype(api.Create)>(dlsym(h, "cusolverDnCreate"));
        api.Destroy = reinterpret_cast<decltype(api.Destroy)>(dlsym(h, "cusolverDnDestroy"));
        api.SetStream = reinterpret_cast<decltype(api.SetStream)>(dlsym(h, "cusolverDnSetStream"));
        api.DsyevdBufferSize =
            reinterpret_cast<decltype(api.DsyevdBufferSize)>(dlsym(h, "cusolverDnDsyevd_bufferSize"));
        api.Dsyevd = reinterpret_cast<decltype(api.Dsyevd)>(dlsym(h, "cusolverDnDsyevd"));
      }
    }
    if (!api.Create || !api.Dsyevd || !api.DsyevdBufferSize || !api.SetStream)
      fail(kConfig, "InvalidArgument", "libcusolver.so.11 could not be loaded (set DFPCA_CUSOLVER_LIB)");
    return api;
  }
};

__global__ void k_reverse_rows(const double* __restrict__ in, i64 rows, i64 cols, double* __restrict__ out) {
  pdl_wait();
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < rows * cols; e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / cols, c = e % cols;
    out[(rows - 1 - r) * cols + c] = in[e];
  }
}
}  // namespace

bool dense_top_eigenpairs(dfpca_context* ctx, const double* sigma, i64 M, int count, double cut_rel,
                          std::vector<double>& lam_out, double* vecs, double& above_cut);

void run_dense_eig(dfpca_context* ctx, const dfpca_surface* cov, const Grid& grid, i64 L_max, double* eigenvalues,
                   double* eigenfunctions, double* fve, double* total_variance, i64* n_components) {
  if (cov->kind != DFPCA_SURFACE_COVARIANCE)
    fail(kConfig, "InvalidArgument", "matrixize expects a covariance surface");
  if (cov->n != grid.G * grid.G) fail(kConfig, "InvalidArgument", "covariance surface has wrong length");
  cudaStream_t st = ctx->stream;
  ctx->begin_stage("eigen");
  MatrixView mv = matrixize_dev(ctx, cov, grid);
  const i64 M = mv.M;
  if (M > (i64(1) << 31) / M) fail(kConfig, "InvalidArgument", "matrix too large for the dense eigensolver");
  // The hand-written path (dense_eig.cu) unless DFPCA_DENSE_EIG=cusolver;
  // it declines (and cuSOLVER's syevd runs) outside its size range.
  const char* mode = std::getenv("DFPCA_DENSE_EIG");
  const int count = static_cast<int>(std::min<i64>(L_max, M));
  if (!(mode && std::string(mode) == "cusolver") && count >= 1) {
    std::vector<double> lam;
    double above = 0.0;
    DevBuf<double> vecs(static_cast<std::size_t>(count) * M), td(static_cast<std::size_t>(count));
    if (dense_top_eigenpairs(ctx, mv.sigma, M, count, 1e-12, lam, vecs.get(), above)) {
      DFPCA_CUDA(cudaMemcpyAsync(td.get(), lam.data(), sizeof(double) * count, cudaMemcpyHostToDevice, st));
      finish_eigensystem(ctx, grid, mv.node_of_row, M, vecs.get(), td.get(), lam, L_max, false, eigenvalues,
                         eigenfunctions, fve, total_variance, n_components, -1, &above);
      return;
    }
  }
  CusolverApi& api = CusolverApi::get();
  // A = Sigma (symmetric: row-major == column-major), overwritten by the eigenvectors
  DevBuf<double> A(static_cast<std::size_t>(M * M)), w(static_cast<std::size_t>(M));
  DFPCA_CUDA(cudaMemcpyAsync(A.get(), mv.sigma, sizeof(double) * M * M, cudaMemcpyDeviceToDevice, st));
  CusolverApi::Handle h = nullptr;
  if (api.Create(&h) != 0) fail(kNumeric, "DeviceError", "cusolverDnCreate failed");
  struct Guard {
    CusolverApi& a;
    CusolverApi::Handle h;
    ~Guard() { a.Destroy(h); }
  } guard{api, h};
  api.SetStream(h, st);
  int lwork = 0;
  if (api.DsyevdBufferSize(h, CusolverApi::kEigModeVector, CusolverApi::kFillLower, static_cast<int>(M), A.get(),
                           static_cast<int>(M), w.get(), &lwork) != 0)
    fail(kNumeric, "DeviceError", "cusolverDnDsyevd_bufferSize failed");
  DevBuf<double> work(static_cast<std::size_t>(std::max(lwork, 1)));
  DevBuf<int> info(1);
  if (api.Dsyevd(h, CusolverApi::kEigModeVector, CusolverApi::kFillLower, static_cast<int>(M), A.get(),
                 static_cast<int>(M), w.get(), work.get(), lwork, info.get()) != 0)
    fail(kNumeric, "DeviceError", "cusolverDnDsyevd failed");
  int hinfo = 0;
  std::vector<double> wa(static_cast<std::size_t>(M));
  DFPCA_CUDA(cudaMemcpyAsync(&hinfo, info.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaMemcpyAsync(wa.data(), w.get(), sizeof(double) * M, cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
  if (hinfo != 0)
    fail(kNumeric, "EigFailure", "symmetric eigensolver did not converge (info=" + std::to_string(hinfo) + ")");
  // ascending -> descending; column j of the column-major A is row j here
  std::vector<double> tilde(wa.rbegin(), wa.rend());
  DevBuf<double> Lt(static_cast<std::size_t>(M * M)), td(static_cast<std::size_t>(M));
  DFPCA_LAUNCH(ctx, k_reverse_rows, grid_for(M * M, 256, 148ll * 32), 256, 0, A.get(), M, M, Lt.get());
  DFPCA_CUDA(cudaMemcpyAsync(td.get(), tilde.data(), sizeof(double) * M, cudaMemcpyHostToDevice, st));
  finish_eigensystem(ctx, grid, mv.node_of_row, M, Lt.get(), td.get(), tilde, L_max, false, eigenvalues,
                     eigenfunctions, fve, total_variance, n_components);
}

void run_eig_residuals(dfpca_context* ctx, const dfpca_surface* cov, const Grid& grid, i64 L,
                       const double* eigenvalues, const double* eigenfunctions, double* residuals) {
  if (L <= 0) return;
  MatrixView mv = matrixize_dev(ctx, cov, grid);
  const i64 M = mv.M;
  std::vector<double> V(static_cast<std::size_t>(M * L));
  for (i64 l = 0; l < L; ++l)
    for (i64 r = 0; r < M; ++r)
      V[static_cast<std::size_t>(r * L + l)] = eigenfunctions[l * grid.G + mv.node_of_row[static_cast<std::size_t>(r)]];
  DevBuf<double> Vd(V.size()), SV(V.size()), lam(static_cast<std::size_t>(L)), out(static_cast<std::size_t>(L));
  cudaStream_t st = ctx->stream;
  DFPCA_CUDA(cudaMemcpyAsync(Vd.get(), V.data(), sizeof(double) * V.size(), cudaMemcpyHostToDevice, st));
  DFPCA_CUDA(cudaMemcpyAsync(lam.get(), eigenvalues, sizeof(double) * L, cudaMemcpyHostToDevice, st));
  gemm_tn(ctx, M, L, M, mv.sigma, M, nullptr, Vd.get(), L, SV.get(), L, false);
  DFPCA_LAUNCH(ctx, k_residual_norms, static_cast<unsigned>(L), 256, 0, SV.get(), Vd.get(), M, L, lam.get(),
               grid.cell_volume(), out.get());
  DFPCA_CUDA(cudaMemcpyAsync(residuals, out.get(), sizeof(double) * L, cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
}

}  // namespace dfpca_gpu
