// Wide-bandwidth t-phase on the FP64 tensor pipe (AxisConv at large radius,
// reference conv.hpp:76-213, which switches to overlap-add FFT at 33 taps,
// conv.hpp:73).  A 1-D convolution of every line of a 64 x 64 plane with a
// (2R+1)-tap kernel is a product with a banded Toeplitz matrix,
//   Y = X B   with B[m][j] = taps[m - j + R]   (along t2, the rows of X),
//   Z = A Y   with A[j][m] = taps[m - j + R]   (along t1),
// so the two t passes of a pair-grid row become DMMA products (mma.sync
// m8n8k4 f64) restricted to the band: ~(2R + 8) multiply-adds per output
// instead of the direct kernel's 2R + 1 FMAs, but at the DMMA rate with 8x
// fewer instructions -- the direct kernels (conv_impl.cuh) become
// FMA/issue-bound as R grows, this one does not.  The Toeplitz fragments are
// read from zero-extended tap tables in shared memory (no branches); the
// plane is staged by cp.async, double-buffered across the persistent CTA's
// rows.  Same outputs, same upper-triangle trim (rows t1 >= j_lo(s)) as
// k_tphase2; the sums are reassociated (DMMA accumulation order), so parity
// with the reference is the 1e-10 surface bar, as for the reference's own FFT
// path.  Used from the measured crossover radius (conv.cu: run_tphase2).
#include <algorithm>
#include <cstdint>

#include "conv.cuh"
#include "conv_detail.cuh"

namespace dfpca_gpu {
namespace {

constexpr int kP = 64;            // plane edge handled (n1, n2 <= 64)
constexpr int kLd = kP + 4;       // smem row stride: 16-byte rows, 2-way bank access for the fragments
constexpr int kRows = kP + 4;     // plane rows incl. the zero rows a last k-step of 4 may touch
constexpr int kTc = kP + 8;       // centre of a zero-extended tap table
constexpr int kTz = 2 * kTc + 1;  // taps at offsets o in [-72, 72] (fragment offsets span [-63, 67])
constexpr int kWarps = 8, kThreadsM = 32 * kWarps;

__device__ inline void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ inline void cp16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ inline void cp8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ inline void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ inline void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct MmaTaps {
  double t[2][3][kTz];  // [axis t1/t2][order][o + kTc], zero outside |o| <= R_axis
};

__global__ void __launch_bounds__(kThreadsM, 2)
    k_tphase2_mma(const double* __restrict__ pw, const double* __restrict__ pv, i64 rows, int n1, int n2,
                  int value_only, conv_detail::TPhaseOut out, const MmaTaps* __restrict__ taps_g, int R1, int R2) {
  pdl_wait();
  extern __shared__ __align__(16) double sm[];
  double* Xb = sm;                      // [2][kRows][kLd]
  double* Y = sm + 2 * kRows * kLd;     // [kRows][kLd]
  double* tz = Y + kRows * kLd;         // MmaTaps
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 3 * kRows * kLd; e += blockDim.x) sm[e] = 0.0;  // zero padding rows / columns
  for (int e = tid; e < 2 * 3 * kTz; e += blockDim.x) tz[e] = reinterpret_cast<const double*>(taps_g)[e];
  __syncthreads();
  const i64 plane = static_cast<i64>(n1) * n2;
  const bool vec = (n2 % 2 == 0) && ((reinterpret_cast<std::uintptr_t>(value_only ? pv : pw) & 15) == 0);
  auto j_lo_of = [&](i64 s) -> int {
    if (out.t1_margin < 0) return 0;
    const long long lo = (out.s_base + s) / out.rn - out.t1_margin;
    return lo <= 0 ? 0 : (lo >= n1 ? n1 : static_cast<int>(lo));
  };
  auto issue = [&](i64 s, int pass, int buf) {
    const double* src = (pass ? pv : pw) + s * plane;
    double* X = Xb + buf * kRows * kLd;
    if (vec) {
      const int per_row = n2 / 2;
      for (int e = tid; e < n1 * per_row; e += blockDim.x) {
        const int r = e / per_row, c = (e % per_row) * 2;
        cp16(X + r * kLd + c, src + r * n2 + c);
      }
    } else {
      for (int e = tid; e < n1 * n2; e += blockDim.x) cp8(X + (e / n2) * kLd + e % n2, src + e);
    }
  };
  // warp tile: 16 rows x 32 columns of the 64 x 64 plane
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32;
  const int lr = lane >> 2, lk = lane & 3;
  const int first_pass = value_only ? 1 : 0;
  i64 s = blockIdx.x;
  int pass = first_pass, buf = 0;
  if (s < rows) issue(s, pass, 0);
  cp_commit();
  while (s < rows) {
    const bool same_row = pass == 0;
    const i64 ns = same_row ? s : s + gridDim.x;
    const int npass = same_row ? 1 : first_pass;
    if (ns < rows) issue(ns, npass, buf ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const double* X = Xb + buf * kRows * kLd;
    const i64 off = s * plane;
    const int max_order = pass == 0 ? 2 : 1;
    const int j_lo = j_lo_of(s);
    for (int r2 = 0; r2 <= max_order; ++r2) {
      // ---- Y = X B_{r2}: along t2 (columns j of the plane)
      {
        const double* tb = tz + (1 * 3 + r2) * kTz + kTc;  // tap(o) = tb[o]
        double acc[2][4][2] = {};
        const int k0 = max(0, (wc - R2) & ~3), k1 = min(n2, wc + 32 + R2);
        for (int k = k0; k < k1; k += 4) {
          const int m = k + lk;
          double a[2], b[4];
#pragma unroll
          for (int i = 0; i < 2; ++i) a[i] = X[(wr + i * 8 + lr) * kLd + m];
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = tb[m - (wc + j * 8 + lr)];
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int row = wr + i * 8 + lr, col = wc + j * 8 + 2 * lk;
            if (row < n1) {
              if (col < n2) Y[row * kLd + col] = acc[i][j][0];
              if (col + 1 < n2) Y[row * kLd + col + 1] = acc[i][j][1];
            }
          }
      }
      __syncthreads();
      // ---- out_{r1} = A_{r1} Y: along t1, output rows t1 >= j_lo
      const int n_r1 = max_order - r2 + 1;  // orders r1 with r1 + r2 <= max_order
      double* outs[3];
      if (pass == 0) {
        const int base = r2 == 0 ? 0 : (r2 == 1 ? 3 : 5);
        for (int r1 = 0; r1 < 3; ++r1) outs[r1] = out.m[min(base + r1, 5)];
      } else {
        const int base = r2 == 0 ? 0 : 2;
        for (int r1 = 0; r1 < 3; ++r1) outs[r1] = out.v[min(base + r1, 2)];
      }
      if (wr + 16 > j_lo && wr < n1) {
        double acc[3][2][4][2] = {};
        const int k0 = max(0, (wr - R1) & ~3), k1 = min(n1, wr + 16 + R1);
        for (int k = k0; k < k1; k += 4) {
          const int m = k + lk;
          double b[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = Y[m * kLd + wc + j * 8 + lr];
#pragma unroll
          for (int r1 = 0; r1 < 3; ++r1) {
            if (r1 < n_r1) {
              const double* ta = tz + (0 * 3 + r1) * kTz + kTc;
              double a[2];
#pragma unroll
              for (int i = 0; i < 2; ++i) a[i] = ta[m - (wr + i * 8 + lr)];
#pragma unroll
              for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[r1][i][j], a[i], b[j]);
            }
          }
        }
#pragma unroll
        for (int r1 = 0; r1 < 3; ++r1) {
          if (r1 < n_r1) {
            double* o = outs[r1] + off;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int row = wr + i * 8 + lr;
              if (row < j_lo || row >= n1) continue;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int col = wc + j * 8 + 2 * lk;
                if (col + 1 < n2 && (n2 % 2) == 0) {
                  *reinterpret_cast<double2*>(o + static_cast<i64>(row) * n2 + col) =
                      make_double2(acc[r1][i][j][0], acc[r1][i][j][1]);
                } else {
                  if (col < n2) o[static_cast<i64>(row) * n2 + col] = acc[r1][i][j][0];
                  if (col + 1 < n2) o[static_cast<i64>(row) * n2 + col + 1] = acc[r1][i][j][1];
                }
              }
            }
          }
        }
      }
      __syncthreads();
    }
    buf ^= 1;
    s = ns;
    pass = npass;
  }
  cp_wait<0>();
}


// ---- s-phase passes (k_pass_cols' work) on the DMMA pipe -----------------
// A pass along an axis of n <= 64 nodes over 64-column tiles of the array:
// out_r = A_r X with A_r[j][m] = taps_r[m - j + R] for the tile X [n][64],
// the same tiles, triangle trims and output windows as k_pass_cols (View::tri,
// View::lo/hi), up to three orders from one staged tile.
struct PassTaps {
  double t[3][kTz];  // [order][o + kTc]
};

__device__ inline void pass_meta(const View& in, int tile, int chunks, int R, int& ob, int& c0, int& rows, int& nout,
                                 int& lo) {
  const int n = static_cast<int>(in.n);
  const int inner = static_cast<int>(in.inner);
  ob = tile / chunks;
  c0 = (tile - ob * chunks) * kP;
  rows = n;
  nout = n;
  lo = static_cast<int>(in.lo);
  const int win_hi = static_cast<int>(in.hi);
  if (win_hi >= 0) {
    nout = win_hi < n ? win_hi : n;
    rows = nout + R < n ? nout + R : n;
  }
  if (in.tri != 0) {
    const int triG = static_cast<int>(in.tri_G), tri_rn = static_cast<int>(in.tri_rn);
    const int c1 = (c0 + kP < inner ? c0 + kP : inner) - 1;
    const int tmax = (c0 / triG == c1 / triG) ? c1 % triG : triG - 1;
    int s1_out = (tmax + static_cast<int>(in.tri_t0)) / tri_rn + 1;
    if (in.tri_row_hi >= 0 && s1_out > in.tri_row_hi) s1_out = static_cast<int>(in.tri_row_hi);
    s1_out -= static_cast<int>(in.tri_row0);
    if (s1_out < 0) s1_out = 0;
    const int triR = in.tri_R, tri_n1 = static_cast<int>(in.tri_n1);
    if (in.tri == 1) {
      const int s1_in = s1_out + triR < tri_n1 ? s1_out + triR : tri_n1;
      if (ob >= s1_in) rows = nout = 0;
    } else if (in.tri == 3) {
      if (ob >= s1_out) rows = nout = 0;
    } else {
      nout = s1_out < n ? s1_out : n;
      rows = nout + triR < n ? nout + triR : n;
    }
  }
}

__global__ void __launch_bounds__(kThreadsM, 2)
    k_pass_cols_mma(View in, View o0, View o1, View o2, int n_out, const PassTaps* __restrict__ taps_g, int R) {
  pdl_wait();
  extern __shared__ __align__(16) double sm[];
  double* Xb = sm;                  // [2][kRows][kLd]
  double* tz = sm + 2 * kRows * kLd;  // PassTaps
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 2 * kRows * kLd; e += blockDim.x) sm[e] = 0.0;
  for (int e = tid; e < 3 * kTz; e += blockDim.x) tz[e] = reinterpret_cast<const double*>(taps_g)[e];
  __syncthreads();
  const int inner = static_cast<int>(in.inner);
  const int chunks = (inner + kP - 1) / kP;
  const int n_tiles = static_cast<int>(in.outer) * chunks;
  const bool vec = (in.js % 2 == 0) && (in.os % 2 == 0) && (inner % 2 == 0) &&
                   ((reinterpret_cast<std::uintptr_t>(in.p) & 15) == 0);
  auto issue = [&](int tile, int b) {
    int ob, c0, rows, nout, lo;
    pass_meta(in, tile, chunks, R, ob, c0, rows, nout, lo);
    const double* src = in.p + static_cast<i64>(ob) * in.os + c0;
    double* X = Xb + b * kRows * kLd;
    const int cols = inner - c0 < kP ? inner - c0 : kP;
    if (vec && cols == kP) {
      for (int e = tid; e < rows * (kP / 2); e += blockDim.x) {
        const int j = e / (kP / 2), c = (e % (kP / 2)) * 2;
        cp16(X + j * kLd + c, src + static_cast<i64>(j) * in.js + c);
      }
    } else {
      for (int e = tid; e < rows * kP; e += blockDim.x) {
        const int j = e / kP, c = e % kP;
        if (c < cols) cp8(X + j * kLd + c, src + static_cast<i64>(j) * in.js + c);
        else X[j * kLd + c] = 0.0;
      }
    }
  };
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32;
  const int lr = lane >> 2, lk = lane & 3;
  int tile = blockIdx.x, buf = 0;
  if (tile < n_tiles) issue(tile, 0);
  cp_commit();
  while (tile < n_tiles) {
    const int next = tile + gridDim.x;
    if (next < n_tiles) issue(next, buf ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    int ob, c0, rows, nout, lo;
    pass_meta(in, tile, chunks, R, ob, c0, rows, nout, lo);
    const double* X = Xb + buf * kRows * kLd;
    if (wr + 16 > lo && wr < nout) {
      double acc[3][2][4][2] = {};
      const int k0 = max(0, (wr - R) & ~3), k1 = min(rows, wr + 16 + R);
      for (int k = k0; k < k1; k += 4) {
        const int m = k + lk;
        double b[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = X[m * kLd + wc + j * 8 + lr];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          if (r < n_out) {
            const double* ta = tz + r * kTz + kTc;
            double a[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) a[i] = ta[m - (wr + i * 8 + lr)];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) dmma(acc[r][i][j], a[i], b[j]);
          }
        }
      }
      const int cols = inner - c0 < kP ? inner - c0 : kP;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        if (r >= n_out) continue;
        const View& o = r == 0 ? o0 : (r == 1 ? o1 : o2);
        double* base = o.p + static_cast<i64>(ob) * o.os + c0;
        const bool ovec = (o.js % 2 == 0) && (o.os % 2 == 0) && ((reinterpret_cast<std::uintptr_t>(o.p) & 15) == 0) &&
                          (c0 % 2 == 0);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int row = wr + i * 8 + lr;
          if (row < lo || row >= nout) continue;
          double* rp = base + static_cast<i64>(row) * o.js;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int col = wc + j * 8 + 2 * lk;
            if (ovec && col + 1 < cols) {
              *reinterpret_cast<double2*>(rp + col) = make_double2(acc[r][i][j][0], acc[r][i][j][1]);
            } else {
              if (col < cols) rp[col] = acc[r][i][j][0];
              if (col + 1 < cols) rp[col + 1] = acc[r][i][j][1];
            }
          }
        }
      }
    }
    __syncthreads();
    buf ^= 1;
    tile = next;
  }
  cp_wait<0>();
}

}  // namespace

bool run_pass_mma(dfpca_context* ctx, const PassSpec& s) {
  if (s.in.n > kP || s.in.n < 1 || s.in.inner < kP / 2 || s.R > kP || s.n_out < 1 || s.n_out > 3) return false;
  const i64 tiles = s.in.outer * ((s.in.inner + kP - 1) / kP);
  if (tiles >= (i64(1) << 31)) return false;
  PassTaps h{};
  for (int r = 0; r < s.n_out; ++r)
    for (int o = -s.R; o <= s.R; ++o) h.t[r][o + kTc] = s.taps[r][o + s.R];
  DevBuf<PassTaps> dt(1);
  DFPCA_CUDA(cudaMemcpyAsync(dt.get(), &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
  const View o1 = s.n_out > 1 ? s.out[1] : s.out[0];
  const View o2 = s.n_out > 2 ? s.out[2] : s.out[0];
  const std::size_t smem = sizeof(double) * (2 * kRows * kLd) + sizeof(PassTaps);
  allow_smem(k_pass_cols_mma, smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pass_cols_mma, kThreadsM, smem);
  const unsigned grid =
      static_cast<unsigned>(std::max<i64>(1, std::min<i64>(tiles, static_cast<i64>(std::max(per_sm, 1)) * ctx->sm_count)));
  DFPCA_LAUNCH(ctx, k_pass_cols_mma, grid, kThreadsM, smem, s.in, s.out[0], o1, o2, s.n_out, dt.get(), s.R);
  return true;
}

bool run_tphase2_mma(dfpca_context* ctx, const TPhase2Spec& s) {
  if (s.n1 > kP || s.n2 > kP || s.n1 < 1 || s.n2 < 1 || s.R[0] > kP || s.R[1] > kP) return false;
  MmaTaps h{};
  for (int ax = 0; ax < 2; ++ax)
    for (int r = 0; r < 3; ++r)
      for (int o = -s.R[ax]; o <= s.R[ax]; ++o) h.t[ax][r][o + kTc] = s.taps[ax][r][o + s.R[ax]];
  DevBuf<MmaTaps> dt(1);
  DFPCA_CUDA(cudaMemcpyAsync(dt.get(), &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
  conv_detail::TPhaseOut out;
  for (int i = 0; i < 6; ++i) out.m[i] = s.mass_out[i];
  for (int i = 0; i < 3; ++i) out.v[i] = s.value_out[i];
  out.s_base = s.s_base;
  out.rn = s.rn;
  out.t1_margin = s.t1_margin;
  const std::size_t smem = sizeof(double) * (3 * kRows * kLd) + sizeof(MmaTaps);
  allow_smem(k_tphase2_mma, smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tphase2_mma, kThreadsM, smem);
  const unsigned grid =
      static_cast<unsigned>(std::max<i64>(1, std::min<i64>(s.rows, static_cast<i64>(std::max(per_sm, 1)) * ctx->sm_count)));
  DFPCA_LAUNCH(ctx, k_tphase2_mma, grid, kThreadsM, smem, s.pw, s.pv, s.rows, static_cast<int>(s.n1),
               static_cast<int>(s.n2), s.value_only ? 1 : 0, out, dt.get(), s.R[0], s.R[1]);
  return true;
}

}  // namespace dfpca_gpu
