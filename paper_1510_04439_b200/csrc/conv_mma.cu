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

}  // namespace

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
