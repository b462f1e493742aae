// FP64 SYRK of the pair grids (K2) on the int8 tensor cores: the Ozaki
// scheme with tcgen05.mma kind::i8.
//
// pv[s][t] = sum_i w_i Y_i(s) Y_i(t) (and pw alike) is the symmetric product
// X^T Y of X = w * Y and Y, both K x G (K = subjects, G = grid nodes).  FP64
// has no tcgen05 kind and DMMA runs at the DFMA rate (37 TFLOP/s, gemm.cu);
// the int8 kind runs ~120x faster per MAC, so the product is computed from
// exact integer products of 7-bit slices:
//
//   per node column m, e_m with max_k |X[k][m]| 2^-e_m <= 127/128, and
//   X[k][m] = 2^e_m (sum_{a=1..S} 2^-7a x_a[m][k] + r),  |r| <= 2^-7S / 2,
//   x_1 in [-127, 127], x_a in [-64, 64] (signed digits of the 56-bit
//   integer rint(X 2^(56-e)), oz_pack16); the same for Y with e'_m, y_b.
//
//   X^T Y [s][t] ~ 2^(e_s + e'_t) sum_{d=2..S+1} 2^-7d P_d[s][t],
//   P_d = sum_{a+b=d} x_a y_b^T  (int8 x int8 -> int32, exact: at most S terms
//   of K * 127^2 each, so K <= 16384 keeps every sum below 2^31).
//
// The dropped pairs (a + b > S + 1) and the slice remainders are each below
// ~K 2^-7S of max |X| max |Y| per column pair; with S = 8 that is ~3e-14
// relative at K = 2000 -- the order of an FP64 dot product's own rounding
// bound (K u sum |x y| ~ 2e-13), far inside the 1e-10 surface tolerance.
// Zero products stay exactly zero (all digits zero).
//
// Kernels: k_oz_colmax (the column scales), k_oz_slice (the slices, in the
// product's staging layout) and k_oz_syrk, one CTA per SM, persistent over
// the upper 128 x 128 tiles: a producer warp streams each (tile, pass,
// 32-byte K chunk) block of slices into a 3-stage ring with bulk copies, one
// warp issues the slice-pair MMAs (M 128, N 128, K 32) into the pass's 4
// int32 TMEM accumulators (d = a + b in [4p, 4p + 4); two passes fill the 512
// columns twice), and 16 epilogue warps add each pass into FP64 registers
// (ascending d), then scale and write every upper-triangle entry of the tile
// and its mirror (entries s > t are written only by the tile owning (t, s):
// exactly symmetric, deterministic).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "gemm.cuh"

namespace dfpca_gpu {
namespace {

constexpr int kOzS = 8;           // 7-bit slices
constexpr int kOzM = 128;         // tile rows (s), UMMA M
constexpr int kOzN = 128;         // tile columns (t), UMMA N
constexpr int kOzKc = 32;         // K bytes per stage = one MMA's K
constexpr int kOzAcc = 4;         // accumulators per pass (4 x 128 TMEM columns)
constexpr int kOzStages = 3;
constexpr int kOzMaxK = 16384;
constexpr int kOzBlk = kOzS * 128 * kOzKc;     // 32 KB: one (128-row block, K chunk) of an operand's slices
constexpr int kOzHalfBlk = kOzBlk / 2;         // its slices 0..3 (pass 0)
constexpr int kOzStage = 2 * kOzBlk;           // 64 KB: both operands
constexpr int kOzSmem = kOzStages * kOzStage + 1024;
// warps: 0 producer (bulk copies), 1 MMA issuer, 2..17 epilogue (TMEM lane
// quadrant w % 4, columns 32 ((w - 2) / 4) ..)
constexpr int kOzEpiWarps = 16;
constexpr int kOzThreads = 32 * (2 + kOzEpiWarps);

__device__ inline unsigned oz_smem(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ inline void oz_mbar_wait(std::uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "OZ_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra OZ_DONE;\n\t"
      "bra OZ_WAIT;\n"
      "OZ_DONE:\n\t}\n" ::"r"(oz_smem(bar)),
      "r"(parity)
      : "memory");
}

__device__ inline void oz_mbar_init_n(std::uint64_t* bar, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(oz_smem(bar)), "r"(n));
}
__device__ inline void oz_mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(oz_smem(bar)) : "memory");
}
__device__ inline void oz_mbar_expect(std::uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(oz_smem(bar)), "r"(bytes) : "memory");
}
__device__ inline void oz_bulk(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(oz_smem(dst)),
      "l"(src), "r"(bytes), "r"(oz_smem(bar))
      : "memory");
}

__device__ inline bool oz_elect() {
  unsigned p;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}\n"
      : "=r"(p));
  return p != 0u;
}

// Shared-memory matrix descriptor (SM100 UMMA): K-major, 32-byte swizzle:
// rows of 32 K bytes, 8-row atoms of 256 bytes (`sbo` = 256 between atoms;
// `lbo` unused, 16).
__device__ inline std::uint64_t oz_desc(unsigned addr, unsigned lbo, unsigned sbo) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((addr >> 4) & 0x3fffu);
  d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3fffu) << 16;
  d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3fffu) << 32;
  d |= static_cast<std::uint64_t>(1) << 46;  // descriptor version (SM100)
  d |= static_cast<std::uint64_t>(6) << 61;  // SWIZZLE_32B
  return d;                                  // base offset 0 (1024-byte aligned atoms)
}

// Instruction descriptor of kind::i8: D s32, A and B signed int8, both
// K-major, M = 128, N = 64.
constexpr std::uint32_t kOzIdesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<std::uint32_t>(kOzN >> 3) << 17) |
                                   (static_cast<std::uint32_t>(kOzM >> 4) << 24);

__device__ inline void oz_mma(unsigned tmem_d, std::uint64_t da, std::uint64_t db, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kOzIdesc), "r"(accumulate ? 1 : 0));
}
__device__ inline void oz_commit_mbar(std::uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(oz_smem(bar))
               : "memory");
}

// 32 consecutive int32 columns of this thread's TMEM lane.
__device__ inline void oz_tmem_ld32(unsigned taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

// ---- slicing ---------------------------------------------------------------

// Column scale exponents of both operands in one pass over A: ex[m] / ey[m]
// hold the bits of max_k |w_k A[k][m]| / max_k |A[k][m]|, combined across CTAs
// with an integer atomicMax (non-negative doubles order like their bits).
__global__ void k_oz_colmax(const double* __restrict__ A, i64 K, i64 M, i64 lda, const double* __restrict__ w,
                            unsigned long long* __restrict__ ex, unsigned long long* __restrict__ ey) {
  pdl_wait();
  const i64 m = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (m >= M) return;
  // a NaN / Inf entry poisons its column: the bits of NaN order above every
  // finite value, and oz_exponent turns them into a NaN column scale, so every
  // product with that row or column comes out NaN (as the FP64 sum would)
  double mx = 0.0, my = 0.0;
  for (i64 k = blockIdx.y; k < K; k += gridDim.y) {
    const double a = A[k * lda + m];
    const double aw = __dmul_rn(w[k], a);
    mx = isfinite(aw) ? fmax(mx, fabs(aw)) : __longlong_as_double(0x7ff8000000000000ll);
    my = isfinite(a) ? fmax(my, fabs(a)) : __longlong_as_double(0x7ff8000000000000ll);
    if (!isfinite(aw) || !isfinite(a)) break;
  }
  const auto bits = [](double v) {
    return isnan(v) ? 0x7ff8000000000000ull : static_cast<unsigned long long>(__double_as_longlong(v));
  };
  if (!(mx == 0.0)) atomicMax(ex + m, bits(mx));
  if (!(my == 0.0)) atomicMax(ey + m, bits(my));
}

// exp2 scale of column m: the smallest e with max |X| 2^-e <= 127/128 (0 for
// an all-zero or a poisoned column).
__device__ inline bool oz_poisoned(unsigned long long maxbits) { return maxbits >= 0x7ff0000000000000ull; }
__device__ inline int oz_exponent(unsigned long long maxbits) {
  const double mx = __longlong_as_double(static_cast<long long>(maxbits));
  if (!(mx > 0.0) || oz_poisoned(maxbits)) return 0;
  int e;
  const double f = frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1)
  return f > 127.0 / 128.0 ? e + 1 : e;
}

// Slices of X = w * A (or A) in the product kernel's staging layout: for row
// block rb (R rows: 128 for the s operand, 64 for the t operand) and 32-byte
// K chunk c, one contiguous block [a][r][32 bytes] (slice a, row r) in the
// 32-byte-swizzled K-major layout the MMA descriptors read (the two 16-byte
// halves of row r swapped when r / 4 is odd), so one bulk copy stages it.  CTA = 32 nodes x 64
// subjects; digits through shared memory, global writes in 16-byte segments.
// The 16 digits of slice 0..7 of 16 consecutive K entries of one operand row,
// packed per slice into 16 bytes: x = 2^e iv 2^-56 with iv = rint(x 2^(56-e))
// (|iv| < 2^56 127/128; the dropped part is below 2^(e-57), the truncation of
// 8 seven-bit digits), then signed digits by round-half-up shifts on the
// integer, d_a = round(iv / 2^(56-7a)), iv -= d_a 2^(56-7a): d_1 in
// [-127, 127], the rest in [-64, 64], exactly x = 2^e sum_a d_a 2^-7a + r.
__device__ inline void oz_pack16(const double (&x)[16], int e, uint4 (&out)[kOzS]) {
  unsigned w[kOzS][4];
#pragma unroll
  for (int a = 0; a < kOzS; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) w[a][q] = 0u;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double xs_ = ldexp(x[j], 56 - e);
    long long iv = isfinite(xs_) ? __double2ll_rn(xs_) : 0ll;  // poisoned rows: scale NaN, digits unused
#pragma unroll
    for (int a = 0; a < kOzS; ++a) {
      const int sh = 56 - 7 * (a + 1);
      long long d;
      if (sh > 0) {
        d = (iv + (1ll << (sh - 1))) >> sh;
        iv -= d << sh;
      } else {
        d = iv;
      }
      w[a][j >> 2] |= (static_cast<unsigned>(d) & 0xffu) << (8 * (j & 3));
    }
  }
#pragma unroll
  for (int a = 0; a < kOzS; ++a) out[a] = make_uint4(w[a][0], w[a][1], w[a][2], w[a][3]);
}

// Slices of both operands (X = w * A on rows [row0, row1) from local row 0,
// Y = A on every row; 128-row blocks, the staging layout above) and the
// column scales 2^e: thread = (row, 16-entry K segment), consecutive threads
// on consecutive rows (coalesced reads of A), digits packed in registers and
// written as 16-byte segments (no shared memory).
__global__ void __launch_bounds__(128) k_oz_slice(const double* __restrict__ A, i64 K, i64 M, i64 lda,
                                                  const double* __restrict__ w,
                                                  const unsigned long long* __restrict__ ex,
                                                  const unsigned long long* __restrict__ ey,
                                                  std::int8_t* __restrict__ xs, std::int8_t* __restrict__ ys,
                                                  double* __restrict__ sx, double* __restrict__ sy, i64 rows_x,
                                                  i64 rows_y, i64 nch, i64 row0, i64 row1, int ry) {
  pdl_wait();
  const i64 m = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  const i64 k0 = static_cast<i64>(blockIdx.y) * 16;
  const i64 c = k0 >> 5, g = (k0 >> 4) & 1;
  for (int op = 0; op < 2; ++op) {
    const i64 rows = op == 0 ? rows_x : rows_y;
    if (m >= rows) continue;
    const i64 gm = op == 0 ? row0 + m : m;  // global row
    const bool valid = op == 0 ? gm < row1 : gm < M;
    const unsigned long long mb = valid ? (op == 0 ? ex : ey)[gm] : 0ull;
    const int e = oz_exponent(mb);
    if (valid && blockIdx.y == 0)
      (op == 0 ? sx : sy)[gm] = oz_poisoned(mb) ? __longlong_as_double(0x7ff8000000000000ll) : ldexp(1.0, e);
    double x[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const i64 k = k0 + j;
      double v = 0.0;
      if (valid && k < K) {
        v = A[k * lda + gm];
        if (op == 0) v = __dmul_rn(w[k], v);
      }
      x[j] = v;
    }
    uint4 d[kOzS];
    oz_pack16(x, e, d);
    std::int8_t* base = op == 0 ? xs : ys;
    const int R = op == 0 ? 128 : ry;  // rows per block of this operand
    const i64 rb = m / R, r = m % R;
    // row r holds its 32 K bytes contiguously; 32-byte swizzle: the 16-byte
    // half g is stored at g ^ (r / 4 % 2)
    std::int8_t* dst = base + (rb * nch + c) * (kOzS * R * kOzKc) + r * 32 + ((g ^ ((r >> 2) & 1)) << 4);
#pragma unroll
    for (int a = 0; a < kOzS; ++a) *reinterpret_cast<uint4*>(dst + a * (R * 32)) = d[a];
  }
}

// ---- the product -----------------------------------------------------------

// The slice pairs of pass p: accumulator d = xa + yb in [4p, 4p + 4).
__host__ __device__ constexpr bool oz_in_pass(int p, int xa, int yb) {
  return xa + yb >= kOzAcc * p && xa + yb < kOzAcc * (p + 1);
}

// tiles[i] = (I, J): s rows [row0 + 128 I, +128), t columns [128 J, +128).
// Warp-specialized: warp 0 (one lane) streams the (tile, pass, chunk) blocks
// into a 3-stage ring with bulk copies (pass 0 needs slices 0..3 only);
// warp 1 issues each chunk's slice-pair MMAs (M 128, N 128, K 32) into the
// pass's 4 accumulators and commits them to the stage's "empty" barrier, and
// each pass's last chunk to "tmem full"; the 16 epilogue warps add each
// pass's accumulators into their registers (2^-7(d+2) scales, ascending d),
// release TMEM ("tmem empty"), and after pass 1 scale and store.
__global__ void __launch_bounds__(kOzThreads, 1)
    k_oz_syrk(const std::int8_t* __restrict__ xs, const std::int8_t* __restrict__ ys, i64 nch,
              const double* __restrict__ sx, const double* __restrict__ sy, i64 M, double* __restrict__ C, i64 ldc,
              const int2* __restrict__ tiles, int n_tiles, i64 row0, i64 row1) {
  pdl_wait();
  extern __shared__ __align__(16) std::uint8_t oz_sm[];
  __shared__ __align__(8) std::uint64_t full[kOzStages], empty[kOzStages], tmem_full, tmem_empty;
  __shared__ unsigned tmem_base_sh;
  std::uint8_t* sm = reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(oz_sm) + 1023) &
                                                     ~static_cast<std::uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(oz_smem(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 32) {
    for (int i = 0; i < kOzStages; ++i) {
      oz_mbar_init_n(&full[i], 1);
      oz_mbar_init_n(&empty[i], 1);
    }
    oz_mbar_init_n(&tmem_full, 1);
    oz_mbar_init_n(&tmem_empty, kOzEpiWarps);  // one arrival per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const unsigned tmem = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {  // producer
      int st = 0;
      unsigned ph = 0;
      for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
        const int2 tl = tiles[ti];
        const std::int8_t* xa = xs + static_cast<i64>(tl.x) * nch * kOzBlk;
        const std::int8_t* yb = ys + static_cast<i64>(tl.y) * nch * kOzBlk;
        for (int p = 0; p < 2; ++p) {
          const unsigned bytes = p == 0 ? kOzHalfBlk : kOzBlk;
          for (i64 c = 0; c < nch; ++c) {
            oz_mbar_wait(&empty[st], ph ^ 1u);  // first pass over the ring: passes at once
            std::uint8_t* dst = sm + st * kOzStage;
            oz_mbar_expect(&full[st], 2 * bytes);
            oz_bulk(dst, xa + c * kOzBlk, bytes, &full[st]);
            oz_bulk(dst + kOzBlk, yb + c * kOzBlk, bytes, &full[st]);
            if (++st == kOzStages) {
              st = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp runs the loop (descriptors and TMEM
    // addresses stay warp-uniform) and one elected lane issues
    const unsigned tm = __shfl_sync(0xffffffffu, tmem, 0);
    const unsigned smem0 = __shfl_sync(0xffffffffu, oz_smem(sm), 0);
    int st = 0;
    unsigned ph = 0, tph = 0;
    for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
      for (int p = 0; p < 2; ++p) {
        oz_mbar_wait(&tmem_empty, tph ^ 1u);  // the epilogue has read the accumulators out
        tph ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        for (i64 c = 0; c < nch; ++c) {
          oz_mbar_wait(&full[st], ph);
          asm volatile("tcgen05.fence::after_thread_sync;\n");
          const unsigned a_base = smem0 + st * kOzStage, b_base = a_base + kOzBlk;
          const std::uint64_t da0 = oz_desc(a_base, 16, 256), db0 = oz_desc(b_base, 16, 256);
          if (oz_elect()) {
            // chunk 0: the first pair issued into each accumulator overwrites it
            unsigned started = c == 0 ? 0u : 0xffu;
            if (p == 0) {
#pragma unroll
              for (int xa = 0; xa < kOzS; ++xa)
#pragma unroll
                for (int yb = 0; yb < kOzS; ++yb) {
                  if (!oz_in_pass(0, xa, yb)) continue;
                  const int d = xa + yb;
                  oz_mma(tm + d * kOzN, da0 + ((xa * 128 * 32) >> 4), db0 + ((yb * 128 * 32) >> 4),
                         (started >> d) & 1u);
                  started |= 1u << d;
                }
            } else {
#pragma unroll
              for (int xa = 0; xa < kOzS; ++xa)
#pragma unroll
                for (int yb = 0; yb < kOzS; ++yb) {
                  if (!oz_in_pass(1, xa, yb)) continue;
                  const int d = xa + yb - kOzAcc;
                  oz_mma(tm + d * kOzN, da0 + ((xa * 128 * 32) >> 4), db0 + ((yb * 128 * 32) >> 4),
                         (started >> d) & 1u);
                  started |= 1u << d;
                }
            }
            oz_commit_mbar(&empty[st]);
            if (c == nch - 1) oz_commit_mbar(&tmem_full);
          }
          __syncwarp();
          if (++st == kOzStages) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else {  // epilogue warps: TMEM lane quadrant q, 32 columns from 32 cg
    const int q = warp & 3, cg = (warp - 2) >> 2;
    unsigned tph = 0;
    for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
      const int2 tl = tiles[ti];
      const i64 s0 = row0 + static_cast<i64>(tl.x) * kOzM, t0 = static_cast<i64>(tl.y) * kOzN + cg * 32;
      const i64 s = s0 + q * 32 + lane;
      double acc[32];
#pragma unroll
      for (int n = 0; n < 32; ++n) acc[n] = 0.0;
      for (int p = 0; p < 2; ++p) {
        oz_mbar_wait(&tmem_full, tph);
        tph ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll 1
        for (int d = 0; d < kOzAcc; ++d) {
          int v[32];
          oz_tmem_ld32(tmem + (static_cast<unsigned>(q * 32) << 16) + d * kOzN + cg * 32, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          const double pw = ldexp(1.0, -7 * (kOzAcc * p + d + 2));
#pragma unroll
          for (int n = 0; n < 32; ++n) acc[n] = fma(static_cast<double>(v[n]), pw, acc[n]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncwarp();
        if (lane == 0) oz_mbar_arrive(&tmem_empty);
      }
      // row s of the slab: every t >= s; the mirror (t, s) when row t is in
      // the slab too (C's row 0 is global row row0)
      if (s < row1) {
        const double fs = sx[s];
#pragma unroll 8
        for (int n = 0; n < 32; ++n) {
          const i64 t = t0 + n;
          if (t < M && s <= t) {
            const double val = acc[n] * fs * sy[t];
            C[(s - row0) * ldc + t] = val;
            if (t < row1) C[(t - row0) * ldc + s] = val;
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ---- the product on CTA pairs ---------------------------------------------
// tcgen05.mma.cta_group::2: one MMA covers M 256 (128 s rows per CTA of the
// pair, each in its own TMEM) x N 128 (each CTA stages its half of the 128 t
// rows: 64), so every SM reads 6 KB of operands per 128 x 128 x 32 MMA
// instead of 8 KB -- the shared-memory operand reads are what bound the
// one-CTA kernel.  Tiles of 256 s rows x 128 t columns; the leader CTA
// (rank 0) issues for the pair.  Barriers: each CTA's producer fills its own
// stage (its own "full"); the peer's warp 1 forwards its "full" to the
// leader ("peer full"); the leader's commits arrive on both CTAs' "empty" and
// "tmem full" (multicast); the 32 epilogue warps of the pair arrive on the
// leader's "tmem empty".
constexpr int kOz2BlkA = kOzS * 128 * kOzKc;       // 32 KB: 128 s rows
constexpr int kOz2BlkB = kOzS * 64 * kOzKc;        // 16 KB: 64 t rows (half of N)
constexpr int kOz2Stage = kOz2BlkA + kOz2BlkB;     // 48 KB
constexpr int kOz2Stages = 4;
constexpr int kOz2Smem = kOz2Stages * kOz2Stage + 1024;
constexpr std::uint32_t kOz2Idesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<std::uint32_t>(128 >> 3) << 17) |
                                    (static_cast<std::uint32_t>(256 >> 4) << 24);

__device__ inline unsigned oz_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ inline void oz_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ inline unsigned oz_mapa(unsigned addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ inline void oz_arrive_remote(unsigned cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
__device__ inline void oz_wait_cluster(std::uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "OZ2_WAIT:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra OZ2_DONE;\n\t"
      "bra OZ2_WAIT;\n"
      "OZ2_DONE:\n\t}\n" ::"r"(oz_smem(bar)),
      "r"(parity)
      : "memory");
}
__device__ inline void oz2_mma(unsigned tmem_d, std::uint64_t da, std::uint64_t db, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kOz2Idesc), "r"(accumulate ? 1 : 0));
}
__device__ inline void oz2_commit_both(std::uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          oz_smem(bar)),
      "h"(static_cast<unsigned short>(3))
      : "memory");
}

// tiles[i] = (I2, J): s rows [row0 + 256 I2, +256) (CTA rank r: +128 r),
// t columns [128 J, +128) (CTA rank r stages rows 128 J + 64 r ..).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kOzThreads, 1)
    k_oz_syrk2(const std::int8_t* __restrict__ xs, const std::int8_t* __restrict__ ys, i64 nch,
               const double* __restrict__ sx, const double* __restrict__ sy, i64 M, double* __restrict__ C, i64 ldc,
               const int2* __restrict__ tiles, int n_tiles, i64 row0, i64 row1) {
  pdl_wait();
  extern __shared__ __align__(16) std::uint8_t oz_sm[];
  __shared__ __align__(8) std::uint64_t full[kOz2Stages], peer_full[kOz2Stages], empty[kOz2Stages], tmem_full,
      tmem_empty;
  __shared__ unsigned tmem_base_sh;
  std::uint8_t* sm = reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(oz_sm) + 1023) &
                                                     ~static_cast<std::uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned rank = oz_rank();
  const int pair = static_cast<int>(blockIdx.x >> 1), n_pairs = static_cast<int>(gridDim.x >> 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(oz_smem(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  if (tid == 32) {
    for (int i = 0; i < kOz2Stages; ++i) {
      oz_mbar_init_n(&full[i], 1);
      oz_mbar_init_n(&peer_full[i], 1);
      oz_mbar_init_n(&empty[i], 1);
    }
    oz_mbar_init_n(&tmem_full, 1);
    oz_mbar_init_n(&tmem_empty, 2 * kOzEpiWarps);  // both CTAs' epilogue warps (leader's barrier)
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  oz_cluster_sync();  // barriers of both CTAs initialised before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const unsigned tmem = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {  // producer: this CTA's A rows and B half
      int st = 0;
      unsigned ph = 0;
      for (int ti = pair; ti < n_tiles; ti += n_pairs) {
        const int2 tl = tiles[ti];
        const std::int8_t* xa = xs + (static_cast<i64>(2 * tl.x + rank) * nch) * kOz2BlkA;
        const std::int8_t* yb = ys + (static_cast<i64>(2 * tl.y + rank) * nch) * kOz2BlkB;
        for (int p = 0; p < 2; ++p) {
          const unsigned ba = p == 0 ? kOz2BlkA / 2 : kOz2BlkA, bb = p == 0 ? kOz2BlkB / 2 : kOz2BlkB;
          for (i64 c = 0; c < nch; ++c) {
            oz_wait_cluster(&empty[st], ph ^ 1u);
            std::uint8_t* dst = sm + st * kOz2Stage;
            oz_mbar_expect(&full[st], ba + bb);
            oz_bulk(dst, xa + c * kOz2BlkA, ba, &full[st]);
            oz_bulk(dst + kOz2BlkA, yb + c * kOz2BlkB, bb, &full[st]);
            if (++st == kOz2Stages) {
              st = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 1) {  // peer: forward each stage's arrival to the leader
      if (lane == 0) {
        int st = 0;
        unsigned ph = 0;
        for (int ti = pair; ti < n_tiles; ti += n_pairs)
          for (int p = 0; p < 2; ++p)
            for (i64 c = 0; c < nch; ++c) {
              oz_mbar_wait(&full[st], ph);
              oz_arrive_remote(oz_mapa(oz_smem(&peer_full[st]), 0));
              if (++st == kOz2Stages) {
                st = 0;
                ph ^= 1u;
              }
            }
      }
    } else {  // leader: MMA issuer (whole warp; one elected lane issues)
      const unsigned tm = __shfl_sync(0xffffffffu, tmem, 0);
      const unsigned smem0 = __shfl_sync(0xffffffffu, oz_smem(sm), 0);
      int st = 0;
      unsigned ph = 0, tph = 0;
      for (int ti = pair; ti < n_tiles; ti += n_pairs) {
        for (int p = 0; p < 2; ++p) {
          oz_wait_cluster(&tmem_empty, tph ^ 1u);
          tph ^= 1u;
          asm volatile("tcgen05.fence::after_thread_sync;\n");
          for (i64 c = 0; c < nch; ++c) {
            oz_mbar_wait(&full[st], ph);
            oz_wait_cluster(&peer_full[st], ph);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const unsigned a_base = smem0 + st * kOz2Stage, b_base = a_base + kOz2BlkA;
            const std::uint64_t da0 = oz_desc(a_base, 16, 256), db0 = oz_desc(b_base, 16, 256);
            if (oz_elect()) {
              unsigned started = c == 0 ? 0u : 0xffu;
              if (p == 0) {
#pragma unroll
                for (int xa = 0; xa < kOzS; ++xa)
#pragma unroll
                  for (int yb = 0; yb < kOzS; ++yb) {
                    if (!oz_in_pass(0, xa, yb)) continue;
                    const int d = xa + yb;
                    oz2_mma(tm + d * 128, da0 + ((xa * 128 * 32) >> 4), db0 + ((yb * 64 * 32) >> 4),
                            (started >> d) & 1u);
                    started |= 1u << d;
                  }
              } else {
#pragma unroll
                for (int xa = 0; xa < kOzS; ++xa)
#pragma unroll
                  for (int yb = 0; yb < kOzS; ++yb) {
                    if (!oz_in_pass(1, xa, yb)) continue;
                    const int d = xa + yb - kOzAcc;
                    oz2_mma(tm + d * 128, da0 + ((xa * 128 * 32) >> 4), db0 + ((yb * 64 * 32) >> 4),
                            (started >> d) & 1u);
                    started |= 1u << d;
                  }
              }
              oz2_commit_both(&empty[st]);
              if (c == nch - 1) oz2_commit_both(&tmem_full);
            }
            __syncwarp();
            if (++st == kOz2Stages) {
              st = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else {  // epilogue warps (both CTAs): TMEM lane quadrant q, 32 columns from 32 cg
    const int q = warp & 3, cg = (warp - 2) >> 2;
    const unsigned leader_empty = oz_mapa(oz_smem(&tmem_empty), 0);
    unsigned tph = 0;
    for (int ti = pair; ti < n_tiles; ti += n_pairs) {
      const int2 tl = tiles[ti];
      const i64 s0 = row0 + static_cast<i64>(tl.x) * 256 + rank * 128, t0 = static_cast<i64>(tl.y) * 128 + cg * 32;
      const i64 s = s0 + q * 32 + lane;
      double acc[32];
#pragma unroll
      for (int n = 0; n < 32; ++n) acc[n] = 0.0;
      for (int p = 0; p < 2; ++p) {
        oz_wait_cluster(&tmem_full, tph);
        tph ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll 1
        for (int d = 0; d < kOzAcc; ++d) {
          int v[32];
          oz_tmem_ld32(tmem + (static_cast<unsigned>(q * 32) << 16) + d * 128 + cg * 32, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          const double pw = ldexp(1.0, -7 * (kOzAcc * p + d + 2));
#pragma unroll
          for (int n = 0; n < 32; ++n) acc[n] = fma(static_cast<double>(v[n]), pw, acc[n]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncwarp();
        if (lane == 0) oz_arrive_remote(leader_empty);
      }
      if (s < row1) {
        const double fs = sx[s];
#pragma unroll 8
        for (int n = 0; n < 32; ++n) {
          const i64 t = t0 + n;
          if (t < M && s <= t) {
            const double val = acc[n] * fs * sy[t];
            C[(s - row0) * ldc + t] = val;
            if (t < row1) C[(t - row0) * ldc + s] = val;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  oz_cluster_sync();  // the pair is done with both TMEMs
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

}  // namespace

bool ozaki_enabled() {
  const char* e = std::getenv("DFPCA_SYRK");
  return !(e && std::string(e) == "dmma");
}

bool ozaki_syrk(dfpca_context* ctx, i64 G, i64 K, const double* A, i64 lda, const double* w, double* C, i64 ldc,
                i64 row0, i64 row1) {
  if (K <= 0 || K > kOzMaxK || G <= 0 || !w) return false;
  row1 = std::min(row1, G);
  if (row0 >= row1) return true;
  const i64 Kp = (K + 63) / 64 * 64;
  const i64 nch = Kp / kOzKc;
  const char* pe = std::getenv("DFPCA_OZ_PAIRS");
  const bool pairs = pe && std::string(pe) == "1";  // CTA-pair kernel (k_oz_syrk2), opt-in
  // row blocks: X in 128 rows (an even count for the pairs), Y in 128 (64 for the pairs)
  const i64 RA0 = (row1 - row0 + kOzM - 1) / kOzM;
  const i64 RA = pairs ? (RA0 + 1) / 2 * 2 : RA0;
  const int ry = pairs ? 64 : 128;
  const i64 RB = (G + 127) / 128 * (128 / ry);
  DevBuf<std::int8_t> xs(static_cast<std::size_t>(RA * nch * kOzBlk)),
      ys(static_cast<std::size_t>(RB * nch * kOzS * ry * kOzKc));
  DevBuf<unsigned long long> ex(static_cast<std::size_t>(G)), ey(static_cast<std::size_t>(G));
  DevBuf<double> sx(static_cast<std::size_t>(G)), sy(static_cast<std::size_t>(G));
  cudaStream_t st = ctx->stream;
  DFPCA_CUDA(cudaMemsetAsync(ex.get(), 0, sizeof(unsigned long long) * G, st));
  DFPCA_CUDA(cudaMemsetAsync(ey.get(), 0, sizeof(unsigned long long) * G, st));
  const dim3 gmax(static_cast<unsigned>((G + 255) / 256), static_cast<unsigned>(std::min<i64>(K, 64)));
  DFPCA_LAUNCH_PDL(ctx, k_oz_colmax, gmax, 256, 0, A, K, G, lda, w, ex.get(), ey.get());
  // every row of the padded row blocks is written (zeros past the rows and past K)
  const i64 rows_x = RA * kOzM, rows_y = RB * ry;
  const dim3 gs(static_cast<unsigned>((std::max(rows_x, rows_y) + 127) / 128), static_cast<unsigned>(Kp / 16));
  DFPCA_LAUNCH_PDL(ctx, k_oz_slice, gs, 128, 0, A, K, G, lda, w, ex.get(), ey.get(), xs.get(), ys.get(), sx.get(),
               sy.get(), rows_x, rows_y, nch, row0, row1, ry);
  // tiles holding some t >= s: (I, J) of 128 x 128 (one CTA), (I2, J) of
  // 256 x 128 (a CTA pair)
  std::vector<int2> tiles;
  const i64 TI = pairs ? RA / 2 : RA, TM = pairs ? 256 : 128, TJ = (G + 127) / 128;
  for (i64 I = 0; I < TI; ++I)
    for (i64 J = 0; J < TJ; ++J)
      if (J * 128 + 127 >= row0 + I * TM) tiles.push_back(make_int2(static_cast<int>(I), static_cast<int>(J)));
  DevBuf<int2> d_tiles(tiles.size());
  DFPCA_CUDA(cudaMemcpyAsync(d_tiles.get(), tiles.data(), sizeof(int2) * tiles.size(), cudaMemcpyHostToDevice, st));
  if (pairs) {
    allow_smem(k_oz_syrk2, kOz2Smem);
    const unsigned grid = static_cast<unsigned>(2 * std::min<i64>(static_cast<i64>(tiles.size()), ctx->sm_count / 2));
    DFPCA_LAUNCH(ctx, k_oz_syrk2, grid, kOzThreads, kOz2Smem, xs.get(), ys.get(), nch, sx.get(), sy.get(), G, C, ldc,
                 d_tiles.get(), static_cast<int>(tiles.size()), row0, row1);
  } else {
    allow_smem(k_oz_syrk, kOzSmem);
    const unsigned grid = static_cast<unsigned>(std::min<i64>(static_cast<i64>(tiles.size()), ctx->sm_count));
    DFPCA_LAUNCH_PDL(ctx, k_oz_syrk, grid, kOzThreads, kOzSmem, xs.get(), ys.get(), nch, sx.get(), sy.get(), G, C, ldc,
                 d_tiles.get(), static_cast<int>(tiles.size()), row0, row1);
  }
  return true;
}

}  // namespace dfpca_gpu
