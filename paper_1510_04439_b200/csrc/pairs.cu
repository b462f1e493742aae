// K2: pair-product grids (reference PairGridSource, fft_smoother.hpp:291-443).
//
//   pw(s,t) = sum_i w_i M_i(s) M_i(t) - diag_mass band
//   pv(s,t) = sum_i w_i V_i(s) V_i(t) - diag_value band
//
// The sum over samples is a SYRK with K = n_pair: computed on the FP64 tensor
// pipe (gemm.cu) for the upper tile triangle and mirrored.  When every sample
// has the same mass grid (the GridNodes / shared-design case, detected at
// binning time) pw is the rank-one product W M(s) M(t) and costs one pass.
//
// Exactness where it matters.  Near the diagonal the reference's pw is
// "sample sum minus band", and for pairs that only share one observation the
// two sums are identical sequences, so the reference gets an exact 0 there
// (which later decides whether a kernel window is empty).  A reordered SYRK
// would leave +-1 ulp there.  k_band_fix therefore recomputes every pw entry
// with a nonzero band in the reference order -- samples ascending, separate
// multiply and add, (w_i M_i(s)) M_i(t) (fft_smoother.hpp:397-402) -- and
// subtracts the band once (:433-434), making those entries bit-identical.
//
// Sparse designs (few observations per subject, e.g. config 4: 5-20 per
// subject on 64^2 nodes) take a different route: the per-sample nonzeros are
// compacted (node-ascending, as the reference's Nonzeros), every sample emits
// one record per (s, t) pair of its nonzeros, a stable radix sort groups the
// records by (s, t) keeping sample order, and one thread per entry adds the
// terms (w_i M_i(s)) M_i(t) in that order -- the reference's sequence of
// operations exactly -- before the band subtraction.  Both grids are then
// bit-identical to the reference's, and the cost follows sum_i nnz_i^2
// instead of n G^2.
#include <cub/cub.cuh>

#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>

#include "gemm.cuh"
#include "pairs.cuh"
#include "shard.hpp"

namespace dfpca_gpu {
namespace {

// pw over rows [row0, row0 + rows), columns [col0, G) of the window
// (pw points at row row0, leading dimension G).
__global__ void k_rank_one(double* __restrict__ pw, const double* __restrict__ m, double W, i64 G, i64 row0,
                           i64 rows, i64 col0) {
  pdl_wait();
  const i64 w = G - col0;
  const i64 total = rows * w;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 r = e / w, t = col0 + e % w;
    pw[r * G + t] = __dmul_rn(__dmul_rn(W, m[row0 + r]), m[t]);
  }
}

// Band fix-up, one warp per band entry (u, code) with a nonzero band.
//  * pw: recomputed exactly in the reference order and minus the band, so the
//    near-diagonal cancellations that decide empty windows are bit-identical.
//    The lanes form the per-sample products (w_i M_i(s)) M_i(t) of 32
//    consecutive samples in parallel (one rounded multiply pair each, as in
//    the reference) and lane 0 adds them in ascending sample order.  With a
//    shared mass grid (identical_mass) M_i(s) = M(s) for every i.
//  * pv: only the band subtraction (pv never decides emptiness; the SYRK sum
//    differs from the reference's by reassociation only).
//  * pw == nullptr: the pv subtraction alone (shared-design covariance, whose
//    mass moments come in closed form, smooth.cu).
__global__ void k_band_fix(const double* __restrict__ diag_mass, const double* __restrict__ diag_value,
                           i64 G, int d, i64 codes, DevGrid g, const double* __restrict__ ps_mass,
                           int identical, const double* __restrict__ w, i64 n_pair, double w_seq,
                           double* __restrict__ pw, double* __restrict__ pv, i64 row0, i64 rows, i64 col0) {
  pdl_wait();
  // window: band entries of rows u in [row0, row0 + rows) and columns t >= col0;
  // pw / pv point at row row0 (leading dimension G)
  const int lane = threadIdx.x & 31;
  const i64 warps = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  const i64 total = rows * codes;
  for (i64 e0 = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5; e0 < total; e0 += warps) {
    const i64 e = e0 + row0 * codes;
    const double dm = diag_mass[e], dv = diag_value[e];
    if (dm == 0.0 && dv == 0.0) continue;
    const i64 u = e / codes;
    i64 code = e % codes;
    int off[kMaxDim];
    for (int k = d - 1; k >= 0; --k) {
      off[k] = static_cast<int>(code % 3) - 1;
      code /= 3;
    }
    i64 rem = u, t = 0;
    bool inside = true;
    for (int k = d - 1; k >= 0; --k) {
      const i64 a = rem % g.shape[k];
      rem /= g.shape[k];
      const i64 bk = a + off[k];
      if (bk < 0 || bk >= g.shape[k]) inside = false;
      t += bk * g.strides[k];
    }
    if (!inside || t < col0) continue;
    const i64 at = (u - row0) * G + t;
    if (pw == nullptr) {  // value grid only (shared-design covariance)
      if (lane == 0) pv[at] = __dsub_rn(pv[at], dv);
      continue;
    }
    double sw = 0.0;
    const double ms0 = identical ? ps_mass[u] : 0.0, mt0 = identical ? ps_mass[t] : 0.0;
    // shared unit masses (every subject observed once at both nodes):
    // (w_i * 1) * 1 == w_i, so the ordered sum is the ordered sum of the
    // weights, W_seq, computed once on the host in the same order
    const bool unit = identical && ms0 == 1.0 && mt0 == 1.0;
    if (unit) sw = w_seq;
    for (i64 i0 = 0; i0 < (unit ? 0 : n_pair); i0 += 32) {
      const i64 i = i0 + lane;
      double pm = 0.0;
      if (i < n_pair) {
        const double ms = identical ? ms0 : ps_mass[i * G + u];
        const double mt = identical ? mt0 : ps_mass[i * G + t];
        pm = __dmul_rn(__dmul_rn(w[i], ms), mt);
      }
      const int cnt = n_pair - i0 < 32 ? static_cast<int>(n_pair - i0) : 32;
      for (int q = 0; q < cnt; ++q) sw = __dadd_rn(sw, __shfl_sync(0xffffffffu, pm, q));
    }
    if (lane == 0) {
      pw[at] = __dsub_rn(sw, dm);
      pv[at] = __dsub_rn(pv[at], dv);
    }
  }
}


// ------------------------------------------------------------ sparse pairs --
constexpr int kSparseThreads = 256;

// nonzero count of every per-sample mass grid (block per sample)
__global__ void __launch_bounds__(kSparseThreads) k_nnz_count(const double* __restrict__ ps_mass, i64 G,
                                                              i64* __restrict__ nnz) {
  pdl_wait();
  using Reduce = cub::BlockReduce<i64, kSparseThreads>;
  __shared__ typename Reduce::TempStorage tmp;
  const double* m = ps_mass + static_cast<i64>(blockIdx.x) * G;
  i64 c = 0;
  for (i64 f = threadIdx.x; f < G; f += kSparseThreads) c += m[f] != 0.0 ? 1 : 0;
  const i64 total = Reduce(tmp).Sum(c);
  if (threadIdx.x == 0) nnz[blockIdx.x] = total;
}

// node-ascending compaction of sample blockIdx.x's nonzeros; per sample the
// local ranges of nonzeros in the window rows [row0, row0 + rows) and in the
// window columns [col0, G)
__global__ void __launch_bounds__(kSparseThreads) k_nnz_compact(const double* __restrict__ ps_mass,
                                                                const double* __restrict__ ps_value, i64 G,
                                                                const i64* __restrict__ nz_off, i64 row0, i64 rows,
                                                                i64 col0, int* __restrict__ nz_f,
                                                                double* __restrict__ nz_m, double* __restrict__ nz_v,
                                                                int* __restrict__ nz_s, i64* __restrict__ ranges) {
  pdl_wait();
  using Scan = cub::BlockScan<int, kSparseThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int base;
  const int i = blockIdx.x;
  const double* m = ps_mass + static_cast<i64>(i) * G;
  const double* v = ps_value + static_cast<i64>(i) * G;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  int a_lo = 0, a_hi = 0, b_lo = 0;  // counts of nonzeros below row0, below row0 + rows, below col0
  for (i64 f0 = 0; f0 < G; f0 += kSparseThreads) {
    const i64 f = f0 + threadIdx.x;
    const int nz = (f < G && m[f] != 0.0) ? 1 : 0;
    int pos, tot;
    Scan(tmp).ExclusiveSum(nz, pos, tot);
    if (nz) {
      const i64 o = nz_off[i] + base + pos;
      nz_f[o] = static_cast<int>(f);
      nz_m[o] = m[f];
      nz_v[o] = v[f];
      nz_s[o] = i;
    }
    a_lo += (nz && f < row0) ? 1 : 0;
    a_hi += (nz && f < row0 + rows) ? 1 : 0;
    b_lo += (nz && f < col0) ? 1 : 0;
    __syncthreads();
    if (threadIdx.x == 0) base += tot;
    __syncthreads();
  }
  using Reduce = cub::BlockReduce<int, kSparseThreads>;
  __shared__ typename Reduce::TempStorage rtmp;
  const int A0 = Reduce(rtmp).Sum(a_lo);
  __syncthreads();
  const int A1 = Reduce(rtmp).Sum(a_hi);
  __syncthreads();
  const int B0 = Reduce(rtmp).Sum(b_lo);
  if (threadIdx.x == 0) {
    ranges[3 * i] = A0;
    ranges[3 * i + 1] = A1;
    ranges[3 * i + 2] = B0;
  }
}

// one record per (window row nonzero a, window column nonzero b) of sample
// blockIdx.x, key = (s - row0) * (G - col0) + (t - col0), records of sample i
// before those of sample i + 1
__global__ void __launch_bounds__(kSparseThreads) k_pair_emit(const i64* __restrict__ nz_off,
                                                              const i64* __restrict__ ranges,
                                                              const i64* __restrict__ rec_off,
                                                              const int* __restrict__ nz_f, i64 G, i64 row0, i64 col0,
                                                              unsigned long long* __restrict__ key,
                                                              unsigned* __restrict__ val, unsigned* __restrict__ ra,
                                                              unsigned* __restrict__ rb) {
  pdl_wait();
  const int i = blockIdx.x;
  const i64 off = nz_off[i], end = nz_off[i + 1];
  const i64 a0 = off + ranges[3 * i], a1 = off + ranges[3 * i + 1], b0 = off + ranges[3 * i + 2];
  const i64 na = a1 - a0, nb = end - b0;
  const i64 cols = G - col0;
  for (i64 q = threadIdx.x; q < na * nb; q += kSparseThreads) {
    const i64 a = a0 + q / nb, b = b0 + q % nb;
    const i64 r = rec_off[i] + q;
    key[r] = static_cast<unsigned long long>(nz_f[a] - row0) * cols + (nz_f[b] - col0);
    val[r] = static_cast<unsigned>(r);
    ra[r] = static_cast<unsigned>(a);
    rb[r] = static_cast<unsigned>(b);
  }
}

// one thread per (s, t) with records: the samples' terms in ascending sample
// order, (w_i M_i(s)) M_i(t) and (w_i V_i(s)) V_i(t) (fft_smoother.hpp:397-402)
__global__ void k_pair_sum(const unsigned long long* __restrict__ key, const unsigned* __restrict__ val, i64 n_rec,
                           const unsigned* __restrict__ ra, const unsigned* __restrict__ rb,
                           const double* __restrict__ nz_m, const double* __restrict__ nz_v,
                           const int* __restrict__ nz_s, const double* __restrict__ w, i64 G, i64 col0,
                           double* __restrict__ pw, double* __restrict__ pv) {
  pdl_wait();
  const i64 cols = G - col0;
  for (i64 r0 = blockIdx.x * (i64)blockDim.x + threadIdx.x; r0 < n_rec; r0 += (i64)gridDim.x * blockDim.x) {
    const unsigned long long k = key[r0];
    if (r0 > 0 && key[r0 - 1] == k) continue;  // not a segment head
    double sm = 0.0, sv = 0.0;
    for (i64 r = r0; r < n_rec && key[r] == k; ++r) {
      const unsigned rec = val[r];
      const unsigned a = ra[rec], b = rb[rec];
      const double wi = w[nz_s[a]];
      sm = __dadd_rn(sm, __dmul_rn(__dmul_rn(wi, nz_m[a]), nz_m[b]));
      sv = __dadd_rn(sv, __dmul_rn(__dmul_rn(wi, nz_v[a]), nz_v[b]));
    }
    const i64 at = static_cast<i64>(k / cols) * G + col0 + static_cast<i64>(k % cols);
    if (pw) pw[at] = sm;
    pv[at] = sv;
  }
}

// the band subtraction alone (fft_smoother.hpp:410-436) over the window
__global__ void k_band_sub(const double* __restrict__ diag_mass, const double* __restrict__ diag_value, i64 G,
                           int d, i64 codes, DevGrid g, double* __restrict__ pw, double* __restrict__ pv, i64 row0,
                           i64 rows, i64 col0) {
  pdl_wait();
  const i64 total = rows * codes;
  for (i64 e0 = blockIdx.x * (i64)blockDim.x + threadIdx.x; e0 < total; e0 += (i64)gridDim.x * blockDim.x) {
    const i64 e = e0 + row0 * codes;
    const double dm = diag_mass[e], dv = diag_value[e];
    if (dm == 0.0 && dv == 0.0) continue;
    const i64 u = e / codes;
    i64 code = e % codes;
    int off[kMaxDim];
    for (int k = d - 1; k >= 0; --k) {
      off[k] = static_cast<int>(code % 3) - 1;
      code /= 3;
    }
    i64 rem = u, t = 0;
    bool inside = true;
    for (int k = d - 1; k >= 0; --k) {
      const i64 a = rem % g.shape[k];
      rem /= g.shape[k];
      const i64 bk = a + off[k];
      if (bk < 0 || bk >= g.shape[k]) inside = false;
      t += bk * g.strides[k];
    }
    if (!inside || t < col0) continue;
    const i64 at = (u - row0) * G + t;
    if (pw) pw[at] = __dsub_rn(pw[at], dm);
    pv[at] = __dsub_rn(pv[at], dv);
  }
}

int key_bits64(unsigned long long max_key) {
  int b = 1;
  while (b < 64 && (max_key >> b) != 0) ++b;
  return b;
}

// Largest record count the sparse route takes (32 B per record).
constexpr i64 kMaxSparseRecords = i64{1} << 27;

// Sparse pair grids over the window (see the file comment).
void build_pair_grids_sparse(dfpca_context* ctx, const dfpca_binned* b, double* pw, double* pv, const PairWindow& w,
                             const DevGrid& dg) {
  cudaStream_t st = ctx->stream;
  const i64 G = b->grid.G, n = b->n_pair;
  const std::vector<i64>& nnz = b->pair_nnz;
  std::vector<i64> nz_off(static_cast<std::size_t>(n) + 1, 0);
  for (i64 i = 0; i < n; ++i) nz_off[static_cast<std::size_t>(i) + 1] = nz_off[static_cast<std::size_t>(i)] + nnz[static_cast<std::size_t>(i)];
  const i64 NZ = nz_off.back();
  DevBuf<i64> d_nz_off(static_cast<std::size_t>(n) + 1), ranges(static_cast<std::size_t>(3 * n));
  DevBuf<int> nz_f(static_cast<std::size_t>(std::max<i64>(NZ, 1))), nz_s(static_cast<std::size_t>(std::max<i64>(NZ, 1)));
  DevBuf<double> nz_m(static_cast<std::size_t>(std::max<i64>(NZ, 1))), nz_v(static_cast<std::size_t>(std::max<i64>(NZ, 1)));
  DFPCA_CUDA(cudaMemcpyAsync(d_nz_off.get(), nz_off.data(), sizeof(i64) * nz_off.size(), cudaMemcpyHostToDevice, st));
  const i64 rows = w.rows, cols = G - w.col0;
  DFPCA_LAUNCH(ctx, k_nnz_compact, static_cast<unsigned>(n), kSparseThreads, 0, b->ps_mass.get(), b->ps_value.get(),
               G, d_nz_off.get(), w.row0, rows, w.col0, nz_f.get(), nz_m.get(), nz_v.get(), nz_s.get(), ranges.get());
  std::vector<i64> rg(static_cast<std::size_t>(3 * n));
  DFPCA_CUDA(cudaMemcpyAsync(rg.data(), ranges.get(), sizeof(i64) * rg.size(), cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
  std::vector<i64> rec_off(static_cast<std::size_t>(n) + 1, 0);
  for (i64 i = 0; i < n; ++i) {
    const std::size_t k = static_cast<std::size_t>(i);
    const i64 na = rg[3 * k + 1] - rg[3 * k], nb = nnz[k] - rg[3 * k + 2];
    rec_off[k + 1] = rec_off[k] + na * nb;
  }
  const i64 R = rec_off.back();
  if (pw) DFPCA_CUDA(cudaMemsetAsync(pw, 0, sizeof(double) * static_cast<std::size_t>(rows * G), st));
  DFPCA_CUDA(cudaMemsetAsync(pv, 0, sizeof(double) * static_cast<std::size_t>(rows * G), st));
  if (R > 0) {
    DevBuf<i64> d_rec_off(rec_off.size());
    DFPCA_CUDA(cudaMemcpyAsync(d_rec_off.get(), rec_off.data(), sizeof(i64) * rec_off.size(), cudaMemcpyHostToDevice,
                               st));
    const std::size_t NR = static_cast<std::size_t>(R);
    DevBuf<unsigned long long> key(NR), key2(NR);
    DevBuf<unsigned> val(NR), val2(NR), ra(NR), rb(NR);
    DFPCA_LAUNCH(ctx, k_pair_emit, static_cast<unsigned>(n), kSparseThreads, 0, d_nz_off.get(), ranges.get(),
                 d_rec_off.get(), nz_f.get(), G, w.row0, w.col0, key.get(), val.get(), ra.get(), rb.get());
    const int bits = key_bits64(static_cast<unsigned long long>(rows) * cols);
    std::size_t sb = 0;
    DFPCA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sb, key.get(), key2.get(), val.get(), val2.get(), R, 0, bits,
                                               st));
    unsigned char* stmp = ctx->scratch_bytes(sb);
    DFPCA_CUDA(cub::DeviceRadixSort::SortPairs(stmp, sb, key.get(), key2.get(), val.get(), val2.get(), R, 0, bits,
                                               st));
    ctx->launches += (bits + 7) / 8 + 1;
    DFPCA_LAUNCH(ctx, k_pair_sum, grid_for(R, 256, 148ll * 32), 256, 0, key2.get(), val2.get(), R, ra.get(),
                 rb.get(), nz_m.get(), nz_v.get(), nz_s.get(), b->pair_weight.get(), G, w.col0, pw, pv);
  }
  DFPCA_LAUNCH(ctx, k_band_sub, grid_for(rows * b->codes, 256), 256, 0, b->diag_mass.get(), b->diag_value.get(), G,
               b->grid.d, b->codes, dg, pw, pv, w.row0, rows, w.col0);
}

}  // namespace

DevGrid upload_grid_axes(dfpca_context* ctx, const Grid& g, DevBuf<double>& storage);

bool pair_grids_sparse(dfpca_context* ctx, const dfpca_binned* b) {
  if (b->pair_route >= 0) return b->pair_route == 1;
  const i64 G = b->grid.G, n = b->n_pair;
  b->pair_route = 0;
  if (n <= 0) return false;
  const char* force = std::getenv("DFPCA_PAIRS");  // tests: "sparse" / "dense"
  if (force && std::strcmp(force, "dense") == 0) return false;
  DevBuf<i64> cnt(static_cast<std::size_t>(n));
  DFPCA_LAUNCH(ctx, k_nnz_count, static_cast<unsigned>(n), kSparseThreads, 0, b->ps_mass.get(), G, cnt.get());
  b->pair_nnz.assign(static_cast<std::size_t>(n), 0);
  DFPCA_CUDA(cudaMemcpyAsync(b->pair_nnz.data(), cnt.get(), sizeof(i64) * static_cast<std::size_t>(n),
                             cudaMemcpyDeviceToHost, ctx->stream));
  DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  double P = 0.0;  // sum_i nnz_i^2: records of the full grid
  for (i64 c : b->pair_nnz) P += static_cast<double>(c) * static_cast<double>(c);
  const bool forced = force && std::strcmp(force, "sparse") == 0;
  // records cost a sort pass each; the SYRK n G^2 / 2 tensor-pipe FMAs: the
  // sparse route wins by far below the 1/64 ratio (config 4: ~1/10^4)
  const bool sparse = P <= static_cast<double>(kMaxSparseRecords) &&
                      (forced || P * 64.0 <= static_cast<double>(n) * static_cast<double>(G) * static_cast<double>(G));
  b->pair_route = sparse ? 1 : 0;
  return sparse;
}

void build_pair_grids(dfpca_context* ctx, const dfpca_binned* b, double* pw, double* pv, const PairWindow* win,
                      const std::function<void(bool pw_from_syrk)>& exchange) {
  const i64 G = b->grid.G;
  const i64 n = b->n_pair;
  PairWindow full;
  full.rows = G;
  const PairWindow& w = win ? *win : full;
  if (pair_grids_sparse(ctx, b)) {  // every rank computes its whole window: no exchange
    DevBuf<double> axes;
    const DevGrid dg = upload_grid_axes(ctx, b->grid, axes);
    build_pair_grids_sparse(ctx, b, pw, pv, w, dg);
    return;
  }
  const i64 tiles = (G + kShardRowTile - 1) / kShardRowTile;
  const i64 tm_end = w.tm_end < 0 ? tiles : w.tm_end;
  // own SYRK rows inside the window buffer
  const i64 own = w.tm_begin * kShardRowTile - w.row0;
  double W = 0.0;
  for (double x : b->pair_weight_h) W += x;  // sequential, as the reference's sample loop
  DevBuf<double> axes;
  const DevGrid dg = upload_grid_axes(ctx, b->grid, axes);  // (synchronizes: before the SYRK is queued)
  if (pw) {
    if (b->identical_mass) {
      DFPCA_LAUNCH(ctx, k_rank_one, grid_for(w.rows * (G - w.col0), 256, 148ll * 16), 256, 0, pw,
                   b->ps_mass.get(), W, G, w.row0, w.rows, w.col0);
    } else {
      gemm_tn(ctx, G, G, n, b->ps_mass.get(), G, b->pair_weight.get(), b->ps_mass.get(), G, pw + own * G, G, true,
              w.tm_begin, tm_end);
    }
  }
  if (pv)
    gemm_tn(ctx, G, G, n, b->ps_value.get(), G, b->pair_weight.get(), b->ps_value.get(), G, pv + own * G, G, true,
            w.tm_begin, tm_end);
  if (exchange) exchange(pw != nullptr && !b->identical_mass);
  if (pv)
    DFPCA_LAUNCH_PDL(ctx, k_band_fix, grid_for(w.rows * b->codes * 32, 256, 148ll * 32), 256, 0,
                 b->diag_mass.get(), b->diag_value.get(), G, b->grid.d, b->codes, dg,
                 b->ps_mass.get(), b->identical_mass ? 1 : 0, b->pair_weight.get(), n, W, pw, pv, w.row0, w.rows,
                 w.col0);
}

}  // namespace dfpca_gpu
