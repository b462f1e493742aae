// Long-format observation tables on the device:
// the reference's read_long_format (io.hpp:115-155) -- header row, sniffed
// delimiter, one record per observation, rows grouped by sample id in order
// of first appearance -- with the bytes parsed on the GPU.
//
//   upload     the file is read by host threads into pinned slots and copied
//              to HBM chunk by chunk (pread and H2D overlap);
//   lines      newline positions: per-tile popcounts of a SWAR byte match,
//              a device scan, then an ordered write (k_nl_count / k_nl_write);
//   records    one thread per line strips '\r', skips empty lines, splits
//              with the reference's field rule and checks the field count
//              (k_split_lines); then one thread per (number column, line)
//              parses a field with numparse.cuh (exact, strtod-identical;
//              k_parse_fields) -- the first failing (line, field) is kept with
//              an atomicMin, so the error is the one the sequential reader
//              raises first;
//   samples    lines whose id differs from the previous record's start a run;
//              run heads are grouped by an exact string sort (stable LSD radix
//              passes over 8-byte chunks, then the length), numbered in order
//              of first appearance, and the records are scattered into the
//              CSR layout sample by sample, file order within a sample.
//
// Only the header line (and, on failure, the failing line) is examined on
// the host, to sniff the delimiter and to word the reference's messages.
#include <sched.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "numparse.cuh"

struct dfpca_table {
  int dim = 0;
  std::int64_t n_samples = 0, n_obs = 0, id_bytes = 0;
  dfpca_gpu::DevBuf<std::int64_t> offsets;  // n_samples + 1
  dfpca_gpu::DevBuf<double> coords, values;
  dfpca_gpu::DevBuf<std::int64_t> id_off;  // n_samples + 1
  dfpca_gpu::DevBuf<char> id_chars;
};

namespace dfpca_gpu {
namespace {

using numparse::Pow5;
using u64 = unsigned long long;

__device__ const Pow5 d_pow5[] = {
#include "pow5_128.inc"
};

constexpr int kThreads = 256;
constexpr int kMaxFields = 32;

// ------------------------------------------------------------------ upload --
constexpr std::size_t kSlotBytes = 8u << 20;

struct IoState {
  int workers = 0;           // pool size (downloads use them all)
  int upload_workers = 0;    // uploads: 8 unless DFPCA_IO_WORKERS sets the pool
  std::vector<char*> slot;   // 2 per worker, pinned, allocated on a worker's first use
  std::vector<cudaStream_t> stream;
  std::vector<cudaEvent_t> slot_done, worker_done;
  std::mutex mu;
  ~IoState() {
    for (char* p : slot)
      if (p) cudaFreeHost(p);
    for (auto s : stream)
      if (s) cudaStreamDestroy(s);
    for (auto e : slot_done)
      if (e) cudaEventDestroy(e);
    for (auto e : worker_done)
      if (e) cudaEventDestroy(e);
  }
  // pinned slots, stream and events of workers [0, W) (caller holds mu)
  void prepare(int W) {
    for (int w = 0; w < W; ++w) {
      if (stream[static_cast<std::size_t>(w)]) continue;
      for (int s = 0; s < 2; ++s) {
        const std::size_t i = static_cast<std::size_t>(2 * w + s);
        DFPCA_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&slot[i]), kSlotBytes, cudaHostAllocDefault));
        DFPCA_CUDA(cudaEventCreateWithFlags(&slot_done[i], cudaEventDisableTiming));
      }
      DFPCA_CUDA(cudaEventCreateWithFlags(&worker_done[static_cast<std::size_t>(w)], cudaEventDisableTiming));
      DFPCA_CUDA(cudaStreamCreateWithFlags(&stream[static_cast<std::size_t>(w)], cudaStreamNonBlocking));
    }
  }
};

// CPUs this process may run on (affinity / cgroup cpusets), not the machine's.
int usable_cpus() {
  cpu_set_t set;
  if (sched_getaffinity(0, sizeof(set), &set) == 0) return std::max(1, CPU_COUNT(&set));
  return static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
}

IoState& io_state(dfpca_context* ctx) {
  if (!ctx->io_state) {
    auto io = std::make_shared<IoState>();
    // downloads use every worker, uploads at most 8 (measured on the 16-core
    // host, 134 MB pageable: download 7.7 ms with 8 workers, 6.1 with 16;
    // upload 5.3 ms with 8, slower with more); an explicit DFPCA_IO_WORKERS
    // sizes both
    io->workers = std::min(16, usable_cpus());
    io->upload_workers = std::min(io->workers, 8);
    if (const char* e = std::getenv("DFPCA_IO_WORKERS"); e && *e) {
      io->workers = std::max(1, std::min(64, std::atoi(e)));
      io->upload_workers = io->workers;
    }
    const auto W = static_cast<std::size_t>(io->workers);
    io->slot.assign(2 * W, nullptr);
    io->slot_done.assign(2 * W, nullptr);
    io->stream.assign(W, nullptr);
    io->worker_done.assign(W, nullptr);
    ctx->io_state = io;
  }
  return *static_cast<IoState*>(ctx->io_state.get());
}

// Copies S bytes produced by fill(dst, offset, len) into d_text, chunk by
// chunk through the pinned slots, on `workers` host threads.
template <class Fill>
void upload_bytes(dfpca_context* ctx, char* d_text, i64 S, Fill fill) {
  IoState& io = io_state(ctx);
  std::lock_guard<std::mutex> lk(io.mu);
  const i64 n_chunks = (S + static_cast<i64>(kSlotBytes) - 1) / static_cast<i64>(kSlotBytes);
  const int W = static_cast<int>(std::min<i64>(io.upload_workers, std::max<i64>(n_chunks, 1)));
  io.prepare(W);
  // the slots' previous copies (an earlier call) were ordered on the worker
  // streams; the destination's stream-ordered allocation is ordered by `ready`
  cudaEvent_t ready;
  DFPCA_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  DFPCA_CUDA(cudaEventRecord(ready, ctx->stream));
  struct Ev {
    cudaEvent_t e;
    ~Ev() { cudaEventDestroy(e); }
  } ready_guard{ready};
  std::vector<std::string> errs(static_cast<std::size_t>(W));
  auto work = [&](int w) {
    if (cudaSetDevice(ctx->device) != cudaSuccess ||
        cudaStreamWaitEvent(io.stream[static_cast<std::size_t>(w)], ready, 0) != cudaSuccess) {
      errs[static_cast<std::size_t>(w)] = "cudaSetDevice failed";
      return;
    }
    int k = 0;
    for (i64 c = w; c < n_chunks; c += W, ++k) {
      const std::size_t s = static_cast<std::size_t>(2 * w + (k & 1));
      if (cudaEventSynchronize(io.slot_done[s]) != cudaSuccess) {
        errs[static_cast<std::size_t>(w)] = "slot event failed";
        return;
      }
      const i64 off = c * static_cast<i64>(kSlotBytes);
      const i64 len = std::min<i64>(static_cast<i64>(kSlotBytes), S - off);
      const std::string e = fill(io.slot[s], off, len);
      if (!e.empty()) {
        errs[static_cast<std::size_t>(w)] = e;
        return;
      }
      if (cudaMemcpyAsync(d_text + off, io.slot[s], static_cast<std::size_t>(len), cudaMemcpyHostToDevice,
                          io.stream[static_cast<std::size_t>(w)]) != cudaSuccess ||
          cudaEventRecord(io.slot_done[s], io.stream[static_cast<std::size_t>(w)]) != cudaSuccess) {
        errs[static_cast<std::size_t>(w)] = "host-to-device copy failed";
        return;
      }
    }
  };
  std::vector<std::thread> th;
  for (int w = 1; w < W; ++w) th.emplace_back(work, w);
  work(0);
  for (auto& t : th) t.join();
  for (int w = 0; w < W; ++w) {
    DFPCA_CUDA(cudaEventRecord(io.worker_done[static_cast<std::size_t>(w)], io.stream[static_cast<std::size_t>(w)]));
    DFPCA_CUDA(cudaStreamWaitEvent(ctx->stream, io.worker_done[static_cast<std::size_t>(w)], 0));
  }
  for (const auto& e : errs)
    if (!e.empty()) fail(kParse, "IoError", e);
}

// Device -> pageable host copy through the pinned slots: each worker
// double-buffers its chunks (D2H of chunk k + 1 overlaps the host memcpy of
// chunk k), so large results leave at pinned speed.
void download_bytes(dfpca_context* ctx, char* dst, const char* d_src, i64 bytes) {
  if (bytes <= 0) return;
  IoState& io = io_state(ctx);
  std::lock_guard<std::mutex> lk(io.mu);
  const i64 slot = static_cast<i64>(kSlotBytes);
  const i64 n_chunks = (bytes + slot - 1) / slot;
  const int W = static_cast<int>(std::min<i64>(io.workers, n_chunks));
  io.prepare(W);
  cudaEvent_t ready;
  DFPCA_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  DFPCA_CUDA(cudaEventRecord(ready, ctx->stream));
  std::vector<std::string> errs(static_cast<std::size_t>(W));
  auto work = [&](int w) {
    const std::size_t ws = static_cast<std::size_t>(w);
    cudaStream_t st = io.stream[ws];
    if (cudaSetDevice(ctx->device) != cudaSuccess || cudaStreamWaitEvent(st, ready, 0) != cudaSuccess) {
      errs[ws] = "device-to-host copy failed";
      return;
    }
    auto issue = [&](i64 c, int b) {
      const i64 off = c * slot, len = std::min<i64>(slot, bytes - off);
      return cudaMemcpyAsync(io.slot[2 * ws + b], d_src + off, static_cast<std::size_t>(len), cudaMemcpyDeviceToHost,
                             st) == cudaSuccess &&
             cudaEventRecord(io.slot_done[2 * ws + b], st) == cudaSuccess;
    };
    if (!issue(w, 0)) {
      errs[ws] = "device-to-host copy failed";
      return;
    }
    int k = 0;
    for (i64 c = w; c < n_chunks; c += W, ++k) {
      const int b = k & 1;
      if ((c + W < n_chunks && !issue(c + W, b ^ 1)) || cudaEventSynchronize(io.slot_done[2 * ws + b]) != cudaSuccess) {
        errs[ws] = "device-to-host copy failed";
        return;
      }
      const i64 off = c * slot, len = std::min<i64>(slot, bytes - off);
      std::memcpy(dst + off, io.slot[2 * ws + b], static_cast<std::size_t>(len));
    }
  };
  std::vector<std::thread> th;
  for (int w = 1; w < W; ++w) th.emplace_back(work, w);
  work(0);
  for (auto& t : th) t.join();
  cudaEventDestroy(ready);
  for (const auto& e : errs)
    if (!e.empty()) fail(kNumeric, "DeviceError", e);
}

}  // namespace

// Pinned host memory is copied directly; large pageable buffers go through
// the pinned slots on the worker threads (the driver's own pageable path runs
// at a fraction of PCIe speed: measured 197 MB in ~16 ms vs ~4 ms pinned).
constexpr i64 kStageMinBytes = i64{8} << 20;

bool is_pinned_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

bool copy_is_staged(const void* host, i64 bytes) { return bytes >= kStageMinBytes && !is_pinned_host(host); }

void copy_h2d(dfpca_context* ctx, void* d_dst, const void* src, i64 bytes) {
  if (bytes <= 0) return;
  if (!copy_is_staged(src, bytes)) {
    DFPCA_CUDA(cudaMemcpyAsync(d_dst, src, static_cast<std::size_t>(bytes), cudaMemcpyHostToDevice, ctx->stream));
    return;
  }
  const char* s = static_cast<const char*>(src);
  upload_bytes(ctx, static_cast<char*>(d_dst), bytes, [&](char* slot, i64 off, i64 len) -> std::string {
    std::memcpy(slot, s + off, static_cast<std::size_t>(len));
    return {};
  });
}

void copy_d2h(dfpca_context* ctx, void* dst, const void* d_src, i64 bytes) {
  if (bytes <= 0) return;
  if (!copy_is_staged(dst, bytes)) {
    DFPCA_CUDA(cudaMemcpyAsync(dst, d_src, static_cast<std::size_t>(bytes), cudaMemcpyDeviceToHost, ctx->stream));
    DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  download_bytes(ctx, static_cast<char*>(dst), static_cast<const char*>(d_src), bytes);
}

namespace {

// ------------------------------------------------------------- newlines --
// High bit of every byte of v that equals '\n' (exact SWAR zero-byte test).
__device__ __forceinline__ u64 newline_bits(u64 v) {
  const u64 x = v ^ 0x0A0A0A0A0A0A0A0Aull;
  const u64 y = (x & 0x7F7F7F7F7F7F7F7Full) + 0x7F7F7F7F7F7F7F7Full;
  return ~(y | x | 0x7F7F7F7F7F7F7F7Full);
}

__global__ void __launch_bounds__(kThreads) k_nl_count(const u64* __restrict__ text, i64 words, i64* counts) {
  pdl_wait();
  using Reduce = cub::BlockReduce<int, kThreads>;
  __shared__ typename Reduce::TempStorage tmp;
  const i64 tiles = (words + kThreads - 1) / kThreads;
  for (i64 t = blockIdx.x; t < tiles; t += gridDim.x) {
    const i64 w = t * kThreads + threadIdx.x;
    const int c = w < words ? __popcll(newline_bits(text[w])) : 0;
    const int s = Reduce(tmp).Sum(c);
    if (threadIdx.x == 0) counts[t] = s;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads) k_nl_write(const u64* __restrict__ text, i64 words,
                                                     const i64* __restrict__ tile_off, i64* nl) {
  pdl_wait();
  using Scan = cub::BlockScan<int, kThreads>;
  __shared__ typename Scan::TempStorage tmp;
  const i64 tiles = (words + kThreads - 1) / kThreads;
  for (i64 t = blockIdx.x; t < tiles; t += gridDim.x) {
    const i64 w = t * kThreads + threadIdx.x;
    u64 m = w < words ? newline_bits(text[w]) : 0ull;
    int pos;
    Scan(tmp).ExclusiveSum(__popcll(m), pos);
    i64 o = tile_off[t] + pos;
    while (m) {
      nl[o++] = w * 8 + (__ffsll(static_cast<long long>(m)) - 1) / 8;
      m &= m - 1;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- records --
struct Lines {
  const char* text;
  i64 S;
  const i64* nl;
  i64 n_nl;
  __device__ void bounds(i64 L, i64& st, i64& en) const {
    st = L == 0 ? 0 : nl[L - 1] + 1;
    en = L < n_nl ? nl[L] : S;
    if (en > st && text[en - 1] == '\r') --en;  // strip_cr (io.hpp:84-87)
  }
};

__device__ __forceinline__ bool ws(char c) { return numparse::is_space(c); }

struct SplitOut {
  i64* is_rec;       // per line: 1 if not empty
  i64* id_start;     // per line
  int* id_len;       // per line
  u64* fb;           // per line x F: (start << 32) | end, relative to the line start; fb[L F] = ~0: bad count
  u64* err;          // (line << 8) | code: 0 field count, 1 + k field k + 1, 255 internal
};

// Pass 1, one thread per line: one scan of the line's bytes records the
// field bounds (the reference's split rule) and checks the field count.
__global__ void __launch_bounds__(kThreads) k_split_lines(Lines ln, i64 n_lines, int F, char delim, SplitOut o) {
  pdl_wait();
  for (i64 L = 1 + blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; L < n_lines;
       L += static_cast<i64>(gridDim.x) * blockDim.x) {
    i64 st, en;
    ln.bounds(L, st, en);
    if (en == st) {
      o.is_rec[L] = 0;
      continue;
    }
    o.is_rec[L] = 1;
    u64* fb = o.fb + L * F;
    const char* t = ln.text;
    int nf = 0;
    if (delim) {
      i64 a = st;
      for (i64 i = st;; ++i) {
        const bool end = i == en;
        if (end || t[i] == delim) {
          if (nf < F) fb[nf] = (static_cast<u64>(a - st) << 32) | static_cast<u64>(i - st);
          ++nf;
          a = i + 1;
          if (end) break;
        }
      }
    } else {
      i64 i = st;
      while (true) {
        while (i < en && ws(t[i])) ++i;
        if (i >= en) break;
        const i64 a = i;
        while (i < en && !ws(t[i])) ++i;
        if (nf < F) fb[nf] = (static_cast<u64>(a - st) << 32) | static_cast<u64>(i - st);
        ++nf;
      }
    }
    if (nf != F) {
      fb[0] = ~0ull;
      atomicMin(o.err, static_cast<u64>(L) << 8);
      continue;
    }
    o.id_start[L] = st + static_cast<i64>(fb[0] >> 32);
    o.id_len[L] = static_cast<int>((fb[0] & 0xffffffffull) - (fb[0] >> 32));
  }
}

// Fast path of numparse::parse_double for the common token shape
// [+-]digits[.digits][(e|E)[+-]digits] with at most 19 mantissa digits, no
// blanks, at most 32 bytes: the token is read with aligned 8-byte loads into
// registers and scanned there (no per-byte memory round trip), giving the same
// (w, q) as the general parser and the same round_decimal; anything else --
// or an undecided rounding -- returns false and the general parser runs.
__device__ __forceinline__ bool fast_decimal(const char* text, i64 a, i64 len, double* out) {
  if (len <= 0 || len > 32) return false;
  const u64* base = reinterpret_cast<const u64*>(text + (a & ~i64{7}));
  const int sh = static_cast<int>(a & 7) * 8;
  const int nw = static_cast<int>(((a & 7) + len + 7) >> 3);
  u64 w[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) w[k] = k < nw ? base[k] : 0ull;
  u64 t[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) t[k] = sh ? ((w[k] >> sh) | (w[k + 1] << (64 - sh))) : w[k];
  u64 mant = 0;
  int nd = 0, frac = 0, ev = 0, ne = 0, estart = -1;
  bool dot = false, expo = false, neg = false, eneg = false, ok = true;
#pragma unroll
  for (int kw = 0; kw < 4; ++kw) {
    if (kw * 8 >= len) break;  // lanes of a warp parse one column: lengths alike
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = kw * 8 + j;
      if (i >= len) break;
      const unsigned c = static_cast<unsigned>((t[kw] >> (8 * j)) & 0xffu);
      const unsigned dg = c - '0';
      if (!expo) {
        if (dg < 10u) {
          mant = mant * 10u + dg;
          ++nd;
          frac += dot ? 1 : 0;
        } else if (c == '.' && !dot) {
          dot = true;
        } else if ((c == '-' || c == '+') && i == 0) {
          neg = c == '-';
        } else if ((c == 'e' || c == 'E') && nd > 0) {
          expo = true;
          estart = i + 1;
        } else {
          ok = false;
        }
      } else {
        if (dg < 10u) {
          ev = ev * 10 + static_cast<int>(dg);
          ++ne;
        } else if ((c == '-' || c == '+') && i == estart) {
          eneg = c == '-';
        } else {
          ok = false;
        }
      }
    }
  }
  if (!ok || nd == 0 || nd > 19 || (expo && (ne == 0 || ne > 4))) return false;
  const u64 sign = neg ? (u64{1} << 63) : 0ull;
  if (mant == 0) {
    *out = numparse::from_bits(sign);
    return true;
  }
  const int q = (eneg ? -ev : ev) - frac;
  if (q < numparse::kQMin || q > numparse::kQMax) return false;
  const numparse::Rounded r = numparse::round_decimal(mant, q, d_pow5);
  if (r.ambiguous) return false;
  return numparse::finish(sign, r.m, r.e2, out) == numparse::kOk;
}

// Pass 2, one thread per (number column k, line): 32 consecutive lines of
// one column per warp, so the lanes parse tokens of like shape; the lines are
// taken in chunks of kFieldChunk with all columns of a chunk next to each
// other, so a line's text is still in L2 when its other columns are parsed.
// Values are stored column-major, vals[k * n_lines + L].
constexpr i64 kFieldChunk = 4096;

__global__ void __launch_bounds__(kThreads) k_parse_fields(Lines ln, i64 n_lines, int F, const i64* is_rec,
                                                           const u64* fb, double* vals, u64* err) {
  pdl_wait();
  const int nv = F - 1;
  const i64 per = n_lines - 1;
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < per * nv;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 chunk = e / (kFieldChunk * nv);
    const i64 r = e - chunk * kFieldChunk * nv;
    const i64 c0 = chunk * kFieldChunk;
    const i64 span = per - c0 < kFieldChunk ? per - c0 : kFieldChunk;  // lines in this chunk
    const int k = static_cast<int>(r / span);
    const i64 L = 1 + c0 + (r - static_cast<i64>(k) * span);
    if (!is_rec[L] || fb[L * F] == ~0ull) continue;
    const u64 f = fb[L * F + 1 + k];
    const i64 st = L == 0 ? 0 : ln.nl[L - 1] + 1;
    const i64 a = st + static_cast<i64>(f >> 32), b = st + static_cast<i64>(f & 0xffffffffull);
    double v = 0.0;
    if (!fast_decimal(ln.text, a, b - a, &v)) {
      // strtod stops at an embedded NUL (the reference passes c_str())
      i64 z = a;
      while (z < b && ln.text[z] != '\0') ++z;
      const int stt = numparse::parse_double(ln.text + a, static_cast<int>(z - a), d_pow5, &v);
      if (stt != numparse::kOk) {
        atomicMin(err, (static_cast<u64>(L) << 8) | (stt == numparse::kInternal ? 255ull : static_cast<u64>(1 + k)));
        continue;
      }
    }
    vals[static_cast<i64>(k) * n_lines + L] = v;
  }
}

__global__ void k_rec_line(const i64* is_rec, const i64* rec_idx, i64 n_lines, i64* rec_line) {
  pdl_wait();
  for (i64 L = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; L < n_lines;
       L += static_cast<i64>(gridDim.x) * blockDim.x)
    if (is_rec[L]) rec_line[rec_idx[L]] = L;
}

__device__ bool same_id(const char* t, i64 a, int la, i64 b, int lb) {
  if (la != lb) return false;
  for (int i = 0; i < la; ++i)
    if (t[a + i] != t[b + i]) return false;
  return true;
}

__global__ void k_run_heads(const char* text, const i64* rec_line, const i64* id_start, const int* id_len, i64 n_rec,
                            i64* head) {
  pdl_wait();
  for (i64 r = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; r < n_rec;
       r += static_cast<i64>(gridDim.x) * blockDim.x) {
    if (r == 0) {
      head[r] = 1;
      continue;
    }
    const i64 L = rec_line[r], P = rec_line[r - 1];
    head[r] = same_id(text, id_start[L], id_len[L], id_start[P], id_len[P]) ? 0 : 1;
  }
}

// Heads: record index, id bounds, length; max id length.
__global__ void k_head_list(const i64* head, const i64* head_idx, const i64* rec_line, const i64* id_start,
                            const int* id_len, i64 n_rec, i64* head_rec, i64* h_start, int* h_len, int* max_len) {
  pdl_wait();
  for (i64 r = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; r < n_rec;
       r += static_cast<i64>(gridDim.x) * blockDim.x) {
    if (!head[r]) continue;
    const i64 h = head_idx[r], L = rec_line[r];
    head_rec[h] = r;
    h_start[h] = id_start[L];
    h_len[h] = id_len[L];
    atomicMax(max_len, id_len[L]);
  }
}

__global__ void k_iota(i64* p, i64 n) {
  pdl_wait();
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    p[i] = i;
}

// chunk c (8 bytes, big-endian, zero padded) of head perm[i]'s id, or its length (c < 0)
__global__ void k_chunk_keys(const char* text, const i64* h_start, const int* h_len, const i64* perm, i64 n, int c,
                             u64* keys) {
  pdl_wait();
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 h = perm[i];
    if (c < 0) {
      keys[i] = static_cast<u64>(h_len[h]);
      continue;
    }
    u64 k = 0;
    for (int b = 0; b < 8; ++b) {
      const int at = c * 8 + b;
      const unsigned char ch = at < h_len[h] ? static_cast<unsigned char>(text[h_start[h] + at]) : 0;
      k = (k << 8) | ch;
    }
    keys[i] = k;
  }
}

__global__ void k_group_flags(const char* text, const i64* h_start, const int* h_len, const i64* perm, i64 n,
                              i64* newgrp, i64* first_flag) {
  pdl_wait();
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 h = perm[i];
    const bool ng =
        i == 0 || !same_id(text, h_start[h], h_len[h], h_start[perm[i - 1]], h_len[perm[i - 1]]);
    newgrp[i] = ng ? 1 : 0;
    first_flag[h] = ng ? 1 : 0;  // stable sorts: a group's first element is its first head
  }
}

// sample of every head = rank (in head order) of its group's first head
__global__ void k_group_sample(const i64* perm, const i64* newgrp, const i64* grp_ex, const i64* rank, i64 n,
                               i64* sample_of_group, i64* first_head_of_sample) {
  pdl_wait();
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    if (!newgrp[i]) continue;
    const i64 s = rank[perm[i]];
    sample_of_group[grp_ex[i]] = s;
    first_head_of_sample[s] = perm[i];
  }
}

__global__ void k_head_sample(const i64* perm, const i64* newgrp, const i64* grp_ex, const i64* sample_of_group,
                              i64 n, u64* head_sample) {
  pdl_wait();
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    head_sample[perm[i]] = static_cast<u64>(sample_of_group[grp_ex[i] + newgrp[i] - 1]);
}

__global__ void k_run_lengths(const i64* sorted_heads, const i64* head_rec, i64 n_heads, i64 n_rec, i64* len) {
  pdl_wait();
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n_heads;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 h = sorted_heads[i];
    len[i] = (h + 1 < n_heads ? head_rec[h + 1] : n_rec) - head_rec[h];
  }
}

__global__ void k_run_base(const i64* sorted_heads, const u64* sorted_sample, const i64* run_off, i64 n_heads,
                           i64 n_samples, i64 n_rec, i64* run_base, i64* offsets) {
  pdl_wait();
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n_heads;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    run_base[sorted_heads[i]] = run_off[i];
    if (i == 0 || sorted_sample[i] != sorted_sample[i - 1]) offsets[sorted_sample[i]] = run_off[i];
    if (i == 0) offsets[n_samples] = n_rec;
  }
}

__global__ void k_scatter(const i64* head, const i64* head_idx, const i64* run_base, const i64* head_rec,
                          const i64* rec_line, const double* vals, i64 n_lines, i64 n_rec, int d, double* coords,
                          double* values) {
  pdl_wait();
  for (i64 r = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; r < n_rec;
       r += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 h = head_idx[r] + head[r] - 1;
    const i64 out = run_base[h] + (r - head_rec[h]);
    const i64 L = rec_line[r];
    for (int k = 0; k < d; ++k) coords[out * d + k] = vals[k * n_lines + L];
    values[out] = vals[static_cast<i64>(d) * n_lines + L];
  }
}

__global__ void k_id_lengths(const i64* first_head, const int* h_len, i64 n_samples, i64* len) {
  pdl_wait();
  for (i64 s = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; s < n_samples;
       s += static_cast<i64>(gridDim.x) * blockDim.x)
    len[s] = h_len[first_head[s]];
}

__global__ void k_id_gather(const char* text, const i64* first_head, const i64* h_start, const int* h_len,
                            const i64* id_off, i64 n_samples, char* out) {
  pdl_wait();
  for (i64 s = blockIdx.x; s < n_samples; s += gridDim.x) {
    const i64 h = first_head[s];
    for (int b = threadIdx.x; b < h_len[h]; b += blockDim.x) out[id_off[s] + b] = text[h_start[h] + b];
  }
}

// ------------------------------------------------------------ host helpers --
template <class T>
T d2h_one(dfpca_context* ctx, const T* p) {
  T v{};
  DFPCA_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  return v;
}

void exclusive_sum(dfpca_context* ctx, const i64* in, i64* out, i64 n) {
  std::size_t bytes = 0;
  DFPCA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, ctx->stream));
  DevBuf<unsigned char> tmp(std::max<std::size_t>(bytes, 1));
  DFPCA_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, n, ctx->stream));
}

template <class V>
void sort_pairs(dfpca_context* ctx, DevBuf<u64>& keys, DevBuf<u64>& keys_alt, DevBuf<V>& vals, DevBuf<V>& vals_alt,
                i64 n, int end_bit = 64) {
  std::size_t bytes = 0;
  DFPCA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.get(), keys_alt.get(), vals.get(), vals_alt.get(),
                                             n, 0, end_bit, ctx->stream));
  DevBuf<unsigned char> tmp(std::max<std::size_t>(bytes, 1));
  DFPCA_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, keys.get(), keys_alt.get(), vals.get(), vals_alt.get(),
                                             n, 0, end_bit, ctx->stream));
  std::swap(keys, keys_alt);
  std::swap(vals, vals_alt);
}

bool host_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// The reference's field rule (io.hpp:55-71) on the host (header, messages).
std::vector<std::string> host_split(const std::string& line, char delim) {
  std::vector<std::string> out;
  if (delim == ' ') {
    std::size_t i = 0;
    while (true) {
      while (i < line.size() && host_ws(line[i])) ++i;
      if (i >= line.size()) break;
      const std::size_t a = i;
      while (i < line.size() && !host_ws(line[i])) ++i;
      out.push_back(line.substr(a, i - a));
    }
    return out;
  }
  std::size_t a = 0;
  for (std::size_t i = 0;; ++i) {
    if (i == line.size() || line[i] == delim) {
      out.push_back(line.substr(a, i - a));
      a = i + 1;
      if (i == line.size()) break;
    }
  }
  return out;
}

// Delimiter with the most header fields, earliest candidate on ties (io.hpp:74-86).
char sniff(const std::string& header) {
  char best = '\t';
  std::size_t most = 0;
  for (char c : {'\t', ',', ';', ' '}) {
    const std::size_t n = host_split(header, c).size();
    if (n > most) {
      most = n;
      best = c;
    }
  }
  return best;
}

std::string d2h_string(dfpca_context* ctx, const char* d, i64 a, i64 b) {
  std::string s(static_cast<std::size_t>(std::max<i64>(b - a, 0)), '\0');
  if (b > a) {
    DFPCA_CUDA(cudaMemcpyAsync(s.data(), d + a, s.size(), cudaMemcpyDeviceToHost, ctx->stream));
    DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return s;
}

// Everything after the upload: d_text holds S bytes (+ zero padding to 8).
dfpca_table* parse_table(dfpca_context* ctx, const std::string& name, const char* d_text, i64 S) {
  cudaStream_t st = ctx->stream;
  if (S == 0) fail(kParse, "ParseError", name + ":1: empty file, expected a header row");
  const i64 words = (S + 7) / 8;
  const i64 tiles = (words + kThreads - 1) / kThreads;
  const unsigned cap = static_cast<unsigned>(ctx->sm_count) * 8;
  ctx->begin_stage("lines");
  DevBuf<i64> tcount(static_cast<std::size_t>(tiles) + 1), toff(static_cast<std::size_t>(tiles) + 1);
  DFPCA_CUDA(cudaMemsetAsync(tcount.get() + tiles, 0, sizeof(i64), st));
  const auto* wtext = reinterpret_cast<const u64*>(d_text);
  DFPCA_LAUNCH(ctx, k_nl_count, static_cast<unsigned>(std::min<i64>(tiles, cap)), kThreads, 0, wtext, words,
               tcount.get());
  exclusive_sum(ctx, tcount.get(), toff.get(), tiles + 1);
  const i64 n_nl = d2h_one(ctx, toff.get() + tiles);
  DevBuf<i64> nl(static_cast<std::size_t>(std::max<i64>(n_nl, 1)));
  DFPCA_LAUNCH(ctx, k_nl_write, static_cast<unsigned>(std::min<i64>(tiles, cap)), kThreads, 0, wtext, words,
               toff.get(), nl.get());
  const i64 last_nl = n_nl ? d2h_one(ctx, nl.get() + n_nl - 1) : -1;
  const i64 n_lines = n_nl + (S > last_nl + 1 ? 1 : 0);
  ctx->end_stage();

  // header (io.hpp:118-127)
  std::string header = d2h_string(ctx, d_text, 0, n_nl ? d2h_one(ctx, nl.get()) : S);
  if (!header.empty() && header.back() == '\r') header.pop_back();
  const char delim = sniff(header);
  const int F = static_cast<int>(host_split(header, delim).size());
  if (F < 3) fail(kParse, "ParseError", name + ":1: header needs at least (id, coordinate, value) columns");
  if (F > kMaxFields)
    fail(kConfig, "InvalidArgument", name + ": " + std::to_string(F - 2) + " coordinate columns (at most " +
                                         std::to_string(kMaxFields - 2) + " supported)");
  const int d = F - 2, nv = F - 1;

  ctx->begin_stage("parse");
  const std::size_t NL = static_cast<std::size_t>(std::max<i64>(n_lines, 1));
  DevBuf<i64> is_rec(NL), rec_idx(NL), id_start(NL);
  DevBuf<int> id_len(NL);
  DevBuf<double> vals(NL * static_cast<std::size_t>(nv));
  DevBuf<u64> err(1);
  DFPCA_CUDA(cudaMemsetAsync(err.get(), 0xff, sizeof(u64), st));
  DFPCA_CUDA(cudaMemsetAsync(is_rec.get(), 0, sizeof(i64), st));  // the header line
  Lines ln{d_text, S, nl.get(), n_nl};
  DevBuf<u64> fb(NL * static_cast<std::size_t>(F));
  if (n_lines > 1) {
    const unsigned cap = static_cast<unsigned>(ctx->sm_count) * 16;
    DFPCA_LAUNCH(ctx, k_split_lines, grid_for(n_lines - 1, kThreads, cap), kThreads, 0, ln, n_lines, F,
                 delim == ' ' ? '\0' : delim,
                 SplitOut{is_rec.get(), id_start.get(), id_len.get(), fb.get(), err.get()});
    DFPCA_LAUNCH(ctx, k_parse_fields, grid_for((n_lines - 1) * nv, kThreads, cap), kThreads, 0, ln, n_lines, F,
                 is_rec.get(), fb.get(), vals.get(), err.get());
  }
  const u64 e = d2h_one(ctx, err.get());
  ctx->end_stage();
  if (e != ~0ull) {
    const i64 L = static_cast<i64>(e >> 8);
    const int code = static_cast<int>(e & 0xff);
    const std::string where = name + ":" + std::to_string(L + 1) + ": ";
    if (code == 255) fail(kNumeric, "DeviceError", where + "number parser overflow");
    const i64 a = L == 0 ? 0 : d2h_one(ctx, nl.get() + L - 1) + 1;
    const i64 b = L < n_nl ? d2h_one(ctx, nl.get() + L) : S;
    std::string line = d2h_string(ctx, d_text, a, b);
    if (!line.empty() && line.back() == '\r') line.pop_back();
    const auto fields = host_split(line, delim);
    if (code == 0)
      fail(kParse, "ParseError", where + "expected " + std::to_string(F) + " fields, found " +
                                     std::to_string(fields.size()));
    fail(kParse, "ParseError", where + "not a number: '" + fields[static_cast<std::size_t>(code)] + "'");
  }

  ctx->begin_stage("group");
  exclusive_sum(ctx, is_rec.get(), rec_idx.get(), n_lines);
  const i64 n_rec = d2h_one(ctx, rec_idx.get() + n_lines - 1) + d2h_one(ctx, is_rec.get() + n_lines - 1);
  if (n_rec == 0) fail(kParse, "ParseError", name + ":" + std::to_string(n_lines) + ": no observation rows");
  const std::size_t NR = static_cast<std::size_t>(n_rec);
  DevBuf<i64> rec_line(NR), head(NR), head_idx(NR);
  const unsigned gl = grid_for(n_lines, kThreads), gr = grid_for(n_rec, kThreads);
  DFPCA_LAUNCH(ctx, k_rec_line, gl, kThreads, 0, is_rec.get(), rec_idx.get(), n_lines, rec_line.get());
  DFPCA_LAUNCH(ctx, k_run_heads, gr, kThreads, 0, d_text, rec_line.get(), id_start.get(), id_len.get(), n_rec,
               head.get());
  exclusive_sum(ctx, head.get(), head_idx.get(), n_rec);
  const i64 n_heads = d2h_one(ctx, head_idx.get() + n_rec - 1) + d2h_one(ctx, head.get() + n_rec - 1);
  const std::size_t NH = static_cast<std::size_t>(n_heads);
  DevBuf<i64> head_rec(NH), h_start(NH);
  DevBuf<int> h_len(NH), max_len(1);
  DFPCA_CUDA(cudaMemsetAsync(max_len.get(), 0, sizeof(int), st));
  DFPCA_LAUNCH(ctx, k_head_list, gr, kThreads, 0, head.get(), head_idx.get(), rec_line.get(), id_start.get(),
               id_len.get(), n_rec, head_rec.get(), h_start.get(), h_len.get(), max_len.get());
  const int maxl = d2h_one(ctx, max_len.get());

  // exact grouping of the run heads by id: stable LSD passes (chunks, then length)
  const unsigned gh = grid_for(n_heads, kThreads);
  DevBuf<i64> perm(NH), perm_alt(NH);
  DevBuf<u64> keys(NH), keys_alt(NH);
  DFPCA_LAUNCH(ctx, k_iota, gh, kThreads, 0, perm.get(), n_heads);
  if (n_heads > 1) {
    const int chunks = (maxl + 7) / 8;
    for (int c = chunks - 1; c >= -1; --c) {
      DFPCA_LAUNCH(ctx, k_chunk_keys, gh, kThreads, 0, d_text, h_start.get(), h_len.get(), perm.get(), n_heads, c,
                   keys.get());
      int bits = 64;
      if (c < 0) {
        bits = 1;
        while (bits < 63 && (1ll << bits) <= maxl) ++bits;
      }
      sort_pairs(ctx, keys, keys_alt, perm, perm_alt, n_heads, bits);
    }
  }
  DevBuf<i64> newgrp(NH), first_flag(NH), grp_ex(NH), rank(NH);
  DFPCA_LAUNCH(ctx, k_group_flags, gh, kThreads, 0, d_text, h_start.get(), h_len.get(), perm.get(), n_heads,
               newgrp.get(), first_flag.get());
  exclusive_sum(ctx, newgrp.get(), grp_ex.get(), n_heads);
  exclusive_sum(ctx, first_flag.get(), rank.get(), n_heads);
  const i64 n_samples = d2h_one(ctx, grp_ex.get() + n_heads - 1) + d2h_one(ctx, newgrp.get() + n_heads - 1);
  const std::size_t NS = static_cast<std::size_t>(n_samples);
  DevBuf<i64> sample_of_group(NS), first_head(NS);
  DFPCA_LAUNCH(ctx, k_group_sample, gh, kThreads, 0, perm.get(), newgrp.get(), grp_ex.get(), rank.get(), n_heads,
               sample_of_group.get(), first_head.get());
  DevBuf<u64> hs(NH), hs_alt(NH);
  DFPCA_LAUNCH(ctx, k_head_sample, gh, kThreads, 0, perm.get(), newgrp.get(), grp_ex.get(), sample_of_group.get(),
               n_heads, hs.get());
  // runs sample by sample, head order within a sample
  DFPCA_LAUNCH(ctx, k_iota, gh, kThreads, 0, perm.get(), n_heads);
  if (n_heads > 1) {
    int bits = 1;
    while (bits < 63 && (1ll << bits) <= n_samples) ++bits;
    sort_pairs(ctx, hs, hs_alt, perm, perm_alt, n_heads, bits);
  }
  DevBuf<i64> rlen(NH + 1), roff(NH + 1), run_base(NH);
  DFPCA_LAUNCH(ctx, k_run_lengths, gh, kThreads, 0, perm.get(), head_rec.get(), n_heads, n_rec, rlen.get());
  exclusive_sum(ctx, rlen.get(), roff.get(), n_heads);
  auto tab = std::make_unique<dfpca_table>();
  tab->dim = d;
  tab->n_samples = n_samples;
  tab->n_obs = n_rec;
  tab->offsets.alloc(NS + 1);
  tab->coords.alloc(NR * static_cast<std::size_t>(d));
  tab->values.alloc(NR);
  DFPCA_LAUNCH(ctx, k_run_base, gh, kThreads, 0, perm.get(), hs.get(), roff.get(), n_heads, n_samples, n_rec,
               run_base.get(), tab->offsets.get());
  ctx->end_stage();
  ctx->begin_stage("scatter");
  DFPCA_LAUNCH(ctx, k_scatter, gr, kThreads, 0, head.get(), head_idx.get(), run_base.get(), head_rec.get(),
               rec_line.get(), vals.get(), n_lines, n_rec, d, tab->coords.get(), tab->values.get());
  // sample ids
  DevBuf<i64> ilen(NS + 1);
  tab->id_off.alloc(NS + 1);
  DFPCA_CUDA(cudaMemsetAsync(ilen.get() + n_samples, 0, sizeof(i64), st));
  DFPCA_LAUNCH(ctx, k_id_lengths, grid_for(n_samples, kThreads), kThreads, 0, first_head.get(), h_len.get(),
               n_samples, ilen.get());
  exclusive_sum(ctx, ilen.get(), tab->id_off.get(), n_samples + 1);
  tab->id_bytes = d2h_one(ctx, tab->id_off.get() + n_samples);
  tab->id_chars.alloc(static_cast<std::size_t>(std::max<i64>(tab->id_bytes, 1)));
  DFPCA_LAUNCH(ctx, k_id_gather, grid_for(n_samples, 1, static_cast<i64>(ctx->sm_count) * 8), 64, 0, d_text,
               first_head.get(), h_start.get(), h_len.get(), tab->id_off.get(), n_samples, tab->id_chars.get());
  DFPCA_CUDA(cudaStreamSynchronize(st));
  ctx->end_stage();
  return tab.release();
}

}  // namespace

dfpca_table* read_long_format_file(dfpca_context* ctx, const char* path) {
  const std::string name = path;
  const int fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) fail(kParse, "IoError", "cannot open '" + name + "' for reading");
  struct Closer {
    int fd;
    ~Closer() { ::close(fd); }
  } closer{fd};
  struct stat sb {};
  if (::fstat(fd, &sb) != 0 || !S_ISREG(sb.st_mode)) fail(kParse, "IoError", "cannot open '" + name + "' for reading");
  const i64 S = static_cast<i64>(sb.st_size);
  const std::size_t padded = static_cast<std::size_t>((S + 7) / 8 * 8 + 8);
  DevBuf<char> text(padded);
  DFPCA_CUDA(cudaMemsetAsync(text.get() + (S / 8) * 8, 0, padded - static_cast<std::size_t>(S / 8) * 8, ctx->stream));
  DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));  // the worker streams write after the padding memset
  ctx->begin_stage("upload");
  upload_bytes(ctx, text.get(), S, [&](char* dst, i64 off, i64 len) -> std::string {
    i64 done = 0;
    while (done < len) {
      const ssize_t r = ::pread(fd, dst + done, static_cast<std::size_t>(len - done), static_cast<off_t>(off + done));
      if (r < 0 && errno == EINTR) continue;
      if (r <= 0) return "failed reading '" + name + "'";
      done += r;
    }
    return {};
  });
  ctx->end_stage();
  return parse_table(ctx, name, text.get(), S);
}

dfpca_table* parse_long_format_bytes(dfpca_context* ctx, const char* name, const char* bytes, i64 S) {
  const std::size_t padded = static_cast<std::size_t>((S + 7) / 8 * 8 + 8);
  DevBuf<char> text(padded);
  DFPCA_CUDA(cudaMemsetAsync(text.get() + (S / 8) * 8, 0, padded - static_cast<std::size_t>(S / 8) * 8, ctx->stream));
  DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->begin_stage("upload");
  upload_bytes(ctx, text.get(), S, [&](char* dst, i64 off, i64 len) -> std::string {
    std::memcpy(dst, bytes + off, static_cast<std::size_t>(len));
    return {};
  });
  ctx->end_stage();
  return parse_table(ctx, name ? name : "<memory>", text.get(), S);
}

void table_copy(dfpca_context* ctx, const dfpca_table* t, i64* offsets, double* coords, double* values, i64* id_off,
                char* id_chars) {
  cudaStream_t st = ctx->stream;
  if (offsets)
    DFPCA_CUDA(cudaMemcpyAsync(offsets, t->offsets.get(), sizeof(i64) * static_cast<std::size_t>(t->n_samples + 1),
                               cudaMemcpyDeviceToHost, st));
  if (coords && t->n_obs)
    download_bytes(ctx, reinterpret_cast<char*>(coords), reinterpret_cast<const char*>(t->coords.get()),
                   static_cast<i64>(sizeof(double)) * t->n_obs * t->dim);
  if (values && t->n_obs)
    download_bytes(ctx, reinterpret_cast<char*>(values), reinterpret_cast<const char*>(t->values.get()),
                   static_cast<i64>(sizeof(double)) * t->n_obs);
  if (id_off)
    DFPCA_CUDA(cudaMemcpyAsync(id_off, t->id_off.get(), sizeof(i64) * static_cast<std::size_t>(t->n_samples + 1),
                               cudaMemcpyDeviceToHost, st));
  if (id_chars && t->id_bytes)
    DFPCA_CUDA(cudaMemcpyAsync(id_chars, t->id_chars.get(), static_cast<std::size_t>(t->id_bytes),
                               cudaMemcpyDeviceToHost, st));
  DFPCA_CUDA(cudaStreamSynchronize(st));
}

void table_shape(const dfpca_table* t, int* dim, i64* n_samples, i64* n_obs, i64* id_bytes) {
  if (dim) *dim = t->dim;
  if (n_samples) *n_samples = t->n_samples;
  if (n_obs) *n_obs = t->n_obs;
  if (id_bytes) *id_bytes = t->id_bytes;
}

void table_delete(dfpca_table* t) { delete t; }

dfpca_binned* run_linear_bin(dfpca_context* ctx, const Grid& grid, i64 n_samples, const i64* obs_offsets,
                             const double* coords, const double* values, bool mean_path, bool cov_path,
                             bool device_inputs);

// linear_bin over a table that is already on the device: only the sample
// offsets come back to the host (the binning plans its chunks with them).
dfpca_binned* bin_table(dfpca_context* ctx, const dfpca_table* t, const Grid& grid, bool mean_path, bool cov_path) {
  if (t->dim != grid.d) fail(kConfig, "InvalidArgument", "dataset/grid dimension mismatch");
  std::vector<i64> off(static_cast<std::size_t>(t->n_samples) + 1);
  DFPCA_CUDA(cudaMemcpyAsync(off.data(), t->offsets.get(), sizeof(i64) * off.size(), cudaMemcpyDeviceToHost,
                             ctx->stream));
  DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  return run_linear_bin(ctx, grid, t->n_samples, off.data(), t->coords.get(), t->values.get(), mean_path, cov_path,
                        true);
}

}  // namespace dfpca_gpu

