// Sharded covariance: block exchanges over a transport and the drivers.
//
//  * NcclTransport: one process per GPU; libnccl is loaded at run time
//    (dlopen), the communicator is created from a unique id the caller
//    broadcasts (dfpca_nccl_unique_id / dfpca_nccl_init).  Exchanges are one
//    grouped ncclSend/ncclRecv per phase on the context stream.
//  * LocalTransport: `world` ranks as host threads of one process, each with
//    its own context and stream on the same device; messages are
//    device-to-device copies ordered by events.  Used to validate the slab
//    decomposition on one GPU (the assembled result must be bit-identical to
//    the one-device covariance); no kernel ever waits on another rank's kernel
//    -- ranks meet only at host-side barriers between exchanges.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>

#include "common.cuh"
#include "shard.hpp"
#include "shard_exec.hpp"

namespace dfpca_gpu {

// ----------------------------------------------------------------- kernels --
// One exchange block as the batched kernels see it: rows [r0, r1), columns
// [c0, c1) (global), transpose flag, its offset in the packed buffer, and the
// first tile / row of the launch that belongs to it.
struct PackDesc {
  i64 r0, r1, c0, c1;
  i64 off;    // packed offset (elements)
  i64 first;  // first tile (pack) or row (unpack) of this block in the launch
  int transpose;
};

__device__ inline int find_block(const PackDesc* __restrict__ d, int n, i64 x) {
  int lo = 0, hi = n - 1;  // last block with first <= x
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (d[mid].first <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// packed[off + (s - r0) * w + (t - c0)] = value (s, t) of each block, read
// from a row-major buffer whose row 0 is global row row0 (ld = G): element
// [s][t], or [t][s] for a transposed block (32 x 32 shared-memory tiles keep
// both sides coalesced).  One launch packs every block of a phase.
__global__ void k_pack_blocks(const double* __restrict__ src, i64 ld, i64 row0, const PackDesc* __restrict__ desc,
                              int n_desc, double* __restrict__ packed) {
  pdl_wait();
  __shared__ double tile[32][33];
  const PackDesc b = desc[find_block(desc, n_desc, blockIdx.x)];
  const i64 w = b.c1 - b.c0, h = b.r1 - b.r0;
  const i64 tw = (w + 31) / 32;
  const i64 t_local = blockIdx.x - b.first;
  const i64 bs = (t_local / tw) * 32, bt = (t_local % tw) * 32;  // tile origin (s, t), block-relative
  double* out = packed + b.off;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  if (!b.transpose) {
    for (int r = ty; r < 32; r += 8) {
      const i64 s = bs + r, t = bt + tx;
      if (s < h && t < w) out[s * w + t] = src[(b.r0 + s - row0) * ld + b.c0 + t];
    }
    return;
  }
  for (int r = ty; r < 32; r += 8) {  // rows t of the source, columns s
    const i64 t = bt + r, s = bs + tx;
    tile[r][tx] = (s < h && t < w) ? src[(b.c0 + t - row0) * ld + b.r0 + s] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const i64 s = bs + r, t = bt + tx;
    if (s < h && t < w) out[s * w + t] = tile[tx][r];
  }
}

// dst[(s - row0) * ld + t] = packed block rows; one CTA per block row, threads
// across the columns (coalesced on both sides).
__global__ void k_unpack_blocks(const double* __restrict__ packed, double* __restrict__ dst, i64 ld, i64 row0,
                                const PackDesc* __restrict__ desc, int n_desc) {
  pdl_wait();
  const PackDesc b = desc[find_block(desc, n_desc, blockIdx.x)];
  const i64 w = b.c1 - b.c0;
  const i64 s = blockIdx.x - b.first;
  const double* in = packed + b.off + s * w;
  double* out = dst + (b.r0 + s - row0) * ld + b.c0;
  for (i64 t = threadIdx.x; t < w; t += blockDim.x) out[t] = in[t];
}

namespace {

// ---- NCCL, loaded at run time ----
struct NcclApi {
  using Comm = void*;
  struct UniqueId {
    char internal[128];
  };
  int (*GetUniqueId)(UniqueId*) = nullptr;
  int (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*Send)(const void*, std::size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*Recv)(void*, std::size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, std::size_t, int, Comm, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, std::size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  static constexpr int kUint64 = 5, kFloat64 = 8, kMax = 2;

  static NcclApi& get() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] { api.load(); });
    if (!api.GetUniqueId) fail(kConfig, "InvalidArgument", "libnccl.so.2 could not be loaded (set DFPCA_NCCL_LIB)");
    return api;
  }
  void load() {
    std::vector<std::string> names;
    if (const char* e = std::getenv("DFPCA_NCCL_LIB")) names.push_back(e);
    names.push_back("libnccl.so.2");
    void* h = nullptr;
    for (const auto& n : names)
      if ((h = dlopen(n.c_str(), RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return;
    auto sym = [h](const char* s) { return dlsym(h, s); };
    GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(sym("ncclGetUniqueId"));
    CommInitRank = reinterpret_cast<decltype(CommInitRank)>(sym("ncclCommInitRank"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
    Send = reinterpret_cast<decltype(Send)>(sym("ncclSend"));
    Recv = reinterpret_cast<decltype(Recv)>(sym("ncclRecv"));
    AllGather = reinterpret_cast<decltype(AllGather)>(sym("ncclAllGather"));
    AllReduce = reinterpret_cast<decltype(AllReduce)>(sym("ncclAllReduce"));
    GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
    GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
    if (!(CommInitRank && Send && Recv && AllGather && AllReduce && GroupStart && GroupEnd)) GetUniqueId = nullptr;
  }
  void check(int r, const char* what) const {
    if (r != 0)
      fail(kNumeric, "DeviceError",
           std::string(what) + ": " + (GetErrorString ? GetErrorString(r) : std::to_string(r)));
  }
};

}  // namespace

class NcclTransport final : public Transport {
 public:
  NcclTransport(int world, int rank, const void* id) : world_(world), rank_(rank) {
    NcclApi& api = NcclApi::get();
    NcclApi::UniqueId uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    api.check(api.CommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclTransport() override {
    if (comm_) NcclApi::get().CommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  void exchange(dfpca_context* ctx, const std::vector<Msg>& sends, const std::vector<Msg>& recvs) override {
    NcclApi& api = NcclApi::get();
    api.check(api.GroupStart(), "ncclGroupStart");
    for (const Msg& m : sends)
      api.check(api.Send(m.buf, static_cast<std::size_t>(m.count), NcclApi::kFloat64, m.peer, comm_, ctx->stream),
                "ncclSend");
    for (const Msg& m : recvs)
      api.check(api.Recv(m.buf, static_cast<std::size_t>(m.count), NcclApi::kFloat64, m.peer, comm_, ctx->stream),
                "ncclRecv");
    api.check(api.GroupEnd(), "ncclGroupEnd");
  }
  unsigned long long max_u64(dfpca_context* ctx, unsigned long long v) override {
    NcclApi& api = NcclApi::get();
    DevBuf<unsigned long long> d(1);
    DFPCA_CUDA(cudaMemcpyAsync(d.get(), &v, sizeof(v), cudaMemcpyHostToDevice, ctx->stream));
    api.check(api.AllReduce(d.get(), d.get(), 1, NcclApi::kUint64, NcclApi::kMax, comm_, ctx->stream),
              "ncclAllReduce");
    unsigned long long out = 0;
    DFPCA_CUDA(cudaMemcpyAsync(&out, d.get(), sizeof(out), cudaMemcpyDeviceToHost, ctx->stream));
    DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
    return out;
  }
  void all_gather(dfpca_context* ctx, const double* send, double* recv, i64 count) override {
    NcclApi& api = NcclApi::get();
    api.check(api.AllGather(send, recv, static_cast<std::size_t>(count), NcclApi::kFloat64, comm_, ctx->stream),
              "ncclAllGather");
  }

 private:
  int world_, rank_;
  NcclApi::Comm comm_ = nullptr;
};

// ---- in-process ranks ----
class LocalHub {
 public:
  explicit LocalHub(int world) : world_(world) {}
  struct Posted {
    const double* buf;
    i64 count;
    cudaEvent_t ready;
  };
  void post(int src, int dst, int seq, const Posted& p) {
    std::lock_guard<std::mutex> lk(m_);
    box_[{src, dst, seq}] = p;
    cv_.notify_all();
  }
  Posted take(int src, int dst, int seq) {
    std::unique_lock<std::mutex> lk(m_);
    cv_.wait(lk, [&] { return abort_ || box_.count({src, dst, seq}) > 0; });
    if (abort_) fail(kNumeric, "DeviceError", "another in-process rank failed");
    return box_.at({src, dst, seq});
  }
  // all ranks arrive; the last one clears the messages of round `seq`
  void barrier(int seq) {
    std::unique_lock<std::mutex> lk(m_);
    const int gen = gen_;
    if (++arrived_ == world_) {
      arrived_ = 0;
      ++gen_;
      for (auto it = box_.begin(); it != box_.end();) {
        if (std::get<2>(it->first) == seq) {
          cudaEventDestroy(it->second.ready);
          it = box_.erase(it);
        } else {
          ++it;
        }
      }
      cv_.notify_all();
      return;
    }
    cv_.wait(lk, [&] { return abort_ || gen_ != gen; });
    if (abort_) fail(kNumeric, "DeviceError", "another in-process rank failed");
  }
  void set_abort() {
    std::lock_guard<std::mutex> lk(m_);
    abort_ = true;
    cv_.notify_all();
  }
  int world() const { return world_; }
  // scratch for the u64 reduction
  std::vector<unsigned long long> u64s;

 private:
  int world_;
  std::mutex m_;
  std::condition_variable cv_;
  std::map<std::tuple<int, int, int>, Posted> box_;
  int arrived_ = 0, gen_ = 0;
  bool abort_ = false;
};

class LocalTransport final : public Transport {
 public:
  LocalTransport(LocalHub* hub, int rank) : hub_(hub), rank_(rank) {}
  int rank() const override { return rank_; }
  int world() const override { return hub_->world(); }
  void exchange(dfpca_context* ctx, const std::vector<Msg>& sends, const std::vector<Msg>& recvs) override {
    const int seq = seq_++;
    for (const Msg& m : sends) {
      cudaEvent_t ev;
      DFPCA_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      DFPCA_CUDA(cudaEventRecord(ev, ctx->stream));
      hub_->post(rank_, m.peer, seq, {m.buf, m.count, ev});
    }
    for (const Msg& m : recvs) {
      const LocalHub::Posted p = hub_->take(m.peer, rank_, seq);
      if (p.count != m.count) fail(kNumeric, "DeviceError", "in-process exchange: message size mismatch");
      DFPCA_CUDA(cudaStreamWaitEvent(ctx->stream, p.ready, 0));
      DFPCA_CUDA(cudaMemcpyAsync(m.buf, p.buf, sizeof(double) * m.count, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    // senders keep their buffers until every receiver has copied
    DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
    hub_->barrier(seq);
  }
  unsigned long long max_u64(dfpca_context* ctx, unsigned long long v) override {
    (void)ctx;
    const int seq = seq_++;
    {
      static std::mutex mu;
      std::lock_guard<std::mutex> lk(mu);
      if (hub_->u64s.size() != static_cast<std::size_t>(world())) hub_->u64s.assign(world(), 0);
      hub_->u64s[rank_] = v;
    }
    hub_->barrier(seq);
    unsigned long long m = 0;
    for (auto x : hub_->u64s) m = x > m ? x : m;
    hub_->barrier(seq_++);
    return m;
  }
  void all_gather(dfpca_context* ctx, const double* send, double* recv, i64 count) override {
    std::vector<Msg> sends, recvs;
    for (int r = 0; r < world(); ++r) {
      if (r == rank_) continue;
      sends.push_back({r, const_cast<double*>(send), count});
      recvs.push_back({r, recv + r * count, count});
    }
    DFPCA_CUDA(cudaMemcpyAsync(recv + rank_ * count, send, sizeof(double) * count, cudaMemcpyDeviceToDevice,
                               ctx->stream));
    exchange(ctx, sends, recvs);
  }

 private:
  LocalHub* hub_;
  int rank_;
  int seq_ = 0;
};

// One rank of `world` with the exchanges dropped: times a rank's slab alone
// (the received regions hold whatever the buffers held -- timing only).
class NullTransport final : public Transport {
 public:
  NullTransport(int world, int rank) : world_(world), rank_(rank) {}
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  // what would arrive is not computed here: zeros stand in for it (left
  // uninitialised, NaN bit patterns in the pool sent those nodes through the
  // solve's exact pass and inflated the projected time)
  void exchange(dfpca_context* ctx, const std::vector<Msg>&, const std::vector<Msg>& recv) override {
    for (const Msg& m : recv)
      if (m.count > 0) DFPCA_CUDA(cudaMemsetAsync(m.buf, 0, sizeof(double) * m.count, ctx->stream));
  }
  unsigned long long max_u64(dfpca_context*, unsigned long long v) override { return v; }
  void all_gather(dfpca_context* ctx, const double* send, double* recv, i64 count) override {
    DFPCA_CUDA(cudaMemcpyAsync(recv + rank_ * count, send, sizeof(double) * count, cudaMemcpyDeviceToDevice,
                               ctx->stream));
  }

 private:
  int world_, rank_;
};

// ------------------------------------------------------------------ exchange --
// Runs one phase of the schedule (shard_blocks) for this rank over `buf`
// (row-major, leading dimension G, row 0 = global row buf_row0).
void run_shard_exchange(dfpca_context* ctx, Transport& tr, const ShardPlan& plan, int phase, double* buf,
                        i64 buf_row0) {
  const int me = tr.rank();
  const i64 G = plan.G;
  const std::vector<ShardBlock> blocks = shard_blocks(plan, phase);
  std::map<int, i64> send_n, recv_n;
  std::vector<ShardBlock> sends, recvs, locals;
  for (const ShardBlock& b : blocks) {
    if (b.src == me && b.dst == me) {
      if (b.transpose) locals.push_back(b);  // direct own rows are already in place
      continue;
    }
    if (b.src == me) {
      sends.push_back(b);
      send_n[b.dst] += b.elems();
    }
    if (b.dst == me) {
      recvs.push_back(b);
      recv_n[b.src] += b.elems();
    }
  }
  i64 n_send = 0, n_recv = 0, n_local = 0;
  for (auto& kv : send_n) n_send += kv.second;
  for (auto& kv : recv_n) n_recv += kv.second;
  for (auto& b : locals) n_local += b.elems();
  DevBuf<double> sbuf(static_cast<std::size_t>(std::max<i64>(1, n_send + n_local)));
  DevBuf<double> rbuf(static_cast<std::size_t>(std::max<i64>(1, n_recv)));
  // message offsets: peers ascending, blocks in schedule order (both sides agree)
  std::map<int, i64> soff, roff;
  {
    i64 o = 0;
    for (auto& kv : send_n) {
      soff[kv.first] = o;
      o += kv.second;
    }
    o = 0;
    for (auto& kv : recv_n) {
      roff[kv.first] = o;
      o += kv.second;
    }
  }
  // one pack launch for every outgoing and local block, in buffer order
  std::vector<PackDesc> pk, up_r, up_l;
  i64 tiles = 0;
  auto add_pack = [&](const ShardBlock& b, i64 off) {
    if (b.elems() <= 0) return;
    pk.push_back({b.r0, b.r1, b.c0, b.c1, off, tiles, b.transpose ? 1 : 0});
    tiles += ((b.r1 - b.r0 + 31) / 32) * ((b.c1 - b.c0 + 31) / 32);
  };
  {
    std::map<int, i64> cur = soff;
    for (const ShardBlock& b : sends) {
      add_pack(b, cur[b.dst]);
      cur[b.dst] += b.elems();
    }
  }
  i64 lo = n_send;
  for (const ShardBlock& b : locals) {
    add_pack(b, lo);
    lo += b.elems();
  }
  auto launch_pack = [&](const std::vector<PackDesc>& d, i64 n_tiles) {
    if (d.empty()) return;
    DevBuf<PackDesc> dd(d.size());
    DFPCA_CUDA(cudaMemcpyAsync(dd.get(), d.data(), sizeof(PackDesc) * d.size(), cudaMemcpyHostToDevice, ctx->stream));
    DFPCA_LAUNCH(ctx, k_pack_blocks, static_cast<unsigned>(n_tiles), 256, 0, buf, G, buf_row0, dd.get(),
                 static_cast<int>(d.size()), sbuf.get());
  };
  auto launch_unpack = [&](const std::vector<PackDesc>& d, i64 n_rows, const double* packed) {
    if (d.empty()) return;
    DevBuf<PackDesc> dd(d.size());
    DFPCA_CUDA(cudaMemcpyAsync(dd.get(), d.data(), sizeof(PackDesc) * d.size(), cudaMemcpyHostToDevice, ctx->stream));
    DFPCA_LAUNCH(ctx, k_unpack_blocks, static_cast<unsigned>(n_rows), 256, 0, packed, buf, G, buf_row0, dd.get(),
                 static_cast<int>(d.size()));
  };
  launch_pack(pk, tiles);
  std::vector<Transport::Msg> smsg, rmsg;
  for (auto& kv : send_n) smsg.push_back({kv.first, sbuf.get() + soff[kv.first], kv.second});
  for (auto& kv : recv_n) rmsg.push_back({kv.first, rbuf.get() + roff[kv.first], kv.second});
  tr.exchange(ctx, smsg, rmsg);
  {
    std::map<int, i64> cur = roff;
    i64 rows = 0;
    for (const ShardBlock& b : recvs) {
      if (b.elems() > 0) {
        up_r.push_back({b.r0, b.r1, b.c0, b.c1, cur[b.src], rows, 0});
        rows += b.r1 - b.r0;
      }
      cur[b.src] += b.elems();
    }
    launch_unpack(up_r, rows, rbuf.get());
  }
  {
    i64 off = n_send, rows = 0;
    for (const ShardBlock& b : locals) {
      if (b.elems() > 0) {
        up_l.push_back({b.r0, b.r1, b.c0, b.c1, off, rows, 0});
        rows += b.r1 - b.r0;
      }
      off += b.elems();
    }
    launch_unpack(up_l, rows, sbuf.get());
  }
}

i64 s1_radius(const Grid& grid, const double* h) {
  return static_cast<i64>(std::ceil(h[0] / grid.spacing[0]));  // make_taps (smooth.cu) on axis s1
}

ShardPlan plan_for(const Grid& grid, const double* h, int world) {
  return make_shard_plan(grid.shape[0], grid.G / grid.shape[0], s1_radius(grid, h), world);
}

void run_covariance_sharded(dfpca_context* ctx, Transport& tr, const dfpca_binned* b, const Grid& grid,
                            const double* h, const double* mean_host, dfpca_surface** out) {
  const ShardPlan plan = plan_for(grid, h, tr.world());
  CovShardExec ex;
  ex.plan = &plan;
  ex.rank = tr.rank();
  const i64 rn = plan.rn;
  ex.exchange_pairs = [&](double* pw, double* pv, bool with_pw) {
    ctx->begin_stage("exchange");
    const i64 row0 = plan.ha(tr.rank()) * rn;
    // an idle rank (empty slab) still takes part, with empty buffers
    run_shard_exchange(ctx, tr, plan, 0, pv, row0);
    if (with_pw) run_shard_exchange(ctx, tr, plan, 0, pw, row0);
    ctx->end_stage();
  };
  ex.exchange_cov = [&](double* slab) { run_shard_exchange(ctx, tr, plan, 1, slab, plan.a(tr.rank()) * rn); };
  ex.max_over_ranks = [&](unsigned long long v) { return tr.max_u64(ctx, v); };
  run_covariance_impl(ctx, b, grid, h, mean_host, &ex, out);
}

}  // namespace dfpca_gpu
namespace dfpca_gpu {
void run_randomized_eig(dfpca_context* ctx, const dfpca_surface* cov, const Grid& grid, i64 q, i64 L_max,
                        unsigned long long seed, double* eigenvalues, double* eigenfunctions, double* fve,
                        double* total_variance, i64* n_components);

// Eigen outputs of one in-process rank.
struct EigOut {
  i64 q = 0, L = 0;
  unsigned long long seed = 0;
  std::vector<double> values, functions, fve;
  double total = 0.0;
  i64 n = 0;
};

// `world` in-process ranks on ctx's device; the slabs are assembled into one
// G x G surface on ctx (validation of the decomposition).  With `eig`, every
// rank then runs the row-sharded randomized eigensolver on its slab and
// eig[r] receives rank r's (replicated) eigensystem.
void run_covariance_emulated(dfpca_context* ctx, int world, const dfpca_binned* b, const Grid& grid,
                             const double* h, const double* mean_host, dfpca_surface** out,
                             std::vector<EigOut>* eig) {
  LocalHub hub(world);
  std::vector<dfpca_surface*> slabs(static_cast<std::size_t>(world), nullptr);
  std::vector<dfpca_context*> rctx(static_cast<std::size_t>(world), nullptr);
  std::vector<Failure> errs(static_cast<std::size_t>(world));
  std::vector<int> failed(static_cast<std::size_t>(world), 0);
  DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<std::thread> threads;
  for (int r = 0; r < world; ++r) {
    threads.emplace_back([&, r] {
      dfpca_context* c = nullptr;
      try {
        if (dfpca_context_create(ctx->device, &c) != 0) fail(kNumeric, "DeviceError", "rank context creation failed");
        rctx[static_cast<std::size_t>(r)] = c;
        DFPCA_CUDA(cudaSetDevice(ctx->device));
        g_alloc_stream = c->stream;
        auto tr = std::make_shared<LocalTransport>(&hub, r);
        c->transport = tr;
        run_covariance_sharded(c, *tr, b, grid, h, mean_host, &slabs[static_cast<std::size_t>(r)]);
        if (eig) {
          EigOut& e = (*eig)[static_cast<std::size_t>(r)];
          e.values.assign(static_cast<std::size_t>(e.L), 0.0);
          e.fve.assign(static_cast<std::size_t>(e.L), 0.0);
          e.functions.assign(static_cast<std::size_t>(e.L * grid.G), 0.0);
          run_randomized_eig(c, slabs[static_cast<std::size_t>(r)], grid, e.q, e.L, e.seed, e.values.data(),
                             e.functions.data(), e.fve.data(), &e.total, &e.n);
        }
        DFPCA_CUDA(cudaStreamSynchronize(c->stream));
        c->collect_stages();
      } catch (const Failure& e) {
        errs[static_cast<std::size_t>(r)] = e;
        failed[static_cast<std::size_t>(r)] = 1;
        hub.set_abort();
      } catch (const std::exception& e) {
        errs[static_cast<std::size_t>(r)] = Failure{kNumeric, "DeviceError", e.what(), -1, -1};
        failed[static_cast<std::size_t>(r)] = 1;
        hub.set_abort();
      }
      if (c) cudaStreamSynchronize(c->stream);
      g_alloc_stream = nullptr;
    });
  }
  for (auto& t : threads) t.join();
  int first = -1;
  for (int r = 0; r < world; ++r)
    if (failed[static_cast<std::size_t>(r)] && (first < 0 || errs[static_cast<std::size_t>(r)].name != "DeviceError"))
      first = r;
  std::unique_ptr<dfpca_surface> full;
  if (first < 0) {
    full = std::make_unique<dfpca_surface>();
    full->grid = grid;
    full->kind = DFPCA_SURFACE_COVARIANCE;
    full->n = grid.G * grid.G;
    full->rows = grid.G;
    full->values.alloc(static_cast<std::size_t>(full->n));
    for (int r = 0; r < world; ++r) {
      const dfpca_surface* s = slabs[static_cast<std::size_t>(r)];
      if (s && s->n > 0)
        DFPCA_CUDA(cudaMemcpyAsync(full->values.get() + s->row0 * grid.G, s->values.get(), sizeof(double) * s->n,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
    }
    DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  for (int r = 0; r < world; ++r) {
    delete slabs[static_cast<std::size_t>(r)];
    if (rctx[static_cast<std::size_t>(r)]) dfpca_context_destroy(rctx[static_cast<std::size_t>(r)]);
  }
  if (first >= 0) throw errs[static_cast<std::size_t>(first)];
  *out = full.release();
}

void run_covariance_dryrun(dfpca_context* ctx, int world, int rank, const dfpca_binned* b, const Grid& grid,
                           const double* h, const double* mean_host, dfpca_surface** out) {
  NullTransport tr(world, rank);
  run_covariance_sharded(ctx, tr, b, grid, h, mean_host, out);
}

void nccl_unique_id(void* out) {
  NcclApi& api = NcclApi::get();
  NcclApi::UniqueId id;
  api.check(api.GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, sizeof(id.internal));
}

std::shared_ptr<Transport> make_nccl_transport(int world, int rank, const void* id) {
  return std::make_shared<NcclTransport>(world, rank, id);
}

// One-rank NCCL communicator driving the same transport calls as a sharded
// run (grouped send/recv to itself, all-gather, max all-reduce) on the
// context stream: checks the run-time binding of libnccl on a one-GPU box.
// Returns the number of mismatching elements (0 = pass).
i64 nccl_selftest(dfpca_context* ctx) {
  NcclApi::UniqueId id;
  NcclApi& api = NcclApi::get();
  api.check(api.GetUniqueId(&id), "ncclGetUniqueId");
  NcclTransport tr(1, 0, id.internal);
  const i64 n = 1 << 16;
  std::vector<double> h(static_cast<std::size_t>(n));
  for (i64 i = 0; i < n; ++i) h[static_cast<std::size_t>(i)] = 0.5 * static_cast<double>(i) - 7.0;
  DevBuf<double> a(n), b(n), c(n);
  DFPCA_CUDA(cudaMemcpyAsync(a.get(), h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  DFPCA_CUDA(cudaMemsetAsync(b.get(), 0, sizeof(double) * n, ctx->stream));
  DFPCA_CUDA(cudaMemsetAsync(c.get(), 0, sizeof(double) * n, ctx->stream));
  tr.exchange(ctx, {Transport::Msg{0, a.get(), n}}, {Transport::Msg{0, b.get(), n}});
  tr.all_gather(ctx, b.get(), c.get(), n);
  const unsigned long long m = tr.max_u64(ctx, 12345ull);
  std::vector<double> hb(static_cast<std::size_t>(n)), hc(static_cast<std::size_t>(n));
  DFPCA_CUDA(cudaMemcpyAsync(hb.data(), b.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  DFPCA_CUDA(cudaMemcpyAsync(hc.data(), c.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  DFPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  i64 bad = m == 12345ull ? 0 : 1;
  for (i64 i = 0; i < n; ++i)
    bad += (hb[static_cast<std::size_t>(i)] != h[static_cast<std::size_t>(i)]) +
           (hc[static_cast<std::size_t>(i)] != h[static_cast<std::size_t>(i)]);
  return bad;
}

}  // namespace dfpca_gpu
