// Execution hooks of a sharded covariance (shard.hpp) seen by the smoother
// (smooth.cu): the slab plan, this rank, and the two exchanges, bound to a
// transport (NCCL across processes, or in-process ranks for validation) by
// shard.cu.
#pragma once

#include <functional>
#include <vector>

#include "internal.hpp"
#include "shard.hpp"

namespace dfpca_gpu {

// Rank-to-rank transport of a sharded run (shard.cu: NCCL or in-process).
class Transport {
 public:
  struct Msg {
    int peer;
    double* buf;
    i64 count;
  };
  virtual ~Transport() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  // all sends and receives of one phase, queued on ctx->stream
  virtual void exchange(dfpca_context* ctx, const std::vector<Msg>& sends, const std::vector<Msg>& recvs) = 0;
  virtual unsigned long long max_u64(dfpca_context* ctx, unsigned long long v) = 0;
  // recv[r * count ..] = rank r's send, for every rank
  virtual void all_gather(dfpca_context* ctx, const double* send, double* recv, i64 count) = 0;
};

struct CovShardExec {
  const ShardPlan* plan = nullptr;
  int rank = 0;
  // exchange 1: completes this rank's pair-grid window (pv, and pw when
  // with_pw: pw came from the SYRK too); every rank makes the same calls
  std::function<void(double* pw, double* pv, bool with_pw)> exchange_pairs;
  // exchange 2: completes the rows of this rank's covariance slab
  std::function<void(double* slab)> exchange_cov;
  // host-side agreement (the maximum over ranks)
  std::function<unsigned long long(unsigned long long)> max_over_ranks;
};

void run_covariance_impl(dfpca_context* ctx, const dfpca_binned* b, const Grid& grid, const double* h,
                         const double* mean_host, const CovShardExec* shard, dfpca_surface** out);

}  // namespace dfpca_gpu
