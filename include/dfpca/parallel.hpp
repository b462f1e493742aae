// Drop-in thread-count knob and chunked parallel loop (API of the reference's
// parallel.hpp).  The hot path runs on the device; parallel_for serves the
// host-side code of the reference that keeps running against these headers
// (direct smoothers, bandwidth search, pipeline helpers).  Chunk boundaries
// depend only on n and chunk, every chunk writes disjoint state, so results
// never depend on the thread count (the reference's contract).
#pragma once

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace dfpca {
namespace detail {
inline int& max_threads_ref() {
  static int n = 1;
  return n;
}
}  // namespace detail

inline void set_max_threads(int n) { detail::max_threads_ref() = std::max(1, n); }
inline int max_threads() { return detail::max_threads_ref(); }

/// fn(begin, end) over [0, n) in chunks of `chunk`, on up to max_threads()
/// threads.  If chunks throw, the exception of the lowest-numbered failing
/// chunk is rethrown after every worker has stopped.
inline void parallel_for(std::size_t n, std::size_t chunk, const std::function<void(std::size_t, std::size_t)>& fn) {
  if (n == 0) return;
  chunk = std::max<std::size_t>(1, chunk);
  const std::size_t chunks = (n + chunk - 1) / chunk;
  const std::size_t threads = std::min<std::size_t>(chunks, static_cast<std::size_t>(max_threads()));
  auto run_chunk = [&](std::size_t c) { fn(c * chunk, std::min(n, c * chunk + chunk)); };
  if (threads <= 1) {
    for (std::size_t c = 0; c < chunks; ++c) run_chunk(c);
    return;
  }
  std::atomic<std::size_t> cursor{0};
  std::atomic<bool> failed{false};
  std::mutex mu;
  std::size_t failed_chunk = chunks;
  std::exception_ptr failure;
  auto worker = [&] {
    for (std::size_t c; !failed.load(std::memory_order_relaxed) && (c = cursor.fetch_add(1)) < chunks;) {
      try {
        run_chunk(c);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (c < failed_chunk) {
          failed_chunk = c;
          failure = std::current_exception();
        }
        failed.store(true, std::memory_order_relaxed);
      }
    }
  };
  std::vector<std::thread> pool;
  pool.reserve(threads - 1);
  for (std::size_t t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  if (failure) std::rethrow_exception(failure);
}

}  // namespace dfpca
