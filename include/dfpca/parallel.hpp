// Drop-in thread-count knob (API of the reference's parallel.hpp).  The GPU
// build runs the hot path on the device, so the value only caps host-side
// helper loops; results never depend on it (the reference's contract).
#pragma once

#include <algorithm>
#include <cstddef>
#include <functional>

namespace dfpca {
namespace detail {
inline int& max_threads_ref() {
  static int n = 1;
  return n;
}
}  // namespace detail

inline void set_max_threads(int n) { detail::max_threads_ref() = std::max(1, n); }
inline int max_threads() { return detail::max_threads_ref(); }

// Sequential chunked loop with the reference's chunk boundaries.
inline void parallel_for(std::size_t n, std::size_t chunk, const std::function<void(std::size_t, std::size_t)>& fn) {
  chunk = std::max<std::size_t>(1, chunk);
  for (std::size_t b = 0; b < n; b += chunk) fn(b, std::min(n, b + chunk));
}

}  // namespace dfpca
