// launch_count.h -- how many kernels this library has launched (fsmc_launch_count):
// bench.py reads it around its timed region to report its own launches.
#pragma once
#include <atomic>

namespace fsmc {
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> c{0};
  return c;
}
inline void count_launch(long long k = 1) { launch_counter().fetch_add(k, std::memory_order_relaxed); }
}  // namespace fsmc
