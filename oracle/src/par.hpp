// ORACLE (test infrastructure only) — tiny deterministic parallel-for over fixed chunks.
// Results never depend on the worker count: every reduction done under it is an
// order-independent min or a per-index write.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <thread>
#include <vector>

namespace orc {

int& worker_count_ref();
inline int worker_count() {
  int n = worker_count_ref();
  if (n <= 0) n = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  return n;
}

template <class F>
void parallel_for(int64_t n, F&& body, int64_t grain = 256) {
  const int w = worker_count();
  if (w <= 1 || n <= grain) {
    for (int64_t i = 0; i < n; ++i) body(i);
    return;
  }
  std::atomic<int64_t> cursor{0};
  auto work = [&]() {
    for (;;) {
      const int64_t lo = cursor.fetch_add(grain);
      if (lo >= n) break;
      const int64_t hi = std::min(n, lo + grain);
      for (int64_t i = lo; i < hi; ++i) body(i);
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < w; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
}

inline void atomic_min_u64(std::atomic<uint64_t>& a, uint64_t v) {
  uint64_t cur = a.load(std::memory_order_relaxed);
  while (v < cur && !a.compare_exchange_weak(cur, v, std::memory_order_relaxed)) {
  }
}

}  // namespace orc
