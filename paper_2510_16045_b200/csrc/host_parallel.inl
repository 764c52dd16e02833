// host_parallel.inl -- static row partition over std::threads with the first worker
// exception rethrown after join (same contract as the reference parallel_for,
// parallel.hpp:24-53: results never depend on the partition).
#pragma once

#include <algorithm>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

namespace amsqb {

template <typename Body>
void parallel_rows(size_t n, int threads, Body&& body) {
  const size_t workers = std::min<size_t>(static_cast<size_t>(resolve_threads(threads)),
                                          n == 0 ? 1 : n);
  if (workers <= 1) {
    body(size_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::mutex mu;
  const size_t chunk = (n + workers - 1) / workers;
  for (size_t w = 0; w < workers; ++w) {
    const size_t b = w * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    pool.emplace_back([&, b, e] {
      try {
        body(b, e);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err) err = std::current_exception();
      }
    });
  }
  for (auto& t : pool) t.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace amsqb
