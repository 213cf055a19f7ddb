// sigker::ThreadPool (include/sigker/thread_pool.hpp, the reference's
// include/sigker/thread_pool.hpp API; the reference has no unit test for it) -- every index
// visited exactly once, chunk partition contiguous, exceptions propagate,
// the pool is reusable after a throw, a one-worker pool runs inline.
#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "sigker/thread_pool.hpp"

#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);         \
      return 1;                                                       \
    }                                                                 \
  } while (0)

int main() {
  for (unsigned w : {1u, 2u, 3u, 8u}) {
    sigker::ThreadPool pool(w);
    CHECK(pool.workers() == w);
    for (std::size_t count : {0ul, 1ul, 7ul, 1000ul}) {
      std::vector<std::atomic<int>> hits(count);
      std::vector<std::size_t> lo(w, 0), hi(w, 0);
      pool.parallel_for(count, [&](unsigned chunk, std::size_t b, std::size_t e) {
        lo[chunk] = b;
        hi[chunk] = e;
        for (std::size_t i = b; i < e; ++i) hits[i]++;
      });
      for (std::size_t i = 0; i < count; ++i) CHECK(hits[i] == 1);
      std::size_t expect = 0;  // chunks tile [0, count) in order
      for (unsigned c = 0; c < w; ++c) {
        if (hi[c] == 0) continue;
        CHECK(lo[c] == expect);
        expect = hi[c];
      }
      CHECK(expect == count);
    }
    bool caught = false;
    try {
      pool.parallel_for(100, [&](unsigned chunk, std::size_t, std::size_t) {
        if (chunk == w - 1) throw std::runtime_error("chunk failure");
      });
    } catch (const std::runtime_error&) {
      caught = true;
    }
    CHECK(caught);
    std::atomic<std::size_t> sum{0};
    pool.parallel_for(100, [&](unsigned, std::size_t b, std::size_t e) {
      for (std::size_t i = b; i < e; ++i) sum += i;
    });
    CHECK(sum == 4950);
  }
  std::printf("thread pool: all checks passed\n");
  return 0;
}
