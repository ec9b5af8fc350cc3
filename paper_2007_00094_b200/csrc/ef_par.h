// ef_par.h — host-side parallel loops for the setup (plan + layout build).
//
// The setup walks every stencil entry several times (885M entries for the
// 320^3 box, 7.1G for 640^3 over 8 ranks); it runs on all host threads
// (EF_SETUP_THREADS overrides).  Loops split [0, n) into contiguous chunks,
// one per thread, so per-thread outputs concatenate in index order.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <thread>
#include <vector>

namespace ef {

inline int par_threads() {
  static const int t = [] {
    const char* e = std::getenv("EF_SETUP_THREADS");
    int v = e ? std::atoi(e) : (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(v, 128));
  }();
  return t;
}

// f(lo, hi, chunk) over contiguous chunks of [0, n); returns the chunk count
template <class F>
int parallel_for(int64_t n, F f, int64_t min_chunk = 1 << 15) {
  if (n <= 0) return 0;
  const int64_t want = (n + min_chunk - 1) / min_chunk;
  const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(par_threads(), want));
  if (chunks == 1) {
    f((int64_t)0, n, 0);
    return 1;
  }
  std::vector<std::thread> th;
  th.reserve(chunks);
  for (int t = 0; t < chunks; ++t) th.emplace_back(f, n * t / chunks, n * (t + 1) / chunks, t);
  for (auto& x : th) x.join();
  return chunks;
}

// std::vector whose resize leaves trivially constructible elements
// uninitialised (every element is written by a parallel loop afterwards)
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = DefaultInitAlloc<U>;
  };
  DefaultInitAlloc() = default;
  template <class U>
  DefaultInitAlloc(const DefaultInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using hvec = std::vector<T, DefaultInitAlloc<T>>;

}  // namespace ef
