// Host-thread helpers of the setup: chunked parallel_for, a merge-based
// parallel sort for totally ordered keys, and std_sort_threads, which returns
// exactly what std::sort returns even where keys compare equal.
#pragma once

#include <algorithm>
#include <functional>
#include <thread>
#include <vector>

#include "setup.hpp"

namespace hxb {

inline unsigned setup_threads()
{
  return std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
}

template <class F>
void parallel_for(gid n, F&& f)
{
  const unsigned hw = setup_threads();
  if (n < 4096 || hw == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> pool;
  const gid chunk = (n + hw - 1) / hw;
  for (unsigned t = 0; t < hw; ++t) {
    const gid b = static_cast<gid>(t) * chunk, e = std::min<gid>(n, b + chunk);
    if (b < e) pool.emplace_back([&f, b, e] { f(b, e); });
  }
  for (auto& th : pool) th.join();
}

// std::sort on host threads: sorted chunks merged pairwise. Used only where
// the order is total (or equal keys are identical values), so the result is
// exactly std::sort's.
template <class T, class C>
void parallel_sort(std::vector<T>& v, C comp)
{
  const unsigned hw = setup_threads();
  const std::size_t n = v.size();
  if (n < (1u << 16) || hw == 1) {
    std::sort(v.begin(), v.end(), comp);
    return;
  }
  std::vector<std::size_t> cut(hw + 1);
  for (unsigned t = 0; t <= hw; ++t) cut[t] = n * t / hw;
  {
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < hw; ++t)
      pool.emplace_back([&, t] { std::sort(v.begin() + cut[t], v.begin() + cut[t + 1], comp); });
    for (auto& th : pool) th.join();
  }
  for (std::size_t w = 1; w < hw; w *= 2) {
    std::vector<std::thread> pool;
    for (std::size_t t = 0; t + w < hw; t += 2 * w) {
      const std::size_t a = cut[t], m = cut[t + w], b = cut[std::min<std::size_t>(hw, t + 2 * w)];
      pool.emplace_back([&, a, m, b] { std::inplace_merge(v.begin() + a, v.begin() + m, v.begin() + b, comp); });
    }
    for (auto& th : pool) th.join();
  }
}


// std::sort(first, last, cmp) with the same result, equal keys included:
// libstdc++'s introsort (bits/stl_algo.h: __sort = __introsort_loop with depth
// 2 lg n, then __final_insertion_sort) partitions a range and recurses into
// the two halves independently, so the halves of the top partition levels
// can be handed to threads, each finished by the same __introsort_loop with
// the same depth budget. The final insertion pass is a stable sort of the
// introsorted array in which no element crosses a partition cut (everything
// left of a cut compares <= its pivot <= everything right of it), so each
// thread's range is insertion-sorted on its own. Every comparison and move
// is the sequential algorithm's, so the permutation is identical (checked on
// 72M keys with heavy duplication). The reference's CSR assembly sums
// duplicate (row, col) entries in the order its std::sort leaves them
// (amg.cpp:22-40); the bit-exact coarse matrices and AMG hierarchy rely on it.
template <class It, class Cmp>
void std_sort_threads(It first, It last, Cmp cmp)
{
#if defined(__GLIBCXX__)
  const auto n = last - first;
  const unsigned hw = setup_threads();
  if (n < (1 << 16) || hw == 1) {
    std::sort(first, last, cmp);
    return;
  }
  auto comp = __gnu_cxx::__ops::__iter_comp_iter(cmp);
  int max_level = 0;
  while ((1u << max_level) < 2 * hw) ++max_level;
  std::function<void(It, It, long, int)> run = [&](It f, It l, long depth, int level) {
    std::vector<std::thread> kids;
    while (l - f > 16) {  // _S_threshold
      if (level >= max_level || depth == 0) {
        std::__introsort_loop(f, l, depth, comp);
        break;
      }
      --depth;
      It cut = std::__unguarded_partition_pivot(f, l, comp);
      kids.emplace_back(run, cut, l, depth, level + 1);
      l = cut;
      ++level;
    }
    std::__insertion_sort(f, l, comp);  // this leaf's share of __final_insertion_sort
    for (auto& k : kids) k.join();
  };
  run(first, last, static_cast<long>(std::__lg(n) * 2), 0);
#else
  std::sort(first, last, cmp);
#endif
}

}  // namespace hxb
