// Host thread pool for the automaton build (build speed).
//
// One process-wide pool of worker threads. parallel_for splits [0, n) into
// grain-sized pieces that the caller and the workers take from an atomic
// counter. A build running while another thread's build holds the pool (the
// drop-in run_partitioned builds one machine per worker thread) runs its loops
// inline: the pool never nests or blocks on itself.
#pragma once

#include <algorithm>
#include <cstddef>
#include <functional>
#include <vector>

namespace acg {

// Threads a parallel_for may use (caller included); ACG_BUILD_THREADS caps it.
unsigned build_threads();

// f(lo, hi) over pieces of [0, n); inline when n <= grain or the pool is busy.
void parallel_for(std::size_t n, std::size_t grain, const std::function<void(std::size_t, std::size_t)>& f);

// Sort on the pool: pieces sorted in parallel, then merged pairwise in rounds.
template <typename T, typename Less>
void parallel_sort(std::vector<T>& v, Less less) {
    const std::size_t n = v.size();
    const std::size_t parts = std::min<std::size_t>(build_threads(), std::max<std::size_t>(1, n / 4096));
    if (parts <= 1) {
        std::sort(v.begin(), v.end(), less);
        return;
    }
    std::vector<std::size_t> cut(parts + 1);
    for (std::size_t i = 0; i <= parts; ++i) cut[i] = n * i / parts;
    parallel_for(parts, 1, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) std::sort(v.begin() + cut[i], v.begin() + cut[i + 1], less);
    });
    std::vector<T> tmp(n);
    std::vector<T>* src = &v;
    std::vector<T>* dst = &tmp;
    for (std::size_t width = 1; width < parts; width *= 2) {
        const std::size_t pairs = (parts + 2 * width - 1) / (2 * width);
        parallel_for(pairs, 1, [&](std::size_t lo, std::size_t hi) {
            for (std::size_t p = lo; p < hi; ++p) {
                const std::size_t a = cut[std::min(parts, 2 * width * p)];
                const std::size_t m = cut[std::min(parts, 2 * width * p + width)];
                const std::size_t b = cut[std::min(parts, 2 * width * p + 2 * width)];
                std::merge(src->begin() + a, src->begin() + m, src->begin() + m, src->begin() + b, dst->begin() + a,
                           less);
            }
        });
        std::swap(src, dst);
    }
    if (src != &v) v.swap(*src);
}

}  // namespace acg
