// Drop-in for the reference's dictionary-partitioned run
// (/root/reference/proj/include/acmatch/partition.hpp:29-170): same types,
// split rule, error behaviour and timing fields (plus device-timed ones).
// run_partitioned is the library's acg_run_partitioned: each worker builds the
// machine for its contiguous chunk of the dictionary on a host thread and
// scans the one device copy of the input; the lists are merged on the device.
// merge_matches (the host merge of given lists) keeps the reference's API.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <functional>
#include <memory>
#include <string_view>
#include <thread>
#include <vector>

#include "acmatch/aho_corasick.hpp"
#include "acmatch/errors.hpp"

namespace acmatch {

// Contiguous dictionary chunks whose sizes differ by at most one (:29-38).
struct PartitionPlan {
    unsigned worker_count = 1;
    std::vector<std::vector<std::uint32_t>> chunks;  // global pattern ids

    std::size_t non_empty_chunks() const noexcept {
        return static_cast<std::size_t>(
            std::count_if(chunks.begin(), chunks.end(), [](const auto& c) { return !c.empty(); }));
    }
};

// worker_count chunks; the first (size mod worker_count) get one extra (:42-60).
inline PartitionPlan split_patterns(const std::vector<Pattern>& patterns, unsigned worker_count) {
    if (worker_count < 1) throw InvalidWorkerCountError("worker count must be >= 1");
    if (patterns.empty()) throw EmptyDictionaryError("dictionary is empty");
    PartitionPlan plan;
    plan.worker_count = worker_count;
    plan.chunks.resize(worker_count);
    const std::size_t q = patterns.size() / worker_count, r = patterns.size() % worker_count;
    std::uint32_t id = 0;
    for (unsigned k = 0; k < worker_count; ++k) {
        const std::size_t len = q + (k < r ? 1 : 0);
        plan.chunks[k].resize(len);
        for (auto& slot : plan.chunks[k]) slot = id++;
    }
    return plan;
}

// Merge of per-worker lists, each already in (end, pattern_id) order
// (:65-89). Chunks are disjoint, so records never repeat: pairwise merging
// in rounds gives the same sequence as the reference's k-way heap merge.
inline std::vector<MatchRecord> merge_matches(const std::vector<std::vector<MatchRecord>>& lists) {
    std::vector<std::vector<MatchRecord>> level;
    for (const auto& l : lists)
        if (!l.empty()) level.push_back(l);
    if (level.empty()) return {};
    while (level.size() > 1) {
        std::vector<std::vector<MatchRecord>> next;
        for (std::size_t i = 0; i + 1 < level.size(); i += 2) {
            std::vector<MatchRecord> m;
            m.reserve(level[i].size() + level[i + 1].size());
            std::merge(level[i].begin(), level[i].end(), level[i + 1].begin(), level[i + 1].end(),
                       std::back_inserter(m), match_before);
            next.push_back(std::move(m));
        }
        if (level.size() % 2) next.push_back(std::move(level.back()));
        level = std::move(next);
    }
    return std::move(level.front());
}

// Results and timings of one partitioned run (:92-99).
struct PartitionedRun {
    std::vector<MatchRecord> matches;        // merged, (end, pattern_id) order
    std::vector<double> per_worker_build_s;  // one entry per launched worker
    std::vector<double> per_worker_scan_s;
    double total_wall_s = 0.0;               // split + builds + scans + merge
    unsigned worker_count = 1;               // as requested
    unsigned workers_launched = 0;           // non-empty chunks
    // new: device-timed columns (CUDA events)
    std::vector<double> per_worker_gpu_scan_s;  // each worker's scan on the device
    double h2d_gpu_s = 0.0;                      // the input's one copy to the device
    double merge_gpu_s = 0.0;                    // the device-side merge of the workers' lists
    double d2h_s = 0.0;                          // the merged list's read-back
};

// The paper's scheme (:101-170), GPU-native (acg_run_partitioned): one worker
// per non-empty chunk, machines built concurrently on host threads, the input
// copied to the device once and scanned by every worker on its own stream,
// the lists merged on the device; a failure in any worker fails the run (the
// lowest chunk's error is rethrown).
inline PartitionedRun run_partitioned(const std::vector<Pattern>& patterns, std::string_view input,
                                      unsigned worker_count) {
    if (worker_count < 1) throw InvalidWorkerCountError("worker count must be >= 1");
    if (patterns.empty()) throw EmptyDictionaryError("dictionary is empty");
    std::vector<std::uint8_t> concat;
    std::vector<std::uint64_t> offs{0};
    for (std::size_t i = 0; i < patterns.size(); ++i) {  // global ids = positions (the split ignores .id)
        concat.insert(concat.end(), patterns[i].bytes.begin(), patterns[i].bytes.end());
        offs.push_back(concat.size());
    }
    acg_partitioned* r = nullptr;
    int device = 0;
    detail::check(acg_run_partitioned(concat.data(), offs.data(), static_cast<std::uint32_t>(patterns.size()),
                                      reinterpret_cast<const std::uint8_t*>(input.data()), input.size(), worker_count,
                                      device, &r));
    std::unique_ptr<acg_partitioned, void (*)(acg_partitioned*)> guard(r, acg_partitioned_destroy);
    PartitionedRun run;
    const std::uint64_t m = acg_partitioned_match_count(r);
    const std::uint32_t* ids = acg_partitioned_ids(r);
    const std::uint64_t* ends = acg_partitioned_ends(r);
    run.matches.resize(m);
    for (std::uint64_t i = 0; i < m; ++i) run.matches[i] = MatchRecord{ids[i], static_cast<std::size_t>(ends[i])};
    std::uint32_t wc = 0, launched = 0;
    const double *build_s = nullptr, *scan_s = nullptr, *gpu_ms = nullptr;
    double total_s = 0, h2d_ms = 0, merge_ms = 0, d2h_ms = 0;
    detail::check(acg_partitioned_timings(r, &wc, &launched, &build_s, &scan_s, &gpu_ms, &total_s, &h2d_ms, &merge_ms,
                                          &d2h_ms));
    run.worker_count = wc;
    run.workers_launched = launched;
    run.per_worker_build_s.assign(build_s, build_s + launched);
    run.per_worker_scan_s.assign(scan_s, scan_s + launched);
    for (std::uint32_t k = 0; k < launched; ++k) run.per_worker_gpu_scan_s.push_back(gpu_ms[k] * 1e-3);
    run.h2d_gpu_s = h2d_ms * 1e-3;
    run.merge_gpu_s = merge_ms * 1e-3;
    run.d2h_s = d2h_ms * 1e-3;
    run.total_wall_s = total_s;
    return run;
}

}  // namespace acmatch
