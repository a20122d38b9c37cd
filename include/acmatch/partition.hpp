// Drop-in for the reference's dictionary-partitioned run
// (/root/reference/proj/include/acmatch/partition.hpp:29-170): same types,
// split rule, error behaviour and timing fields. Each worker thread builds
// the machine for its contiguous chunk of the dictionary and scans the whole
// input on the GPU (workers' scans run concurrently, one scanner each); the
// per-worker lists are merged into global (end, pattern_id) order.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <functional>
#include <future>
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
};

namespace detail {

struct WorkerOutcome {
    std::vector<MatchRecord> found;  // global ids, (end, pattern_id) order
    double build_s = 0, scan_s = 0;
};

// One worker: build the chunk's machine (local ids 0..k-1), scan the whole
// input on the GPU, map local ids back to global (the map ascends, so the
// order is kept).
inline WorkerOutcome partition_worker(const std::vector<Pattern>& patterns, const std::vector<std::uint32_t>& ids,
                                      std::string_view input) {
    using clock = std::chrono::steady_clock;
    const auto b0 = clock::now();
    std::vector<Pattern> local;
    local.reserve(ids.size());
    for (const std::uint32_t g : ids) local.push_back(Pattern{static_cast<std::uint32_t>(local.size()), patterns[g].bytes});
    const Automaton machine = build(std::move(local));
    const auto s0 = clock::now();
    WorkerOutcome out;
    out.found = scan(machine, input);
    const auto s1 = clock::now();
    for (MatchRecord& r : out.found) r.pattern_id = ids[r.pattern_id];
    out.build_s = std::chrono::duration<double>(s0 - b0).count();
    out.scan_s = std::chrono::duration<double>(s1 - s0).count();
    return out;
}

}  // namespace detail

// The paper's scheme (:101-170): one worker per non-empty dictionary chunk,
// all started at once; a failure in any worker fails the run (the lowest
// chunk's error is rethrown, after every worker has finished).
inline PartitionedRun run_partitioned(const std::vector<Pattern>& patterns, std::string_view input,
                                      unsigned worker_count) {
    const auto t0 = std::chrono::steady_clock::now();
    const PartitionPlan plan = split_patterns(patterns, worker_count);
    std::vector<std::future<detail::WorkerOutcome>> pending;
    for (const auto& chunk : plan.chunks)
        if (!chunk.empty())
            pending.push_back(std::async(std::launch::async, detail::partition_worker, std::cref(patterns),
                                         std::cref(chunk), input));
    for (auto& f : pending) f.wait();

    PartitionedRun run;
    run.worker_count = worker_count;
    run.workers_launched = static_cast<unsigned>(pending.size());
    std::vector<std::vector<MatchRecord>> lists;
    for (auto& f : pending) {
        detail::WorkerOutcome w = f.get();  // rethrows that worker's error
        run.per_worker_build_s.push_back(w.build_s);
        run.per_worker_scan_s.push_back(w.scan_s);
        lists.push_back(std::move(w.found));
    }
    run.matches = merge_matches(lists);
    run.total_wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return run;
}

}  // namespace acmatch
