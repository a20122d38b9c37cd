// Times run_partitioned (drop-in headers, GPU scan) at 1 and N workers on the
// reference acceptance criterion 7 workload (reference corpus generator).
// Build here (needs /root/reference): see tools/build_partition_timing.sh
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include "acmatch/aho_corasick.hpp"
#include "acmatch/corpus.hpp"
#include "acmatch/partition.hpp"
using namespace acmatch;

int main(int argc, char** argv) {
    CorpusSpec spec;
    spec.input_bytes = 4u << 20;
    spec.pattern_count = 120000;
    spec.min_len = 8;
    spec.max_len = 16;
    spec.plant_fraction = 0.2;
    spec.seed = 20260810;
    const Corpus c = generate_corpus(spec);
    const unsigned hw = argc > 1 ? static_cast<unsigned>(std::atoi(argv[1])) : std::thread::hardware_concurrency();
    for (unsigned w : {1u, hw, 1u, hw}) {
        const PartitionedRun r = run_partitioned(c.patterns, c.input, w);
        double mb = 0, ms = 0;
        for (double x : r.per_worker_build_s) mb = std::max(mb, x);
        for (double x : r.per_worker_scan_s) ms = std::max(ms, x);
        std::printf("workers %2u: wall %.4f s  max build %.4f s  max scan %.4f s  matches %zu\n", w, r.total_wall_s,
                    mb, ms, r.matches.size());
    }
}
