// Tests of the drop-in's EXTENSIONS (not reference tests): the GPU-native
// run_partitioned's device timings, the device-timed benchmark rows and the
// pipelined scan of a page-locked file. Built by oracle/Makefile against the
// drop-in headers (reference bench.hpp / corpus.hpp from the reference tree),
// run by tests/test_dropin.py on the GPU.
#include <gtest/gtest.h>

#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#include "acmatch/bench_gpu.hpp"
#include "acmatch/io.hpp"
#include "acmatch/partition.hpp"

namespace {

std::vector<acmatch::Pattern> words(std::initializer_list<const char*> w) {
    std::vector<acmatch::Pattern> p;
    for (const char* s : w) p.push_back(acmatch::Pattern{static_cast<std::uint32_t>(p.size()), s});
    return p;
}

}  // namespace

TEST(RunPartitionedGpu, DeviceTimingsAndMergedOrder) {
    const auto pats = words({"HE", "SHE", "HIS", "HERS", "E", "S"});
    std::string text;
    for (int i = 0; i < 5000; ++i) text += "USHERSHISHE";
    for (unsigned n : {1u, 2u, 3u, 6u, 9u}) {
        const auto run = acmatch::run_partitioned(pats, text, n);
        const auto ref = acmatch::scan(acmatch::build(pats), text);
        EXPECT_EQ(run.matches, ref);
        EXPECT_EQ(run.workers_launched, std::min<unsigned>(n, 6));
        ASSERT_EQ(run.per_worker_gpu_scan_s.size(), run.workers_launched);
        for (double g : run.per_worker_gpu_scan_s) EXPECT_GT(g, 0.0);
        EXPECT_GE(run.merge_gpu_s, 0.0);
        EXPECT_GT(run.total_wall_s, 0.0);
    }
}

TEST(BenchGpu, RowsAndCsv) {
    const auto pats = words({"AC", "CGT", "TTT", "A"});
    std::string text;
    for (int i = 0; i < 20000; ++i) text += "ACGTTTAC";
    acmatch::BenchConfig cfg;
    cfg.worker_counts = {4, 1, 2};
    cfg.repeats = 2;
    cfg.warmup = 1;
    const auto rows = acmatch::run_benchmark_gpu(pats, text, cfg);
    ASSERT_EQ(rows.size(), 3u);
    EXPECT_EQ(rows[0].workers, 1u);
    EXPECT_EQ(rows[2].workers, 4u);
    for (const auto& r : rows) {
        EXPECT_EQ(r.matches, rows[0].matches);
        EXPECT_GT(r.avg_gpu_scan_s, 0.0);
        EXPECT_GT(r.throughput, 0.0);
    }
    std::ostringstream os;
    acmatch::write_csv_gpu(rows, os);
    const std::string out = os.str();
    EXPECT_EQ(out.substr(0, acmatch::kCsvHeader.size()), std::string(acmatch::kCsvHeader));
    EXPECT_NE(out.find(",avg_gpu_scan_s,avg_h2d_gpu_s,avg_merge_gpu_s,avg_d2h_s\n"), std::string::npos);
    EXPECT_EQ(std::count(out.begin(), out.end(), '\n'), 4);
}

TEST(PinnedInput, PipelinedScanEqualsScan) {
    const auto pats = words({"GATTACA", "TACA", "A", "CC"});
    std::string text;
    for (int i = 0; i < 300000; ++i) text += "GATTACACCGT"[i % 11];
    const std::string path = "/tmp/acg_dropin_ext_input.bin";
    acmatch::write_bytes(path, text);
    const acmatch::PinnedInput in(path);
    ASSERT_EQ(in.size(), text.size());
    const auto a = acmatch::build(pats);
    EXPECT_EQ(acmatch::scan(a, in), acmatch::scan(a, std::string_view(text)));
    std::remove(path.c_str());
}
