// Eq. (1) rows of the reference's benchmark harness with device-timed columns
// (SURVEY §8(f) rank 4). The reference's rows (proj/include/acmatch/
// bench.hpp:34-51: workers, input bytes, dictionary size, matches, mean
// build/scan/total seconds, stddev, matches per second) are host wall times
// of run_partitioned; here each row also carries the CUDA-event times the
// GPU-native run_partitioned reports (partition.hpp drop-in): the workers'
// scans on the device (slowest worker, as the reference's critical-path
// columns), the input's one H2D copy, the device merge and the read-back.
// The reference's BenchConfig, BenchRow, kCsvHeader, write_csv and
// throughput are used as they are (bench.hpp comes from the reference).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <ostream>
#include <string>
#include <string_view>
#include <vector>

#include "acmatch/bench.hpp"
#include "acmatch/partition.hpp"

namespace acmatch {

struct GpuBenchRow : BenchRow {
    double avg_gpu_scan_s = 0.0;  // slowest worker's device scan time, mean over repeats
    double avg_h2d_gpu_s = 0.0;
    double avg_merge_gpu_s = 0.0;
    double avg_d2h_s = 0.0;
};

inline const std::string& csv_header_gpu() {
    static const std::string h = std::string(kCsvHeader) + ",avg_gpu_scan_s,avg_h2d_gpu_s,avg_merge_gpu_s,avg_d2h_s";
    return h;
}

// run_benchmark (bench.hpp:83-122) over the GPU-native run_partitioned:
// warm-up runs, timed repeats, means of the per-run critical paths, results
// checked identical across repeats; rows ordered by worker count.
inline std::vector<GpuBenchRow> run_benchmark_gpu(const std::vector<Pattern>& patterns, std::string_view input,
                                                  const BenchConfig& config) {
    if (config.worker_counts.empty()) throw Error("worker_counts must not be empty");
    for (unsigned n : config.worker_counts)
        if (n < 1) throw InvalidWorkerCountError("worker count must be >= 1");
    if (config.repeats < 1) throw Error("repeats must be >= 1");
    std::vector<unsigned> counts = config.worker_counts;
    std::sort(counts.begin(), counts.end());
    auto mean = [](const std::vector<double>& v) { return std::accumulate(v.begin(), v.end(), 0.0) / v.size(); };
    auto slowest = [](const std::vector<double>& v) { return v.empty() ? 0.0 : *std::max_element(v.begin(), v.end()); };
    std::vector<GpuBenchRow> rows;
    for (const unsigned n : counts) {
        for (unsigned w = 0; w < config.warmup; ++w) (void)run_partitioned(patterns, input, n);
        std::vector<double> b, s, t, g, h, m, d;
        std::vector<MatchRecord> first;
        for (unsigned r = 0; r < config.repeats; ++r) {
            PartitionedRun run = run_partitioned(patterns, input, n);
            b.push_back(slowest(run.per_worker_build_s));
            s.push_back(slowest(run.per_worker_scan_s));
            g.push_back(slowest(run.per_worker_gpu_scan_s));
            t.push_back(run.total_wall_s);
            h.push_back(run.h2d_gpu_s);
            m.push_back(run.merge_gpu_s);
            d.push_back(run.d2h_s);
            if (r == 0) first = std::move(run.matches);
            else if (run.matches != first) throw Error("match results changed between repeats");
        }
        GpuBenchRow row;
        row.workers = n;
        row.input_bytes = input.size();
        row.dictionary_size = patterns.size();
        row.matches = first.size();
        row.avg_build_s = mean(b);
        row.avg_scan_s = mean(s);
        row.avg_total_s = mean(t);
        double var = 0.0;
        for (double x : t) var += (x - row.avg_total_s) * (x - row.avg_total_s);
        row.stddev_total_s = std::sqrt(var / t.size());
        row.throughput = throughput(row.matches, row.avg_total_s);
        row.avg_gpu_scan_s = mean(g);
        row.avg_h2d_gpu_s = mean(h);
        row.avg_merge_gpu_s = mean(m);
        row.avg_d2h_s = mean(d);
        rows.push_back(row);
    }
    return rows;
}

// The reference's CSV (write_csv, bench.hpp:163-190) with the device columns appended.
inline void write_csv_gpu(const std::vector<GpuBenchRow>& rows, std::ostream& os) {
    os << csv_header_gpu() << '\n';
    auto g9 = [](std::string& line, double v) {
        char buf[40];
        std::snprintf(buf, sizeof buf, "%.9g", v);
        line += buf;
    };
    for (const GpuBenchRow& r : rows) {
        std::string line = std::to_string(r.workers) + ',' + std::to_string(r.input_bytes) + ',' +
                           std::to_string(r.dictionary_size) + ',' + std::to_string(r.matches);
        for (double v : {r.avg_build_s, r.avg_scan_s, r.avg_total_s, r.stddev_total_s, r.throughput, r.avg_gpu_scan_s,
                         r.avg_h2d_gpu_s, r.avg_merge_gpu_s, r.avg_d2h_s}) {
            line += ',';
            g9(line, v);
        }
        os << line << '\n';
    }
}

}  // namespace acmatch
