// The paper's dictionary-partitioned run, GPU-native.
//
// Reference: run_partitioned / split_patterns / merge_matches
// (proj/include/acmatch/partition.hpp:29-170): the dictionary is cut into
// worker_count contiguous chunks (sizes differ by at most one, the first
// size mod worker_count get one extra), each non-empty chunk's worker builds
// its own machine and scans the whole input, and the per-worker lists are
// k-way merged into (end, pattern_id) order with global ids.
//
// Here the input is copied to the device ONCE and every worker scans that
// device copy on its own stream (builds run on host threads concurrently);
// the lists stay on the device: each worker's packed records are remapped to
// global ids (chunk ids are contiguous: global = chunk start + local) into
// one buffer, merged pairwise with a merge-path kernel (log2 k rounds), and
// widened to (id, end) for one D2H of the final list. Per-worker host times
// (build, scan) follow the reference's fields; device times of each scan and
// of the merge are reported besides.
#pragma once

#include "acg.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <thread>
#include <vector>


struct acg_partitioned {
    std::vector<std::uint32_t> ids;
    std::vector<std::uint64_t> ends;
    std::vector<double> build_s, scan_s, gpu_scan_ms;
    double total_s = 0, merge_ms = 0, h2d_ms = 0, d2h_ms = 0;
    std::uint32_t worker_count = 1, launched = 0;
};

namespace part {

constexpr int kMergeItems = 64;  // outputs per thread of the merge-path kernel (one diagonal search per 64)

// records of worker k: (end << ib | local) -> (end << gb | start + local)
__global__ void remap_kernel(const unsigned long long* in, unsigned long long m, std::uint32_t ib, std::uint32_t gb,
                             std::uint32_t start, unsigned long long* out) {
    const unsigned long long mask = (1ull << ib) - 1;
    for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < m; i += gridDim.x * 256ull) {
        const unsigned long long r = in[i];
        out[i] = ((r >> ib) << gb) | (start + (r & mask));
    }
}

// out[0, na+nb) = merge of sorted a and b (keys unique): each thread finds its
// diagonal's split by binary search (merge path), then merges kMergeItems outputs.
__global__ void merge_path_kernel(const unsigned long long* a, unsigned long long na, const unsigned long long* b,
                                  unsigned long long nb, unsigned long long* out) {
    const unsigned long long total = na + nb;
    for (unsigned long long d = (blockIdx.x * 256ull + threadIdx.x) * kMergeItems; d < total;
         d += gridDim.x * 256ull * kMergeItems) {
        unsigned long long lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
        while (lo < hi) {
            const unsigned long long mid = (lo + hi) >> 1;
            if (a[mid] < b[d - mid - 1]) lo = mid + 1;
            else hi = mid;
        }
        unsigned long long i = lo, j = d - lo;
        const unsigned long long e = d + kMergeItems < total ? d + kMergeItems : total;
        for (unsigned long long o = d; o < e; ++o) {
            const bool take_a = j >= nb || (i < na && a[i] < b[j]);
            out[o] = take_a ? a[i++] : b[j++];
        }
    }
}

__global__ void widen_kernel(const unsigned long long* keys, unsigned long long m, std::uint32_t gb, std::uint32_t* ids,
                             unsigned long long* ends) {
    const unsigned long long mask = (1ull << gb) - 1;
    for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < m; i += gridDim.x * 256ull) {
        ids[i] = static_cast<std::uint32_t>(keys[i] & mask);
        ends[i] = keys[i] >> gb;
    }
}

std::uint32_t bits_for(std::uint64_t n) {
    std::uint32_t b = 1;
    while ((1ull << b) < n) ++b;
    return b;
}

struct Worker {
    std::uint32_t start = 0, len = 0;
    acg_automaton* a = nullptr;
    acg_scanner* s = nullptr;
    cudaStream_t st = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int rc = ACG_OK;
    std::string err;
    double build_s = 0, scan_s = 0;
    float gpu_ms = 0;
};

}  // namespace part

extern "C" {

int acg_run_partitioned(const uint8_t* concat, const uint64_t* offsets, uint32_t n_patterns, const uint8_t* text,
                        uint64_t n, uint32_t worker_count, int device, acg_partitioned** out) {
    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    if (!out || !offsets || (!text && n)) return acg_internal_set_error(ACG_ERR_INVALID, "null argument");
    *out = nullptr;
    // split_patterns (partition.hpp:42-60)
    if (worker_count < 1) return acg_internal_set_error(ACG_ERR_INVALID_WORKER_COUNT, "worker count must be >= 1");
    if (n_patterns == 0) return acg_internal_set_error(ACG_ERR_EMPTY_DICTIONARY, "dictionary is empty");
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        return acg_internal_set_error(ACG_ERR_NO_DEVICE, "no usable CUDA device");
    }
    auto res = std::make_unique<acg_partitioned>();
    res->worker_count = worker_count;
    const std::uint32_t q = n_patterns / worker_count, r = n_patterns % worker_count;
    using namespace part;
    std::vector<Worker> ws;
    for (std::uint32_t k = 0, id = 0; k < worker_count; ++k) {
        const std::uint32_t len = q + (k < r ? 1u : 0u);
        if (len) ws.push_back(Worker{id, len});
        id += len;
    }
    res->launched = static_cast<std::uint32_t>(ws.size());

    int rc = ACG_OK;
    auto cuda_fail = [&](cudaError_t e, const char* what) {
        cudaGetLastError();
        return acg_internal_set_error(e == cudaErrorMemoryAllocation ? ACG_ERR_OUT_OF_MEMORY : ACG_ERR_CUDA,
                                      (std::string(cudaGetErrorString(e)) + " (" + what + ")").c_str());
    };
    cudaStream_t st = nullptr;
    std::uint8_t* d_text = nullptr;
    unsigned long long *keys = nullptr, *tmp = nullptr, *d_ends = nullptr;
    std::uint32_t* d_ids = nullptr;
    cudaEvent_t m0 = nullptr, m1 = nullptr, h0 = nullptr, h1 = nullptr;
    auto cleanup = [&] {
        for (auto& w : ws) {
            if (w.st) cudaStreamSynchronize(w.st);
            if (w.s) acg_scanner_destroy(w.s);
            if (w.a) acg_automaton_destroy(w.a);
            if (w.e0) cudaEventDestroy(w.e0);
            if (w.e1) cudaEventDestroy(w.e1);
            if (w.st) cudaStreamDestroy(w.st);
        }
        if (st) {
            for (void* p : {static_cast<void*>(d_text), static_cast<void*>(keys), static_cast<void*>(tmp),
                            static_cast<void*>(d_ends), static_cast<void*>(d_ids)})
                if (p) cudaFreeAsync(p, st);
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
        for (cudaEvent_t e : {m0, m1, h0, h1})
            if (e) cudaEventDestroy(e);
    };
#define PART_CUDA(call)                      \
    do {                                     \
        const cudaError_t e_ = (call);       \
        if (e_ != cudaSuccess) {             \
            rc = cuda_fail(e_, #call);       \
            cleanup();                       \
            return rc;                       \
        }                                    \
    } while (0)
    PART_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&m0, &m1, &h0, &h1}) PART_CUDA(cudaEventCreate(e));
    // the input, once, for every worker
    PART_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_text), std::max<std::uint64_t>(n, 16), st));
    PART_CUDA(cudaEventRecord(h0, st));
    if (n) PART_CUDA(cudaMemcpyAsync(d_text, text, n, cudaMemcpyHostToDevice, st));
    PART_CUDA(cudaEventRecord(h1, st));
    PART_CUDA(cudaStreamSynchronize(st));

    // one thread per non-empty chunk: build its machine, scan the device input
    auto work = [&](Worker& w) {
        const auto b0 = clock::now();
        std::vector<std::uint64_t> loff(w.len + 1);
        for (std::uint32_t i = 0; i <= w.len; ++i) loff[i] = offsets[w.start + i] - offsets[w.start];
        w.rc = acg_build(concat ? concat + offsets[w.start] : nullptr, loff.data(), w.len, &w.a);
        const auto s0 = clock::now();
        w.build_s = std::chrono::duration<double>(s0 - b0).count();
        if (!w.rc) acg_internal_auto_layout(w.a, text, n);
        if (!w.rc) w.rc = cudaSetDevice(device) == cudaSuccess ? ACG_OK : ACG_ERR_CUDA;
        if (!w.rc) w.rc = acg_scanner_create(w.a, device, ACG_SCAN_LIST, &w.s);
        if (!w.rc && (cudaStreamCreateWithFlags(&w.st, cudaStreamNonBlocking) != cudaSuccess ||
                      cudaEventCreate(&w.e0) != cudaSuccess || cudaEventCreate(&w.e1) != cudaSuccess))
            w.rc = ACG_ERR_CUDA;
        if (!w.rc && cudaEventRecord(w.e0, w.st) != cudaSuccess) w.rc = ACG_ERR_CUDA;
        if (!w.rc) w.rc = acg_scanner_run(w.s, d_text, n, 0, 0, w.st);
        if (!w.rc) w.rc = acg_scanner_sync(w.s);  // (replays, if any, run here)
        if (!w.rc && cudaEventRecord(w.e1, w.st) != cudaSuccess) w.rc = ACG_ERR_CUDA;
        if (!w.rc && cudaEventSynchronize(w.e1) == cudaSuccess) cudaEventElapsedTime(&w.gpu_ms, w.e0, w.e1);
        w.scan_s = std::chrono::duration<double>(clock::now() - s0).count();
        if (w.rc) w.err = acg_last_error();
    };
    {
        std::vector<std::thread> threads;
        for (std::size_t k = 1; k < ws.size(); ++k) threads.emplace_back(work, std::ref(ws[k]));
        work(ws[0]);
        for (auto& t : threads) t.join();
    }
    for (auto& w : ws)  // the lowest chunk's error (partition.hpp:140-146)
        if (w.rc) {
            rc = acg_internal_set_error(w.rc, w.err.c_str());
            cleanup();
            return rc;
        }

    // merge on the device (partition.hpp:65-89)
    if (const cudaError_t stale = cudaGetLastError(); stale != cudaSuccess && std::getenv("ACG_DEBUG"))
        std::fprintf(stderr, "[acg] run_partitioned: stale CUDA error before the merge: %s\n", cudaGetErrorString(stale));
    const std::uint32_t gb = part::bits_for(n_patterns);
    std::uint64_t m = 0;
    std::vector<std::uint64_t> seg_off, seg_len;
    for (auto& w : ws) {
        const std::uint64_t mk = acg_scanner_match_count(w.s);
        seg_off.push_back(m);
        seg_len.push_back(mk);
        m += mk;
    }
    PART_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&keys), std::max<std::uint64_t>(m, 1) * 8, st));
    PART_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), std::max<std::uint64_t>(m, 1) * 8, st));
    PART_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_ids), std::max<std::uint64_t>(m, 1) * 4, st));
    PART_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_ends), std::max<std::uint64_t>(m, 1) * 8, st));
    PART_CUDA(cudaEventRecord(m0, st));  // (merge time: kernels only)
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    auto grid = [&](std::uint64_t items) {
        return static_cast<unsigned>(std::max<std::uint64_t>(1, std::min<std::uint64_t>((items + 255) / 256, 8ull * sms)));
    };
    for (std::size_t k = 0; k < ws.size(); ++k) {
        if (!seg_len[k]) continue;
        std::uint32_t ib = 0;
        const auto* rec = reinterpret_cast<const unsigned long long*>(acg_scanner_device_records(ws[k].s, &ib));
        remap_kernel<<<grid(seg_len[k]), 256, 0, st>>>(rec, seg_len[k], ib, gb, ws[k].start, keys + seg_off[k]);
        PART_CUDA(cudaGetLastError());
    }
    // pairwise merge rounds over the chunk-ordered segments
    while (seg_len.size() > 1) {
        std::vector<std::uint64_t> no, nl;
        for (std::size_t i = 0; i < seg_len.size(); i += 2) {
            if (i + 1 == seg_len.size()) {
                PART_CUDA(cudaMemcpyAsync(tmp + seg_off[i], keys + seg_off[i], seg_len[i] * 8, cudaMemcpyDeviceToDevice, st));
                no.push_back(seg_off[i]);
                nl.push_back(seg_len[i]);
                continue;
            }
            const std::uint64_t tot = seg_len[i] + seg_len[i + 1];
            if (tot)
                merge_path_kernel<<<grid((tot + kMergeItems - 1) / kMergeItems), 256, 0, st>>>(
                    keys + seg_off[i], seg_len[i], keys + seg_off[i + 1], seg_len[i + 1], tmp + seg_off[i]);
            PART_CUDA(cudaGetLastError());
            no.push_back(seg_off[i]);
            nl.push_back(tot);
        }
        std::swap(keys, tmp);
        seg_off.swap(no);
        seg_len.swap(nl);
    }
    if (m) widen_kernel<<<grid(m), 256, 0, st>>>(keys, m, gb, d_ids, d_ends);
    PART_CUDA(cudaGetLastError());
    PART_CUDA(cudaEventRecord(m1, st));
    res->ids.resize(m);
    res->ends.resize(m);
    const auto d0 = clock::now();
    if (m) {
        PART_CUDA(cudaMemcpyAsync(res->ids.data(), d_ids, m * 4, cudaMemcpyDeviceToHost, st));
        PART_CUDA(cudaMemcpyAsync(res->ends.data(), d_ends, m * 8, cudaMemcpyDeviceToHost, st));
    }
    PART_CUDA(cudaStreamSynchronize(st));
    res->d2h_ms = std::chrono::duration<double, std::milli>(clock::now() - d0).count();
    float ms = 0;
    cudaEventElapsedTime(&ms, m0, m1);
    res->merge_ms = ms;
    cudaEventElapsedTime(&ms, h0, h1);
    res->h2d_ms = ms;
    for (auto& w : ws) {
        res->build_s.push_back(w.build_s);
        res->scan_s.push_back(w.scan_s);
        res->gpu_scan_ms.push_back(w.gpu_ms);
    }
#undef PART_CUDA
    cleanup();
    res->total_s = std::chrono::duration<double>(clock::now() - t0).count();
    *out = res.release();
    return ACG_OK;
}

uint64_t acg_partitioned_match_count(const acg_partitioned* r) { return r ? r->ids.size() : 0; }
const uint32_t* acg_partitioned_ids(const acg_partitioned* r) { return r ? r->ids.data() : nullptr; }
const uint64_t* acg_partitioned_ends(const acg_partitioned* r) { return r ? r->ends.data() : nullptr; }

int acg_partitioned_timings(const acg_partitioned* r, uint32_t* worker_count, uint32_t* workers_launched,
                            const double** build_s, const double** scan_s, const double** gpu_scan_ms, double* total_s,
                            double* h2d_ms, double* merge_ms, double* d2h_ms) {
    if (!r) return acg_internal_set_error(ACG_ERR_INVALID, "null result");
    if (worker_count) *worker_count = r->worker_count;
    if (workers_launched) *workers_launched = r->launched;
    if (build_s) *build_s = r->build_s.data();
    if (scan_s) *scan_s = r->scan_s.data();
    if (gpu_scan_ms) *gpu_scan_ms = r->gpu_scan_ms.data();
    if (total_s) *total_s = r->total_s;
    if (h2d_ms) *h2d_ms = r->h2d_ms;
    if (merge_ms) *merge_ms = r->merge_ms;
    if (d2h_ms) *d2h_ms = r->d2h_ms;
    return ACG_OK;
}

void acg_partitioned_destroy(acg_partitioned* r) { delete r; }

}  // extern "C"
