// libacg.so: the C ABI of include/acg.h — host automaton, device DFA upload,
// scanner workspace and the kernel pipeline
//   sparse mode: K1s sparse_scan_kernel (truncated automaton, event log)
//                K1f fixup_kernel<COUNT> (exact replay of cold excursions)
//   exact mode:  K1x exact_scan_kernel<COUNT>
//   K2 cub::DeviceScan       exclusive prefix of chunk counts -> record slots (u64)
//   K3 compact + fixup_kernel<WRITE> / exact_scan_kernel<WRITE>: ordered packed records
//   K4 pattern_counts_kernel per-pattern counts from per-state visits
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "../../include/acg.h"
#include "automaton.hpp"
#include "ctab.hpp"
#include "scan_kernels.cuh"
#include "filter_kernels.cuh"
#include "exact_kernels.cuh"
#include "format_kernels.cuh"

namespace {

thread_local std::string g_last_error;
const bool g_debug = [] {  // ACG_DEBUG=1: per-run decisions on stderr (experiments)
    const char* e = std::getenv("ACG_DEBUG");
    return e && e[0] == '1';
}();

// Device start-up happens when the library is loaded rather than inside the
// caller's first scan: driver initialisation (cuInit, ~0.6 s on a B200 node),
// the primary context of the process's device (LOCAL_RANK under torchrun,
// else 0) and the loading of the kernels a first small scan uses (CUDA loads
// kernels lazily, on first launch). A drop-in user's first acmatch::scan then
// costs about what later ones do (the reference's acceptance runner bounds
// its first criterion, a 5-byte scan, at 1 s). ACG_EAGER_INIT=0 turns it off
// (e.g. for a process that forks CUDA-using children); without a device it
// does nothing.
void warm_up_device(int device);
struct EagerDriverInit {
    EagerDriverInit() {
        const char* e = std::getenv("ACG_EAGER_INIT");
        if (e && e[0] == '0') return;
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count <= 0) {
            (void)cudaGetLastError();
            return;
        }
        int dev = 0;
        if (const char* lr = std::getenv("LOCAL_RANK")) dev = std::atoi(lr);
        if (dev < 0 || dev >= count) dev = 0;
        warm_up_device(dev);
        (void)cudaGetLastError();
    }
};  // instantiated at the end of this file's globals (after the pools it uses)

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define ACG_CUDA(call)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) {                                                                    \
            return fail(e_ == cudaErrorMemoryAllocation ? ACG_ERR_OUT_OF_MEMORY : ACG_ERR_CUDA,     \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                        \
        }                                                                                           \
    } while (0)

// Device memory comes from each device's stream-ordered pool (cudaMallocAsync
// / cudaFreeAsync) with the release threshold lifted, so workspace growth and
// automaton teardown never synchronise the device or return memory to the
// driver (run_partitioned builds, scans and drops one automaton per worker on
// every run). Buffers are allocated on the stream that first uses them;
// destructors run only after the owner synchronised its streams and free on
// the device's housekeeping stream (never destroyed).
std::mutex g_hk_mu;
std::map<int, cudaStream_t> g_hk;

cudaStream_t hk_stream(int device) {
    std::lock_guard<std::mutex> lock(g_hk_mu);
    auto it = g_hk.find(device);
    if (it != g_hk.end()) return it->second;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        std::uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaStream_t st = nullptr;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaGetLastError();
    cudaSetDevice(prev);
    g_hk[device] = st;
    return st;
}

int current_device_or0() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return d;
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    std::size_t n = 0;  // capacity in elements
    int dev = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, hk_stream(dev));
    }
    // grows in stream order on `st` (the old contents are not kept)
    cudaError_t reserve(std::size_t want, cudaStream_t st) {
        if (want <= n && p) return cudaSuccess;
        dev = current_device_or0();
        (void)hk_stream(dev);  // the pool's release threshold is set before its first use
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
        n = 0;
        const std::size_t cap = std::max<std::size_t>(want, 1);
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), cap * sizeof(T), st);
        if (e == cudaErrorMemoryAllocation) {
            // the pool keeps freed blocks: return the unused ones to the
            // driver (after the frees completed) and try once more
            cudaGetLastError();
            cudaStreamSynchronize(st);
            cudaStreamSynchronize(hk_stream(dev));
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
            e = cudaMallocAsync(reinterpret_cast<void**>(&p), cap * sizeof(T), st);
        }
        if (e == cudaSuccess) n = cap;
        else p = nullptr;
        return e;
    }
};

// Small pinned host words for scanner scalars, carved from slabs that are
// never freed (cudaFreeHost would synchronise the device).
std::mutex g_pin_mu;
std::vector<unsigned long long*> g_pin_free;

unsigned long long* pinned_take() {
    std::lock_guard<std::mutex> lock(g_pin_mu);
    if (g_pin_free.empty()) {
        constexpr int kPieces = 512, kWords = 8;
        unsigned long long* slab = nullptr;
        if (cudaMallocHost(&slab, kPieces * kWords * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
        for (int i = kPieces - 1; i >= 0; --i) g_pin_free.push_back(slab + i * kWords);
    }
    unsigned long long* p = g_pin_free.back();
    g_pin_free.pop_back();
    return p;
}
void pinned_give(unsigned long long* p) {
    std::lock_guard<std::mutex> lock(g_pin_mu);
    g_pin_free.push_back(p);
}

struct DeviceDfa {
    int device = 0;
    std::shared_ptr<const acg::Dfa> dfa;
    DevBuf<std::uint32_t> next, out_off, out_ids, depth;
    DevBuf<unsigned long long> outinfo;
    DevBuf<std::uint16_t> hot16, hotH, follows, follows_esc;
    DevBuf<std::uint8_t> symmap;
    DevBuf<std::uint32_t> qbloom;  // filter mode: kQWords Bloom words
    DevBuf<std::uint32_t> qbloom2;  // level-2 filter (large dictionaries)
    DevBuf<std::uint32_t> qtab, qb_off, qb_ent, pat_off;  // filter mode: exact q-gram table, patterns
    DevBuf<std::uint8_t> pat_bytes;
    DevBuf<unsigned long long> pat_code;  // filter mode: 2-bit codes of each pattern's first 64 bytes
    // output step (format_kernels.cuh): per pattern, its raw bytes [0] / JSON-escaped bytes [1]; built on first use
    std::mutex fmt_mu;
    DevBuf<std::uint8_t> fmt_str[2];
    DevBuf<unsigned long long> fmt_off[2];
    std::uint32_t hot_bytes = 0;   // exact table image: (H+1)*K u16, padded to 16
    std::uint32_t hotH_bytes = 0;  // truncated automaton: H*K u16, padded to 16 (sparse mode)
    DevBuf<std::uint16_t> hotG;    // generic alphabets: SPARSE-G truncated automaton (exact_kernels.cuh)
    std::uint32_t hotG_bytes = 0;
    // compressed hot automaton (ctab.hpp): shared-memory image, state words, id -> rank
    DevBuf<std::uint32_t> ctab, ct_next;
    DevBuf<std::uint16_t> ct_rank;
    DevBuf<unsigned long long> ct_info;  // event payload (id, or slots + rank) -> packed output info
    std::uint32_t ctab_bytes = 0;
    int smem_optin = 0;
    int num_sms = 0;
};

template <typename T>
cudaError_t upload(DevBuf<T>& dst, const T* src, std::size_t n, cudaStream_t st) {
    cudaError_t e = dst.reserve(n, st);
    if (e != cudaSuccess) return e;
    if (n) e = cudaMemcpyAsync(dst.p, src, n * sizeof(T), cudaMemcpyHostToDevice, st);
    return e;
}

}  // namespace

struct acg_automaton {
    acg::Nfa nfa;
    std::uint32_t hot_limit = 0;  // max shared-memory rows (0 = as many as fit)
    std::vector<std::uint64_t> profile;  // per NFA state visit counts on a sample (optional)
    mutable std::mutex mu;
    mutable std::map<int, std::shared_ptr<DeviceDfa>> dev;
    // host DFA (dense table, hot tables, CSR outputs), compiled by acg_build for
    // the sm_100 shared-memory budget; recompiled only if a layout knob changes
    mutable std::shared_ptr<acg::Dfa> dfa;
    mutable std::size_t dfa_budget = 0;
};

struct acg_result {
    std::vector<std::uint32_t> ids;
    std::vector<std::uint64_t> ends;
    std::vector<std::uint64_t> counts;
    std::uint64_t follows = 0;
};

struct acg_scanner {
    const acg_automaton* a = nullptr;
    int device = 0;
    std::uint32_t flags = 0;
    std::shared_ptr<DeviceDfa> dd;
    cudaStream_t stream = nullptr;       // own compute stream
    cudaStream_t last = nullptr;
    // workspace
    DevBuf<std::uint32_t> active_list, scalars32;
    DevBuf<unsigned long long> chunk_counts;  // scalars32[0] = active count
    DevBuf<unsigned long long> chunk_offs, visits, counts, records, scalars64;  // [0]=follows [1..3]=digest
    DevBuf<std::uint8_t> text;
    DevBuf<std::uint8_t> cub_tmp;
    DevBuf<std::uint8_t> fmt_out;                 // output step: formatted bytes of one window
    DevBuf<unsigned long long> fmt_tiles;         // per-tile byte sums, then offsets
    unsigned long long* pinned = nullptr;  // 8 host words
    cudaEvent_t order_ev = nullptr;        // orders a run on a new stream after the previous one
    // geometry of the last run
    acg::kern::ScanArgs args{};
    unsigned long long n_chunks = 0;
    unsigned long long chunk = 0;
    std::uint32_t launches = 0;
    unsigned grid = 0;
    bool have_run = false;
    bool synced = false;
    unsigned long long replays = 0;  // sync-time re-runs / re-emissions (an overflowed buffer was regrown)
    unsigned long long m_total = 0;
    // tuning
    std::uint32_t U = 0, tpb = acg::kern::kTPB;  // U = 0: per-mode default
    std::uint32_t U_run = 4;  // interleave of the last run
    std::uint32_t tpb_run = acg::kern::kTPB;
    bool tpb_set = false;  // block size fixed by acg_scanner_set_geometry
    unsigned long long chunk_override = 0;
    // last run's arguments (a sparse run whose task list overflowed is re-run at sync)
    const std::uint8_t* run_text = nullptr;
    std::uint64_t run_n = 0, run_emit = 0, run_base = 0;
    unsigned long long min_task_cap = 0;
    // mode: requested (ACG_MODE_*), used by the last run, and the event rate seen
    int mode_req = 0;
    int mode_run = 0;
    double last_event_rate = -1.0;
    double last_filter_rate = -1.0;  // filter mode: passing samples per text byte
    unsigned long long last_filter_max = 0, last_filter_n = 0;  // fullest survivor region, text size
    // filter mode: KQ survivors (count in scalars32[3]), V0 record scratch
    // (count in scalars64[5]), per-chunk fill counters, heavy chunks (count in scalars32[2])
    DevBuf<unsigned long long> qcands, qscratch;
    DevBuf<unsigned long long> qcand_win;
    DevBuf<std::uint32_t> qwarp_n;
    DevBuf<std::uint32_t> qfill, qheavy;
    bool regrow = false;  // enqueue_write after a record-buffer regrowth
    // filter mode region pipeline (V1 + ORDER): per-region counts, overflow
    // scalars; qlegacy = replay through the per-chunk pipeline (a region held
    // more matches than ORDER sorts); min_mcap = slab capacity after an overflow
    DevBuf<std::uint32_t> qreg_n, qscal;
    std::vector<std::pair<void*, std::size_t>> zeros;  // run-start zeroing (flush_zeros)
    bool qlegacy = false;
    std::uint32_t min_mcap = 0;
    std::uint32_t last_mcap = 0;
    unsigned long long task_regions = 0;  // sparse mode: fix-up task regions of the last run
    // exact mode: records per owned byte of the last exact run (-1 = unknown);
    // scratch_run = the last run used the single-pass slabs
    double exact_density = -1.0;
    unsigned long long exact_max = 0, exact_chunk = 0;  // largest chunk count of the last exact run, its chunk size
    unsigned long long exact_chunks = 0;                 // ... and its number of chunks
    DevBuf<unsigned long long> slab_size, slab_off;      // per-chunk slabs (sizes, prefix)
    bool scratch_run = false;
    bool hist_run = false;  // per-pattern counts by a histogram of the records (exact mode with a list)
    bool hist_fused = false;  // ... taken by the slab copy (+ K4 over the re-walked chunks' visits)
    DevBuf<unsigned long long> scratch;
    // exact mode, event pipeline (exact_kernels.cuh): event slabs + pool, per-chunk
    // event counts, per-chunk slab offsets, pool counter; the last event run's
    // geometry and totals size the next one's slabs
    DevBuf<std::uint32_t> xev, xev_count, xev_slab, xev_pool;
    DevBuf<std::uint32_t> gfin, gfin_count, gfin_pool;  // SPARSE-G: the fix-up's final events (chunk + 1 slots per chunk)
    bool g_run = false;                                  // the last run walked SPARSE-G
    bool c_run = false;                                  // the last run walked the compressed hot automaton (KC)
    bool kc_geom = false;                                // ... and its geometry (short chunks walked in rounds)
    std::uint32_t walk_pool_blocks = 0;                  // pool blocks of the last walk's event slabs
    acg::kern::EventArgs eargs{};
    acg::kern::CtabArgs cargs{};                         // KC's tables (E1/E2 map its event payloads)
    bool ev_run = false;
    unsigned long long xev_chunk = 0, xev_chunks = 0, xev_total = 0, xev_n = 0;
    std::uint32_t xev_min_pool = 0;
    DevBuf<std::uint32_t> events, ev_count, cands, cand_n, cand_list, cand_cnt, tasks, task_cnt;
    std::uint32_t ev_cap = 0;
    // optional per-kernel timing (ACG_SCAN_PROFILE)
    cudaEvent_t ev[6] = {};
    float kernel_ms[5] = {};
    std::uint32_t ev_mask = 0x3F;  // events recorded by the last profiled run
};

namespace {

std::size_t hot_budget(int smem_optin) {
    // dynamic smem = hot table + 256-byte symbol map; keep 1 KiB slack
    const long b = static_cast<long>(smem_optin) - 256 - 1024;
    return b > 0 ? static_cast<std::size_t>(b) : 0;
}

constexpr int kSm100SmemOptin = 232448;  // cudaDevAttrMaxSharedMemoryPerBlockOptin on B200 (227 KiB)

// The automaton's host DFA for a device's shared-memory budget (a->mu held).
std::shared_ptr<acg::Dfa> host_dfa_locked(const acg_automaton* a, int smem_optin) {
    std::size_t budget = hot_budget(smem_optin);
    const std::size_t full_budget = budget;
    if (a->hot_limit) budget = std::min<std::size_t>(budget, (a->hot_limit + 1ull) * 2ull * 256ull);
    if (!a->dfa || a->dfa_budget != budget) {
        auto dfa = std::make_shared<acg::Dfa>();
        acg::compile_dfa(a->nfa, budget, a->profile.empty() ? nullptr : &a->profile, *dfa, a->hot_limit, full_budget);
        a->dfa = std::move(dfa);
        a->dfa_budget = budget;
    }
    return a->dfa;
}

int get_device_dfa(const acg_automaton* a, int device, std::shared_ptr<DeviceDfa>* out) {
    std::lock_guard<std::mutex> lock(a->mu);
    auto it = a->dev.find(device);
    if (it != a->dev.end()) {
        *out = it->second;
        return ACG_OK;
    }
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= 0) {
        cudaGetLastError();
        return fail(ACG_ERR_NO_DEVICE, "no CUDA device available (libacg requires an sm_100 GPU)");
    }
    if (device < 0 || device >= count) return fail(ACG_ERR_NO_DEVICE, "device index out of range");
    ACG_CUDA(cudaSetDevice(device));
    auto dd = std::make_shared<DeviceDfa>();
    dd->device = device;
    ACG_CUDA(cudaDeviceGetAttribute(&dd->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    ACG_CUDA(cudaDeviceGetAttribute(&dd->num_sms, cudaDevAttrMultiProcessorCount, device));
    dd->dfa = host_dfa_locked(a, dd->smem_optin);
    const acg::Dfa& d = *dd->dfa;
    const cudaStream_t up = hk_stream(device);
    ACG_CUDA(upload(dd->next, d.next.data(), d.next.size(), up));
    ACG_CUDA(upload(dd->out_off, d.out_off.data(), d.out_off.size(), up));
    ACG_CUDA(upload(dd->out_ids, d.out_ids.data(), d.out_ids.size(), up));
    ACG_CUDA(upload(dd->outinfo, reinterpret_cast<const unsigned long long*>(d.outinfo.data()), d.outinfo.size(), up));
    ACG_CUDA(upload(dd->depth, d.depth.data(), d.depth.size(), up));
    ACG_CUDA(upload(dd->follows, d.follows.data(), d.follows.size(), up));
    ACG_CUDA(upload(dd->follows_esc, d.follows_esc.data(), d.follows_esc.size(), up));
    ACG_CUDA(upload(dd->symmap, d.symmap, 256, up));
    // shared-memory images padded to 16 bytes for vector staging
    dd->hot_bytes = static_cast<std::uint32_t>((d.hot16.size() * 2 + 15) & ~std::size_t(15));
    std::vector<std::uint16_t> hot(dd->hot_bytes / 2, 0xFFFF);
    std::copy(d.hot16.begin(), d.hot16.end(), hot.begin());
    ACG_CUDA(upload(dd->hot16, hot.data(), hot.size(), up));
    if (d.sparse_ok) {
        dd->hotH_bytes = static_cast<std::uint32_t>((d.hotH.size() * 2 + 15) & ~std::size_t(15));
        std::vector<std::uint16_t> hh(dd->hotH_bytes / 2, 0);
        std::copy(d.hotH.begin(), d.hotH.end(), hh.begin());
        ACG_CUDA(upload(dd->hotH, hh.data(), hh.size(), up));
    }
    if (!d.ctab.empty()) {
        dd->ctab_bytes = static_cast<std::uint32_t>((d.ctab.size() * 4 + 15) & ~std::size_t(15));
        std::vector<std::uint32_t> img(dd->ctab_bytes / 4, 0);
        std::copy(d.ctab.begin(), d.ctab.end(), img.begin());
        ACG_CUDA(upload(dd->ctab, img.data(), img.size(), up));
        ACG_CUDA(upload(dd->ct_next, d.ct_next.data(), d.ct_next.size(), up));
        ACG_CUDA(upload(dd->ct_rank, d.ct_rank.data(), d.ct_rank.size(), up));
        {
            const std::uint32_t n_out = d.Cn - d.Hn;
            std::vector<unsigned long long> pinfo(static_cast<std::size_t>(d.ct_slots) + n_out, 0ull);
            for (std::uint32_t i = 0; i < d.ct_slots; ++i)
                if (d.ct_rank[i] != acg::kCtNoRank) pinfo[i] = d.outinfo[d.Hn + d.ct_rank[i]];
            for (std::uint32_t r = 0; r < n_out; ++r) pinfo[d.ct_slots + r] = d.outinfo[d.Hn + r];
            ACG_CUDA(upload(dd->ct_info, pinfo.data(), pinfo.size(), up));
        }
    }
    if (!d.hotG.empty()) {
        dd->hotG_bytes = static_cast<std::uint32_t>((d.hotG.size() * 2 + 15) & ~std::size_t(15));
        std::vector<std::uint16_t> hg(dd->hotG_bytes / 2, 0);
        std::copy(d.hotG.begin(), d.hotG.end(), hg.begin());
        ACG_CUDA(upload(dd->hotG, hg.data(), hg.size(), up));
    }
    if (d.filter_ok) {
        ACG_CUDA(upload(dd->qbloom, d.qbloom.data(), d.qbloom.size(), up));
        if (!d.qbloom2.empty()) ACG_CUDA(upload(dd->qbloom2, d.qbloom2.data(), d.qbloom2.size(), up));
        ACG_CUDA(upload(dd->qtab, d.qtab.data(), d.qtab.size(), up));
        ACG_CUDA(upload(dd->qb_off, d.qb_off.data(), d.qb_off.size(), up));
        ACG_CUDA(upload(dd->qb_ent, d.qb_ent.data(), d.qb_ent.size(), up));
        ACG_CUDA(upload(dd->pat_off, d.pat_off32.data(), d.pat_off32.size(), up));
        ACG_CUDA(upload(dd->pat_bytes, a->nfa.pat_bytes.data(), a->nfa.pat_bytes.size(), up));
        ACG_CUDA(upload(dd->pat_code, reinterpret_cast<const unsigned long long*>(d.pat_code.data()), d.pat_code.size(), up));
    }
    ACG_CUDA(cudaStreamSynchronize(up));  // host staging vectors die here; buffers ready for any stream
    a->dev[device] = dd;
    *out = dd;
    return ACG_OK;
}

using acg::kern::ScanArgs;

std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, int> g_attr_smem;  // (kernel, device) -> configured opt-in smem

template <typename Kern>
cudaError_t prepare_smem(Kern k, std::size_t smem) {
    // opt-in smem limit, configured once per (kernel, device)
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_attr_mu);
    int& have = g_attr_smem[{reinterpret_cast<const void*>(k), dev}];
    if (have < static_cast<int>(smem)) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        have = static_cast<int>(smem);
    }
    return cudaSuccess;
}

template <int U, int MODE, int PASS, bool STATS>
cudaError_t launch_exact(const ScanArgs& args, unsigned grid, unsigned tpb, std::size_t smem, cudaStream_t st) {
    auto k = acg::kern::exact_scan_kernel<U, MODE, PASS, STATS>;
    if (cudaError_t e = prepare_smem(k, smem)) return e;
    k<<<grid, tpb, smem, st>>>(args);
    return cudaGetLastError();
}

template <int MODE, int PASS>
cudaError_t launch_exact_u(std::uint32_t U, const ScanArgs& args, unsigned grid, unsigned tpb, std::size_t smem,
                           cudaStream_t st) {
    switch (U) {
        case 1: return launch_exact<1, MODE, PASS, false>(args, grid, tpb, smem, st);
        case 2: return launch_exact<2, MODE, PASS, false>(args, grid, tpb, smem, st);
        case 8: return launch_exact<8, MODE, PASS, false>(args, grid, tpb, smem, st);
        default: return launch_exact<4, MODE, PASS, false>(args, grid, tpb, smem, st);
    }
}

cudaError_t launch_exact_pass(int alpha, int pass, bool stats, std::uint32_t U, const ScanArgs& args, unsigned grid,
                              unsigned tpb, std::size_t smem, cudaStream_t st) {
    using namespace acg::kern;
    if (stats)  // exact ScanStats: count pass only, interleave 2
        return alpha == acg::kAlphaDna4 ? launch_exact<2, 0, kCount, true>(args, grid, tpb, smem, st)
                                        : launch_exact<2, 1, kCount, true>(args, grid, tpb, smem, st);
    if (alpha == acg::kAlphaDna4)
        return pass == kCount   ? launch_exact_u<0, kCount>(U, args, grid, tpb, smem, st)
               : pass == kWrite ? launch_exact_u<0, kWrite>(U, args, grid, tpb, smem, st)
                                : launch_exact_u<0, kScratch>(U, args, grid, tpb, smem, st);
    return pass == kCount   ? launch_exact_u<1, kCount>(U, args, grid, tpb, smem, st)
           : pass == kWrite ? launch_exact_u<1, kWrite>(U, args, grid, tpb, smem, st)
                            : launch_exact_u<1, kScratch>(U, args, grid, tpb, smem, st);
}

template <int U, int MODE>
cudaError_t launch_event(const ScanArgs& a, const acg::kern::EventArgs& e, unsigned grid, unsigned tpb,
                         std::size_t smem, cudaStream_t st) {
    auto k = acg::kern::exact_event_kernel<U, MODE>;
    if (cudaError_t err = prepare_smem(k, smem)) return err;
    k<<<grid, tpb, smem, st>>>(a, e);
    return cudaGetLastError();
}

cudaError_t launch_event_walk(int alpha, std::uint32_t U, const ScanArgs& a, const acg::kern::EventArgs& e,
                              unsigned grid, unsigned tpb, std::size_t smem, cudaStream_t st) {
    if (alpha == acg::kAlphaDna4) {
        switch (U) {
            case 1: return launch_event<1, 0>(a, e, grid, tpb, smem, st);
            case 2: return launch_event<2, 0>(a, e, grid, tpb, smem, st);
            case 8: return launch_event<8, 0>(a, e, grid, tpb, smem, st);
            default: return launch_event<4, 0>(a, e, grid, tpb, smem, st);
        }
    }
    switch (U) {
        case 1: return launch_event<1, 1>(a, e, grid, tpb, smem, st);
        case 4: return launch_event<4, 1>(a, e, grid, tpb, smem, st);
        case 8: return launch_event<8, 1>(a, e, grid, tpb, smem, st);
        default: return launch_event<2, 1>(a, e, grid, tpb, smem, st);
    }
}

constexpr unsigned sparse_tpb(unsigned U) { return U == 1 ? 1024u : 512u; }

template <int U>
cudaError_t launch_sparse(const ScanArgs& args, unsigned grid, unsigned tpb, std::size_t smem, cudaStream_t st) {
    auto k = acg::kern::sparse_scan_kernel<U, (U <= 2 ? 4 : 2), sparse_tpb(U)>;
    if (cudaError_t e = prepare_smem(k, smem)) return e;
    k<<<grid, tpb, smem, st>>>(args);
    return cudaGetLastError();
}

// Sparse-mode fix-up: F1 re-walk (tasks), F2 excursion walks, F3 resolve.
unsigned fixup_rewalk_grid(unsigned long long bufs, int sms) {
    return static_cast<unsigned>(std::max<unsigned long long>(1, std::min<unsigned long long>((bufs + 31) / 32, sms)));
}
template <int U>
cudaError_t launch_fixup_u(const ScanArgs& args, std::size_t smem, int sms, cudaStream_t st) {
    using namespace acg::kern;
    const unsigned long long bufs = (args.n_chunks + 32ull * U - 1) / (32ull * U);
    const unsigned g1 = fixup_rewalk_grid(bufs, sms);
    {
        auto k = fixup_rewalk_kernel<U>;
        if (cudaError_t e = prepare_smem(k, smem)) return e;
        k<<<g1, 1024, smem, st>>>(args);
        if (cudaError_t e = cudaGetLastError()) return e;
    }
    {
        const unsigned g2 = std::max(1u, std::min<unsigned>(g1 * 32u * 2u / 8u, static_cast<unsigned>(sms) * 8u));
        fixup_walk_kernel<U><<<g2, 256, 0, st>>>(args, g1 * 32u);
        if (cudaError_t e = cudaGetLastError()) return e;
    }
    {
        auto k = fixup_resolve_kernel<U>;
        if (cudaError_t e = prepare_smem(k, smem)) return e;
        const unsigned g = static_cast<unsigned>(std::max<unsigned long long>(1, std::min<unsigned long long>((bufs + 15) / 16, sms)));
        k<<<g, 512, smem, st>>>(args);
        if (cudaError_t e = cudaGetLastError()) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_fixup(std::uint32_t U, const ScanArgs& args, std::size_t smem, int sms, cudaStream_t st) {
    switch (U) {
        case 1: return launch_fixup_u<1>(args, smem, sms, st);
        case 2: return launch_fixup_u<2>(args, smem, sms, st);
        default: return launch_fixup_u<4>(args, smem, sms, st);
    }
}

cudaError_t launch_sparse_u(std::uint32_t U, const ScanArgs& args, unsigned grid, unsigned tpb, std::size_t smem,
                            cudaStream_t st) {
    switch (U) {
        case 1: return launch_sparse<1>(args, grid, tpb, smem, st);
        case 2: return launch_sparse<2>(args, grid, tpb, smem, st);
        default: return launch_sparse<4>(args, grid, tpb, smem, st);
    }
}

std::size_t smem_bytes(const DeviceDfa& dd) { return dd.hot_bytes + 256; }
std::size_t smem_sparse(const DeviceDfa& dd) { return dd.hotH_bytes; }

constexpr unsigned long long kTaskBudget = 48ull << 30;
// sparse mode: walk offsets (halo + chunk) are 17-bit fields of the K1s events
// and F1 tasks; a chunk is at least kSparseMinChunk bytes
constexpr unsigned long long kSparseMaxWalk = 1ull << 17;
constexpr unsigned long long kSparseMinChunk = 256 + 64;
constexpr double kSparseMaxEventRate = 0.005;
constexpr std::uint32_t kHistMaxPatterns = 56 * 1024;  // record histogram: u32 bins in shared memory  // AUTO: sparse mode below this event rate
constexpr unsigned long long kEventBoundBudget = 16ull << 30;  // first-run event slabs at the 1-per-byte bound
constexpr unsigned long long kScratchBudget = 64ull << 30;  // exact-mode single-pass slabs (bytes)

// Slab budget: at most kScratchBudget and 60 % of the device memory free now
// (plus what the scanner's slabs already hold).
double scratch_budget(double held) {
    std::size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return static_cast<double>(kScratchBudget) / 4;
    }
    return std::min(static_cast<double>(kScratchBudget), 0.6 * static_cast<double>(free_b) + held);
}  // sparse fix-up task memory cap (bytes)

// KQ geometry: NW warps per SM, R blocks in flight per warp. ACG_QKERNEL
// picks another instantiation (experiments only).
struct QKernelChoice {
    int nw = 20, r = 2;  // 20 warps at 96 registers: cfg1 0.2311 -> 0.2276 ms/step, cfg2 3.15 -> 3.07 against 16 at 118
};
QKernelChoice qfilter_choice() {
    static const QKernelChoice c = [] {
        QKernelChoice q;
        const char* e = std::getenv("ACG_QKERNEL");
        if (e && std::strcmp(e, "16x3") == 0) q.nw = 16, q.r = 3;
        else if (e && std::strcmp(e, "24x2") == 0) q.nw = 24;
        else if (e && std::strcmp(e, "24x1") == 0) q.nw = 24, q.r = 1;
        else if (e && std::strcmp(e, "16x2") == 0) q.nw = 16;
        // the experimental pipelines (fused / post-confirm / bitmap level 1) exist at 16x2 only
        for (const char* sw : {"ACG_QFUSED", "ACG_QPOST", "ACG_QBITMAP"}) {
            const char* v = std::getenv(sw);
            if (v && v[0] == '1') q.nw = 16, q.r = 2;
        }
        return q;
    }();
    return c;
}
unsigned qfilter_warps() { return static_cast<unsigned>(qfilter_choice().nw); }
// Fused KQ (a consumer warp confirms survivors while the others stream; no
// V1 launch): region pipeline, 16x2 geometry; ACG_QFUSED=1 turns it on. Off by
// default: measured 0.294 ms against 0.226 + 0.028 (V1) unfused on cfg1 — the
// producers lose registers (96 at 544 threads) and the consumer issue slots.
// V1 inside KQ after the streaming loop (each CTA confirms its own warps'
// survivors): ACG_QPOST=1 (experiment).
bool qfilter_post(const ScanArgs& a) {
    static const bool on = [] {
        // off by default: measured 0.2558 ms/step on cfg1 against 0.2483 with the
        // separate V1 launch (512 threads per SM hide the confirmations' L2 latency
        // worse than V1's 2048, and the CTAs' streaming ends nearly together)
        const char* e = std::getenv("ACG_QPOST");
        return e && e[0] == '1';
    }();
    return on && a.reg_n;
}
bool qfilter_fused(const ScanArgs& a) {
    static const bool on = [] {
        const char* e = std::getenv("ACG_QFUSED");
        return e && e[0] == '1';
    }();
    const QKernelChoice c = qfilter_choice();
    return on && a.reg_n && c.nw == 16 && c.r == 2;
}
// Programmatic dependent launch: the kernel may be scheduled while the previous
// kernel on the stream drains (it waits for that grid's results with
// griddepcontrol.wait before reading them): hides launch latency between the
// filter pipeline's stages. ACG_PDL=0 launches plainly.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_smem(void (*k)(KArgs...), unsigned grid, unsigned threads, std::size_t smem, cudaStream_t st,
                            Args&&... args) {
    static const bool on = [] {
        const char* e = std::getenv("ACG_PDL");
        return !(e && e[0] == '0');
    }();
    if (!on) {
        k<<<grid, threads, smem, st>>>(std::forward<Args>(args)...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned threads, cudaStream_t st, Args&&... args) {
    return launch_pdl_smem(k, grid, threads, 0, st, std::forward<Args>(args)...);
}

template <typename Kern>
cudaError_t launch_q(Kern k, const ScanArgs& a, unsigned threads, std::size_t smem, int sms, cudaStream_t st) {
    cudaError_t e = prepare_smem(k, smem);
    if (e != cudaSuccess) return e;
    // programmatic: KQ stages its Bloom filter while the previous kernel drains
    return launch_pdl_smem(k, static_cast<unsigned>(sms), threads, smem, st, a);
}
cudaError_t launch_qfilter(const ScanArgs& a, int sms, cudaStream_t st) {
    using namespace acg::kern;
    const QKernelChoice c = qfilter_choice();
    const std::size_t bloom = static_cast<std::size_t>(a.qwords) * 4;
    if (qfilter_fused(a) && !a.qbm) {
        if (a.qbloom2) return launch_q(qfilter_ldg_kernel<16, 2, true, true>, a, 32 * 17, bloom, sms, st);
        return launch_q(qfilter_ldg_kernel<16, 2, false, true>, a, 32 * 17, bloom, sms, st);
    }
    if (qfilter_post(a)) {
        if (a.qbloom2) return launch_q(qfilter_ldg_kernel<16, 2, true, false, false, true>, a, 32 * 16, bloom, sms, st);
        if (a.qbm) return launch_q(qfilter_ldg_kernel<16, 2, false, false, true, true>, a, 32 * 16, bloom, sms, st);
        return launch_q(qfilter_ldg_kernel<16, 2, false, false, false, true>, a, 32 * 16, bloom, sms, st);
    }
    if (a.qbloom2 && c.nw == 24 && c.r == 1) return launch_q(qfilter_ldg_kernel<24, 1, true, false, false, false, 25>, a, 32 * 24, bloom, sms, st);
    if (a.qbloom2 && c.nw == 20) return launch_q(qfilter_ldg_kernel<20, 2, true, false, false, false, 25>, a, 32 * 20, bloom, sms, st);
    if (a.qbloom2) {
        static const int ldv = [] {  // ACG_Q2LD: level-2 probe load flavour (experiments)
            const char* e = std::getenv("ACG_Q2LD");
            return e ? std::atoi(e) : 25;  // .cg probes (no L1 allocation), L1::no_allocate text: cfg2 0.956 -> 0.80 ms per 2 GiB
        }();
        if (ldv == 0) return launch_q(qfilter_ldg_kernel<16, 2, true, false>, a, 32 * 16, bloom, sms, st);
        return launch_q(qfilter_ldg_kernel<16, 2, true, false, false, false, 25>, a, 32 * 16, bloom, sms, st);
    }
    if (a.qbm) return launch_q(qfilter_ldg_kernel<16, 2, false, false, true>, a, 32 * 16, bloom, sms, st);
    if (c.nw == 24) return launch_q(qfilter_ldg_kernel<24, 2, false, false>, a, 32 * 24, bloom, sms, st);
    if (c.r == 3) return launch_q(qfilter_ldg_kernel<16, 3, false, false>, a, 32 * 16, bloom, sms, st);
    {
        static const int tld = [] {  // ACG_QTLD: text load flavour (experiments)
            const char* e = std::getenv("ACG_QTLD");
            return e ? std::atoi(e) : 3;  // L1::no_allocate (cfg1 KQ 0.2188 -> 0.2166 ms against ld.global.cs)
        }();
        if (c.nw == 20) return launch_q(qfilter_ldg_kernel<20, 2, false, false, false, false, 24>, a, 32 * 20, bloom, sms, st);
        if (tld == 3) return launch_q(qfilter_ldg_kernel<16, 2, false, false, false, false, 24>, a, 32 * 16, bloom, sms, st);
    }
    return launch_q(qfilter_ldg_kernel<16, 2, false, false>, a, 32 * 16, bloom, sms, st);
}

// Enqueue K3 (compaction + ordered write) for the current geometry.
int enqueue_write(acg_scanner* s, cudaStream_t st) {
    using namespace acg::kern;
    const DeviceDfa& dd = *s->dd;
    ACG_CUDA(cudaMemsetAsync(s->scalars32.p, 0, sizeof(std::uint32_t), st));
    if (s->mode_run != ACG_MODE_FILTER && !s->scratch_run && !s->ev_run) {  // (filter mode sweeps the chunk offsets itself)
        const unsigned g = static_cast<unsigned>(std::min<unsigned long long>((s->n_chunks + 2047) / 2048, 1024ull));
        compact_active_kernel<<<std::max(g, 1u), 256, 0, st>>>(s->chunk_counts.p, static_cast<long long>(s->n_chunks),
                                                               s->active_list.p, s->scalars32.p);
        ACG_CUDA(cudaGetLastError());
        ++s->launches;
    }
    ScanArgs wa = s->args;
    const bool want_list = s->flags & ACG_SCAN_LIST;
    wa.records = want_list ? s->records.p : nullptr;
    wa.rec_cap = want_list ? s->records.n : 0;
    wa.visits = nullptr;  // both modes count visits in their count pass
    if (s->mode_run == ACG_MODE_FILTER && !s->qlegacy) {  // region pipeline: ORDER again (slabs are intact)
        ScanArgs oa = wa;
        const std::uint32_t W = static_cast<std::uint32_t>(s->n_chunks);
        acg::kern::qorder_region_kernel<<<(W + kQOrderWarps - 1) / kQOrderWarps, 32 * kQOrderWarps, 0, st>>>(
            oa, s->chunk_offs.p);
        ACG_CUDA(cudaGetLastError());
    } else if (s->mode_run == ACG_MODE_FILTER) {
        // records into their chunk's slots: from the scratch list, or (record
        // buffer regrown) by confirming the survivors again
        ACG_CUDA(cudaMemsetAsync(s->qfill.p, 0, s->n_chunks * sizeof(std::uint32_t), st));
        if (s->regrow) {
            acg::kern::qconfirm_kernel<kWrite><<<8 * dd.num_sms, 256, 0, st>>>(wa);
        } else {
            acg::kern::qscatter_kernel<<<4 * dd.num_sms, 256, 0, st>>>(wa);
        }
        ACG_CUDA(cudaGetLastError());
        ++s->launches;
        ACG_CUDA(s->qheavy.reserve(s->n_chunks, st));
        ACG_CUDA(cudaMemsetAsync(s->scalars32.p + 2, 0, sizeof(std::uint32_t), st));
        {
            const unsigned g = static_cast<unsigned>(std::max<unsigned long long>(
                1, std::min<unsigned long long>((s->n_chunks + 255) / 256, 8ull * dd.num_sms)));
            acg::kern::qsort_chunks_kernel<<<g, 256, 0, st>>>(wa, s->qheavy.p, s->scalars32.p + 2);
        }
        ACG_CUDA(cudaGetLastError());
        ++s->launches;
        auto k = acg::kern::qheavy_kernel;
        ACG_CUDA(prepare_smem(k, dd.hotH_bytes));
        k<<<dd.num_sms, 256, dd.hotH_bytes, st>>>(wa, s->qheavy.p, s->scalars32.p + 2);
        ACG_CUDA(cudaGetLastError());
    } else if (s->mode_run == ACG_MODE_SPARSE) {
        wa.visits = nullptr;  // counted with the candidates in the count pass
        auto k = acg::kern::sparse_emit_kernel;
        ACG_CUDA(prepare_smem(k, smem_sparse(dd)));
        const unsigned g = static_cast<unsigned>(std::max<unsigned long long>(
            1, std::min<unsigned long long>((s->n_chunks + 255) / 256, static_cast<unsigned long long>(dd.num_sms))));
        k<<<g, 256, smem_sparse(dd), st>>>(wa);
        ACG_CUDA(cudaGetLastError());
    } else if (s->ev_run) {
        // E2: events -> ordered records at each chunk's slot range
        const unsigned g = static_cast<unsigned>(
            std::max<unsigned long long>(1, std::min<unsigned long long>((s->n_chunks + 7) / 8, 16ull * dd.num_sms)));
        // KC counted the records itself (no E1): E2 also takes the visit histogram, once
        // (not when re-expanding after a record-buffer regrowth)
        const bool vis = s->cargs.counted && (s->flags & ACG_SCAN_COUNTS) && !s->regrow;
        if (vis) {
            wa.visits = s->visits.p;
            const std::size_t vb = static_cast<std::size_t>(s->eargs.n_out) * 4;
            static const unsigned vis_bps = [] {  // ACG_E2_VIS_BLOCKS: experiments
                const char* e = std::getenv("ACG_E2_VIS_BLOCKS");
                return e ? static_cast<unsigned>(std::atoi(e)) : 8u;  // (cfg3: 2 -> 2.55 ms, 4 -> 1.48, 6 -> 1.82, 8 -> 1.45)
            }();
            const unsigned gv = std::min<unsigned>(g, vis_bps * dd.num_sms);  // fewer blocks: each flushes its bins
            auto k = acg::kern::event_expand_kernel<true, true>;
            ACG_CUDA(prepare_smem(k, vb));
            k<<<gv, 256, vb, st>>>(wa, s->eargs, s->cargs);
        } else if (s->c_run) {
            acg::kern::event_expand_kernel<true, false><<<g, 256, 0, st>>>(wa, s->eargs, s->cargs);
        } else {
            acg::kern::event_expand_kernel<false, false><<<g, 256, 0, st>>>(wa, s->eargs, s->cargs);
        }
        ACG_CUDA(cudaGetLastError());
    } else if (s->scratch_run) {
        // slabs -> slot ranges; overflowed chunks are re-walked by the WRITE pass.
        // Per-pattern counts (not after a regrowth): histogram of what the copy
        // moves + the re-walked chunks' visits (K4)
        s->hist_fused = s->hist_run && !s->regrow;
        if (s->hist_fused) {
            const std::uint32_t P = s->a->nfa.n_patterns;
            ACG_CUDA(cudaMemsetAsync(s->counts.p, 0, P * sizeof(unsigned long long), st));
            auto k = acg::kern::scratch_copy_kernel<true>;
            const std::size_t smem = static_cast<std::size_t>(P) * 4;
            ACG_CUDA(prepare_smem(k, smem));
            k<<<2 * dd.num_sms, 1024, smem, st>>>(wa, s->active_list.p, s->scalars32.p, P, s->counts.p);
            wa.visits = s->visits.p;
        } else {
            const unsigned g = static_cast<unsigned>(
                std::max<unsigned long long>(1, std::min<unsigned long long>((s->n_chunks + 7) / 8, 16ull * dd.num_sms)));
            acg::kern::scratch_copy_kernel<false><<<g, 256, 0, st>>>(wa, s->active_list.p, s->scalars32.p, 0, nullptr);
        }
        ACG_CUDA(cudaGetLastError());
        ++s->launches;
        ACG_CUDA(launch_exact_pass(dd.dfa->mode, kWrite, false, s->U_run, wa, s->grid, s->tpb_run, smem_bytes(dd), st));
    } else {
        ACG_CUDA(launch_exact_pass(dd.dfa->mode, kWrite, false, s->U_run, wa, s->grid, s->tpb_run, smem_bytes(dd), st));
    }
    ++s->launches;
    if (s->hist_run && !s->hist_fused) {
        // per-pattern counts = histogram of the final record list (instead of
        // per-state visit atomics in the walk); re-run with the records after a regrowth
        const std::uint32_t P = s->a->nfa.n_patterns;
        ACG_CUDA(cudaMemsetAsync(s->counts.p, 0, P * sizeof(unsigned long long), st));
        auto k = acg::kern::record_hist_kernel;
        const std::size_t smem = static_cast<std::size_t>(P) * 4;
        ACG_CUDA(prepare_smem(k, smem));
        k<<<2 * dd.num_sms, 1024, smem, st>>>(s->records.p, s->chunk_offs.p + s->n_chunks, s->records.n, dd.dfa->id_bits, P,
                                               s->counts.p);
        ACG_CUDA(cudaGetLastError());
        ++s->launches;
    }
    return ACG_OK;
}

// Chunk geometry for owned bytes [emit_from, n): one chunk per stream, all
// streams of a full grid (one CTA per SM: the hot table takes the SM's smem).
constexpr unsigned long long kCtabChunk = 2048;  // KC: owned bytes per chunk (upper bound)

void plan_geometry(acg_scanner* s, std::uint64_t owned) {
    const DeviceDfa& dd = *s->dd;
    const unsigned long long streams = static_cast<unsigned long long>(dd.num_sms) * s->tpb_run * s->U_run;
    const unsigned long long halo = dd.dfa->halo;
    if (s->mode_run == ACG_MODE_FILTER && !s->qlegacy) {  // output regions = KQ warp regions
        const unsigned long long tw = static_cast<unsigned long long>(dd.num_sms) * qfilter_warps();
        const unsigned long long nb = (s->run_n + 2047) / 2048;
        s->chunk = std::max<unsigned long long>(1, (nb + tw - 1) / tw) * 2048;
        s->n_chunks = owned ? tw : 0;
        s->grid = static_cast<unsigned>(dd.num_sms);
        return;
    }
    if (s->mode_run == ACG_MODE_FILTER) {  // fixed 8 KiB chunks of 128 dirty-bit blocks
        s->chunk = static_cast<unsigned long long>(acg::kQChunkBlocks) * acg::kQBlock;
        s->n_chunks = (owned + s->chunk - 1) / s->chunk;
        s->grid = static_cast<unsigned>(dd.num_sms);
        return;
    }
    unsigned long long chunk = s->chunk_override;
    if (!chunk) {
        // KC walks short chunks in rounds (neighbouring lanes on neighbouring chunks):
        // the fewest full rounds with chunks of at most kCtabChunk bytes
        static const unsigned long long kc_env = [] {  // ACG_KC_CHUNK: experiments
            const char* e = std::getenv("ACG_KC_CHUNK");
            return e ? std::strtoull(e, nullptr, 10) : 0ull;
        }();
        const unsigned long long kc_chunk =
            std::max<unsigned long long>(kc_env ? kc_env : kCtabChunk, 32 * halo);  // warm-up <= 3 %
        const unsigned long long rounds =
            s->kc_geom ? std::max<unsigned long long>(1, (owned + streams * kc_chunk - 1) / (streams * kc_chunk)) : 1;
        chunk = (owned + streams * rounds - 1) / (streams * rounds);
        chunk = std::max<unsigned long long>(chunk, std::max<unsigned long long>(256, 2 * halo));
    }
    chunk = (chunk + 15) & ~15ull;
    if (s->kc_geom && !s->chunk_override) {
        static const unsigned long long kc_align = [] {  // ACG_KC_ALIGN: experiments
            const char* e = std::getenv("ACG_KC_ALIGN");
            return e ? std::strtoull(e, nullptr, 10) : 256ull;
        }();
        // chunks start on 256-byte boundaries: the text loads' L2 prefetch granule (cfg3: KC 4.27 -> 3.12 ms per 2 GiB)
        chunk = (chunk + kc_align - 1) / kc_align * kc_align;
    }
    // sparse mode: walk length (halo + chunk) a multiple of the 64-byte refill
    // (an explicit chunk override is kept as is: odd walks take the per-byte path)
    if (s->mode_run == ACG_MODE_SPARSE) {
        chunk = std::min<unsigned long long>(chunk, kSparseMaxWalk - halo - 64);  // event offsets are 17-bit
        if (!s->chunk_override) chunk = ((chunk + halo + 63) & ~63ull) - halo;
    }
    s->chunk = chunk;
    s->n_chunks = (owned + chunk - 1) / chunk;
    const unsigned long long per_block = static_cast<unsigned long long>(s->tpb_run) * s->U_run;
    s->grid = static_cast<unsigned>(std::max<unsigned long long>(1, (s->n_chunks + per_block - 1) / per_block));
}

// Run-start zeroing: counters and histograms to clear are collected and
// cleared by ONE kernel launch right before the run's first kernel (instead
// of a memset per buffer, each a separate GPU operation).
void zero_later(acg_scanner* s, void* p, std::size_t bytes) {
    if (p && bytes) s->zeros.push_back({p, bytes});
}
cudaError_t flush_zeros(acg_scanner* s, cudaStream_t st) {
    if (s->zeros.empty()) return cudaSuccess;
    acg::kern::ZeroList zl{};
    std::size_t i = 0;
    cudaError_t e = cudaSuccess;
    for (const auto& z : s->zeros) {
        if ((reinterpret_cast<std::uintptr_t>(z.first) | z.second) & 3) {  // not word-aligned: plain memset
            e = cudaMemsetAsync(z.first, 0, z.second, st);
            if (e != cudaSuccess) break;
            continue;
        }
        zl.ptr[i] = static_cast<std::uint32_t*>(z.first);
        zl.words[i] = z.second / 4;
        if (++i == acg::kern::ZeroList::kMax) {
            zl.n = static_cast<int>(i);
            e = launch_pdl(acg::kern::zero_regions_kernel, 128, 256, st, zl);
            if (e != cudaSuccess) return e;
            ++s->launches;
            i = 0;
        }
    }
    if (e == cudaSuccess && i) {
        zl.n = static_cast<int>(i);
        e = launch_pdl(acg::kern::zero_regions_kernel, 128, 256, st, zl);
        if (e != cudaSuccess) return e;
        ++s->launches;
    }
    s->zeros.clear();
    return e == cudaSuccess ? cudaGetLastError() : e;
}

// Work on `st` after everything this scanner enqueued before (possibly on
// another stream): its workspace is reused and may be regrown on `st`.
cudaError_t adopt_stream(acg_scanner* s, cudaStream_t st) {
    if (s->last && s->last != st) {
        cudaError_t e = cudaEventRecord(s->order_ev, s->last);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, s->order_ev, 0);
        if (e != cudaSuccess) return e;
    }
    s->last = st;
    return cudaSuccess;
}

// Event pipeline eligibility: an event packs the owned offset in its chunk and
// the output rank into 32 bits; the exact ScanStats walk keeps its own kernel.
// ACG_EXACT_EVENTS=0 keeps the inline-emission walk (experiments).
constexpr std::size_t kEventBinsMax = 200 * 1024;  // E1 visit bins in shared memory up to this
unsigned bits_for(unsigned long long v) {
    unsigned b = 1;
    while (b < 63 && (1ull << b) < v) ++b;
    return b;
}
bool event_slots_ok(const acg_scanner* s, std::uint32_t n_out, bool stats) {
    static const bool on = [] {
        const char* e = std::getenv("ACG_EXACT_EVENTS");
        return !(e && e[0] == '0');
    }();
    return on && !stats && n_out > 0 && bits_for(n_out) + bits_for(s->chunk) <= 32;
}

// SPARSE-G (generic alphabets, BFS hot set): ACG_SPARSEG=1 turns it on.
// Off by default: exact, but measured 3.32 ms per 256 MiB of cfg3 against 1.38
// for the KE walk — the walk logs an excursion event at ~every cold entry and
// the one-thread-per-chunk replay (XG) is a long dependent chain of text and
// L2 table loads (XG + E1 1.84 ms).
bool sparseg_ok(const acg_scanner* s, std::uint32_t n_out) {
    static const bool on = [] {
        const char* e = std::getenv("ACG_SPARSEG");
        return e && e[0] == '1';
    }();
    const DeviceDfa& dd = *s->dd;
    const acg::Dfa& d = *dd.dfa;
    return on && dd.hotG.p && dd.hotG_bytes + 256 <= static_cast<std::uint32_t>(dd.smem_optin) &&
           bits_for(n_out + d.H) + bits_for(s->chunk + d.halo) <= 32;
}

// KC (ctab.hpp): the compressed hot automaton walk; ACG_CTAB=0 keeps KE.
bool ctab_built(const acg_scanner* s) {
    static const bool on = [] {
        const char* e = std::getenv("ACG_CTAB");
        return !(e && e[0] == '0');
    }();
    const DeviceDfa& dd = *s->dd;
    return on && dd.ctab.p && dd.dfa->ct_slots && dd.ctab_bytes + 256 <= static_cast<std::uint32_t>(dd.smem_optin);
}
bool ctab_ok(const acg_scanner* s, std::uint32_t n_out) {
    return ctab_built(s) && bits_for(s->dd->dfa->ct_slots + n_out) + bits_for(s->chunk) <= 32;
}

template <int U, int D, bool DEEP, bool COLD>
cudaError_t launch_ctab(const ScanArgs& a, const acg::kern::EventArgs& e, const acg::kern::CtabArgs& ct, unsigned grid,
                        unsigned tpb, std::size_t smem, cudaStream_t st) {
    auto k = acg::kern::ctab_event_kernel<U, D, DEEP, COLD>;
    if (cudaError_t err = prepare_smem(k, smem)) return err;
    k<<<grid, tpb, smem, st>>>(a, e, ct);
    return cudaGetLastError();
}

// (instantiations: the all-hot deep walk only at D = 3, U <= 2 — cfg3's; the rest keep the cold branch)
template <int U, int D>
cudaError_t launch_ctab_v(bool deep, bool cold, const ScanArgs& a, const acg::kern::EventArgs& e,
                          const acg::kern::CtabArgs& ct, unsigned grid, unsigned tpb, std::size_t smem, cudaStream_t st) {
    if (deep) {
        if (D == 3 && U <= 2 && !cold) return launch_ctab<U, D, true, false>(a, e, ct, grid, tpb, smem, st);
        return launch_ctab<U, D, true, true>(a, e, ct, grid, tpb, smem, st);
    }
    return launch_ctab<U, D, false, true>(a, e, ct, grid, tpb, smem, st);
}

cudaError_t launch_ctab_walk(std::uint32_t U, std::uint32_t D, const ScanArgs& a, const acg::kern::EventArgs& e,
                             const acg::kern::CtabArgs& ct, unsigned grid, unsigned tpb, std::size_t smem,
                             cudaStream_t st) {
    const unsigned t2 = std::min(tpb, 512u);  // (one stream per thread: up to 1024 threads; 512 above)
    const bool deep = ct.deep, cold = ct.cold;
    if (D == 3) {
        switch (U) {
            case 1: return launch_ctab_v<1, 3>(deep, cold, a, e, ct, grid, tpb, smem, st);
            case 4: return launch_ctab_v<4, 3>(deep, cold, a, e, ct, grid, t2, smem, st);
            default: return launch_ctab_v<2, 3>(deep, cold, a, e, ct, grid, t2, smem, st);
        }
    }
    switch (U) {
        case 1: return launch_ctab_v<1, 2>(deep, cold, a, e, ct, grid, tpb, smem, st);
        case 4: return launch_ctab_v<4, 2>(deep, cold, a, e, ct, grid, t2, smem, st);
        default: return launch_ctab_v<2, 2>(deep, cold, a, e, ct, grid, t2, smem, st);
    }
}

template <int U>
cudaError_t launch_sparseg(const ScanArgs& a, const acg::kern::EventArgs& e, std::uint32_t n_out, unsigned grid,
                           unsigned tpb, std::size_t smem, cudaStream_t st) {
    auto k = acg::kern::sparseg_walk_kernel<U>;
    if (cudaError_t err = prepare_smem(k, smem)) return err;
    k<<<grid, tpb, smem, st>>>(a, e, n_out);
    return cudaGetLastError();
}
cudaError_t launch_sparseg_walk(std::uint32_t U, const ScanArgs& a, const acg::kern::EventArgs& e, std::uint32_t n_out,
                                unsigned grid, unsigned tpb, std::size_t smem, cudaStream_t st) {
    switch (U) {
        case 1: return launch_sparseg<1>(a, e, n_out, grid, tpb, smem, st);
        case 4: return launch_sparseg<4>(a, e, n_out, std::min(grid, grid), std::min(tpb, 512u), smem, st);
        default: return launch_sparseg<2>(a, e, n_out, grid, tpb, smem, st);
    }
}

// Event slabs for this run: per chunk from the previous event run's counts
// when the geometry repeats (exact + 1/8 + 17 slots), else uniform from its
// density (x 1.25 + 17; chunk/16 + 33 without history); overflow goes to the
// 256-event block pool (a pool overflow replays the run at sync).
cudaError_t plan_events(acg_scanner* s, std::uint32_t n_out, cudaStream_t st) {
    using acg::kern::kEvBlock;
    const unsigned long long nc = s->n_chunks, owned = s->run_n - s->run_emit;
    acg::kern::EventArgs& e = s->eargs;
    e = acg::kern::EventArgs{};
    const bool known = s->xev_n > 0;
    const bool same = known && s->xev_chunk == s->chunk && s->xev_chunks == nc && s->xev_n == owned;
    unsigned long long prim;
    cudaError_t err = s->xev_count.reserve(nc, st);
    if (err != cudaSuccess) return err;
    if (same) {
        if ((err = s->xev_slab.reserve(2 * (nc + 1), st)) != cudaSuccess) return err;
        std::uint32_t* sizes = s->xev_slab.p;
        std::uint32_t* offs = s->xev_slab.p + nc + 1;
        const unsigned g = static_cast<unsigned>(std::min<unsigned long long>((nc + 255) / 256, 8ull * s->dd->num_sms));
        acg::kern::event_slab_sizes_kernel<<<std::max(g, 1u), 256, 0, st>>>(s->xev_count.p, static_cast<long long>(nc),
                                                                         sizes, offs);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        std::size_t tmp = 0;
        cub::DeviceScan::InclusiveSum(nullptr, tmp, sizes, offs + 1, static_cast<int>(nc), st);
        if ((err = s->cub_tmp.reserve(std::max(tmp, s->cub_tmp.n), st)) != cudaSuccess) return err;
        tmp = s->cub_tmp.n;
        if ((err = cub::DeviceScan::InclusiveSum(s->cub_tmp.p, tmp, sizes, offs + 1, static_cast<int>(nc), st)) !=
            cudaSuccess)
            return err;
        prim = s->xev_total + s->xev_total / 8 + 17 * nc;  // >= the prefix's end
        e.slab_off = offs;
    } else {
        const double dens = known ? static_cast<double>(s->xev_total) / static_cast<double>(s->xev_n) : 1.0 / 16;
        unsigned long long cap = static_cast<unsigned long long>(1.25 * dens * static_cast<double>(s->chunk)) + 17;
        // a chunk logs at most one event per owned byte (one state per step, owned
        // blocks only): slabs of chunk + 1 slots never overflow. Without a density
        // from an earlier run, take that bound when it fits the budget (a first
        // run on dense output would otherwise chain thousands of pool blocks per
        // chunk through one global counter)
        if (!known) cap = (static_cast<double>(nc) * (s->chunk + 1) * 4.0 <= static_cast<double>(kEventBoundBudget))
                              ? s->chunk + 1
                              : s->chunk / 16 + 33;
        cap = std::min<unsigned long long>(cap, 0xFFFFFFFull);
        e.ecap = static_cast<std::uint32_t>(cap);
        prim = cap * nc;
    }
    unsigned long long pool = std::max<unsigned long long>(1024, (known ? prim / 4 : prim) / kEvBlock);
    pool = std::max<unsigned long long>(pool, s->xev_min_pool);
    if (prim + pool * kEvBlock >= 0xFFFFFFF0ull) {  // 32-bit slot indices: shrink the pool, keep it >= 1024 blocks
        if (prim + 1024ull * kEvBlock >= 0xFFFFFFF0ull) return cudaErrorInvalidValue;
        pool = (0xFFFFFFF0ull - prim) / kEvBlock;
    }
    if ((err = s->xev.reserve(prim + pool * kEvBlock, st)) != cudaSuccess) return err;
    if ((err = s->xev_pool.reserve(1, st)) != cudaSuccess) return err;
    e.ev = s->xev.p;
    e.ev_count = s->xev_count.p;
    e.pool_used = s->xev_pool.p;
    e.pool_base = static_cast<std::uint32_t>(prim);
    e.pool_blocks = static_cast<std::uint32_t>(pool);
    e.ob = bits_for(n_out);
    e.n_out = n_out;
    e.ev_total = s->scalars64.p + 8;
    return cudaSuccess;
}

int scanner_run(acg_scanner* s, const std::uint8_t* d_text, std::uint64_t n, std::uint64_t emit_from,
                std::uint64_t base, cudaStream_t st) {
    using namespace acg::kern;
    if (emit_from > n) return fail(ACG_ERR_INVALID, "emit_from beyond the text");
    if ((reinterpret_cast<std::uintptr_t>(d_text) & 15) || (emit_from & 15))
        return fail(ACG_ERR_INVALID, "device text and emit_from must be 16-byte aligned");
    ACG_CUDA(cudaSetDevice(s->device));
    ACG_CUDA(adopt_stream(s, st));
    const DeviceDfa& dd = *s->dd;
    const acg::Dfa& d = *dd.dfa;
    const bool want_list = s->flags & ACG_SCAN_LIST;
    const bool want_counts = s->flags & ACG_SCAN_COUNTS;
    const bool stats = s->flags & ACG_SCAN_STATS;
    s->launches = 0;
    s->hist_run = false;
    s->hist_fused = false;
    s->zeros.clear();
    s->scratch_run = false;
    s->ev_run = false;
    s->g_run = false;
    s->c_run = false;
    s->synced = false;
    s->last = st;
    s->run_text = d_text;
    s->run_n = n;
    s->run_emit = emit_from;
    s->run_base = base;
    const std::uint64_t owned = n - emit_from;
    // mode: sparse (truncated automaton + fix-up) when the automaton allows it
    // and excursions were rare on the previous run; exact otherwise
    int mode = s->mode_req;
    const bool filter_ok = d.filter_ok && d.sparse_ok;  // heavy chunks replay with A_H
    if (mode == ACG_MODE_FILTER && !filter_ok) mode = ACG_MODE_AUTO;
    if (mode == ACG_MODE_AUTO && filter_ok && (s->last_filter_rate < 0 || s->last_filter_rate < 1.0 / 256))
        mode = ACG_MODE_FILTER;
    // sparse mode's event log and fix-up tasks carry 17-bit walk offsets
    // (scan_kernels.cuh: K1s events, F1 tasks): walks of halo + chunk bytes must
    // fit, so a dictionary with a pattern longer than ~128 KiB runs EXACT
    const bool sparse_walk_ok = d.sparse_ok && static_cast<unsigned long long>(d.halo) + kSparseMinChunk <= kSparseMaxWalk;
    if (stats || (mode != ACG_MODE_FILTER && !sparse_walk_ok)) mode = ACG_MODE_EXACT;
    if (mode == ACG_MODE_AUTO)
        // measured on the BASELINE configs: sparse wins at 8.5e-4 events per walked
        // byte (cfg0: 3x faster than exact) and loses badly at 0.025 (cfg4) and
        // 0.0625 (cfg2: fix-up replay dominates). Without a measured rate, sparse
        // only when every state is hot (no excursions at all: cfg0); a first run of
        // sparse on a dense-output automaton (cfg4) is 19x slower than exact
        mode = ((s->last_event_rate < 0 && d.S <= d.H) ||
                (s->last_event_rate >= 0 && s->last_event_rate < kSparseMaxEventRate))
                   ? ACG_MODE_SPARSE
                   : ACG_MODE_EXACT;
    s->mode_run = mode;
    if (mode != ACG_MODE_EXACT) s->exact_chunks = 0;  // chunk_counts no longer hold an exact run's counts
    // default interleave: sparse 1; exact 4 on DNA, 2 on generic alphabets (cfg3
    // at 512 MiB: U=1 5.70 ms, U=2 4.87 ms, U=4 6.77 ms — cold-row L2 waits grow with U)
    // (the compressed-automaton walk KC is issue-bound, not latency-bound: one stream per thread)
    const bool kc_likely = mode == ACG_MODE_EXACT && !stats && ctab_built(s);
    s->U_run = stats ? 2u
                     : (s->U ? s->U
                             : (mode == ACG_MODE_SPARSE ? 1u : (d.mode == acg::kAlphaDna4 ? 4u : (kc_likely ? 1u : 2u))));
    if (mode == ACG_MODE_SPARSE && s->U_run > 4) s->U_run = 4;
    // exact mode at interleave <= 2 runs 1024 threads per SM (twice the warps to
    // hide cold-row L2 latency) unless the caller fixed the block size
    s->tpb_run = mode == ACG_MODE_SPARSE                ? sparse_tpb(s->U_run)
                 : (s->tpb_set || s->U_run > 2 || stats) ? s->tpb
                                                        : 2 * acg::kern::kTPB;
    if (mode != ACG_MODE_SPARSE && (s->U_run > 2 || stats))  // those kernels are bounded at kTPB threads
        s->tpb_run = std::min<std::uint32_t>(s->tpb_run, acg::kern::kTPB);
    s->kc_geom = kc_likely;
    if (kc_likely && s->U_run > 1) s->tpb_run = std::min<std::uint32_t>(s->tpb_run, acg::kern::kTPB);  // KC: 1024 threads at U = 1 only
    plan_geometry(s, owned);
    const bool prof = s->flags & ACG_SCAN_PROFILE;

    const std::uint32_t n_out_states = d.Cn - d.Hn;  // [Hn, Cn)
    ACG_CUDA(s->chunk_counts.reserve(s->n_chunks, st));
    ACG_CUDA(s->chunk_offs.reserve(s->n_chunks + 1, st));
    ACG_CUDA(s->active_list.reserve(s->n_chunks, st));
    ACG_CUDA(s->visits.reserve(n_out_states, st));
    ACG_CUDA(s->counts.reserve(d.out_ids.empty() ? 1 : s->a->nfa.n_patterns, st));
    if (!s->records.p) ACG_CUDA(s->records.reserve(1u << 20, st));
    std::size_t cub_bytes = 0;
    const unsigned long long* in_it = s->chunk_counts.p;
    cub::DeviceScan::InclusiveSum(nullptr, cub_bytes, in_it, s->chunk_offs.p + 1, static_cast<int>(std::max<unsigned long long>(s->n_chunks, 1)), st);
    ACG_CUDA(s->cub_tmp.reserve(cub_bytes, st));

    zero_later(s, s->scalars64.p, 5 * sizeof(unsigned long long));
    zero_later(s, s->chunk_offs.p, sizeof(unsigned long long));
    if (want_counts) {
        zero_later(s, s->visits.p, std::max<std::size_t>(n_out_states, 1) * sizeof(unsigned long long));
        zero_later(s, s->counts.p, s->a->nfa.n_patterns * sizeof(unsigned long long));
    }
    if (s->n_chunks == 0) {
        ACG_CUDA(flush_zeros(s, st));
        s->args = ScanArgs{};
        s->have_run = true;
        s->mode_run = mode;
        return ACG_OK;
    }

    ScanArgs& a = s->args;
    a = ScanArgs{};
    a.text = d_text;
    a.n = static_cast<long long>(n);
    a.emit_from = static_cast<long long>(emit_from);
    a.base = base;
    a.chunk = static_cast<long long>(s->chunk);
    a.halo = static_cast<long long>(d.halo);
    a.n_chunks = static_cast<long long>(s->n_chunks);
    a.next = dd.next.p;
    a.hot16 = dd.hot16.p;
    a.out_off = dd.out_off.p;
    a.out_ids = dd.out_ids.p;
    a.outinfo = dd.outinfo.p;
    a.depth = dd.depth.p;
    a.follows = dd.follows.p;
    a.follows_esc = dd.follows_esc.p;
    a.symmap = dd.symmap.p;
    a.K = d.K;
    a.H = d.H;
    a.Hn = d.Hn;
    a.Cn = d.Cn;
    a.smem_table_bytes = (mode == ACG_MODE_SPARSE || (mode == ACG_MODE_FILTER && d.sparse_ok)) ? dd.hotH_bytes : dd.hot_bytes;
    a.hotH = dd.hotH.p;
    a.chunk_counts = s->chunk_counts.p;
    a.active_list = s->active_list.p;
    a.active_count = s->scalars32.p;
    a.chunk_offs = s->chunk_offs.p;
    a.visits = want_counts ? s->visits.p : nullptr;
    a.records = s->records.p;
    a.rec_cap = s->records.n;
    a.id_bits = d.id_bits;
    a.follows_total = stats ? s->scalars64.p : nullptr;

    // K1: count pass
    if (prof) ACG_CUDA(cudaEventRecord(s->ev[0], st));
    s->ev_mask = 0x3F;
    if (mode == ACG_MODE_FILTER) {
        if (s->qlegacy) {
            zero_later(s, s->chunk_counts.p, s->n_chunks * sizeof(unsigned long long));
            ACG_CUDA(s->qfill.reserve(s->n_chunks, st));
        }
        a.qbloom = dd.qbloom.p;
        a.qtab = dd.qtab.p;
        a.qtab_bits = d.qtab_bits;
        a.qb_off = dd.qb_off.p;
        a.qb_ent = dd.qb_ent.p;
        a.pat_bytes = dd.pat_bytes.p;
        a.pat_off = dd.pat_off.p;
        a.q = d.q;
        a.qsh = d.q >= 16 ? 1u : 1u << (32 - 2 * d.q);
        a.max_len = d.max_len;
        a.pcounts = want_counts ? s->counts.p : nullptr;
        a.qfill = s->qfill.p;
        if (want_list && s->qlegacy) {
            ACG_CUDA(s->qscratch.reserve(s->records.n, st));
            a.qscratch = s->qscratch.p;
            a.qscratch_n = s->scalars64.p + 5;
            zero_later(s, s->scalars64.p + 5, sizeof(unsigned long long));
        }
        // survivors: one region per KQ consumer warp, sized from the previous run's
        // rate (x4 headroom over the even share); a full region is detected at sync
        // and the scan re-run with larger regions
        const unsigned warps_per_sm = qfilter_warps();
        const unsigned long long warps = static_cast<unsigned long long>(dd.num_sms) * warps_per_sm;
        // (after a run of the same size: 1.25 x its fullest region — V1 strides over
        // every slot, so slack costs it time)
        const double rate = s->last_filter_rate > 0 ? s->last_filter_rate : 1.0 / 4096;
        unsigned long long cap = static_cast<unsigned long long>(4.0 * rate * static_cast<double>(n) / warps) + 64;
        if (s->last_filter_max && s->last_filter_n == n)
            cap = std::min(cap, s->last_filter_max + s->last_filter_max / 4 + 32);
        cap = std::min<unsigned long long>(0x7FFFFFFFull / warps, std::max(cap, s->min_task_cap));
        ACG_CUDA(s->qcands.reserve(cap * warps, st));
        ACG_CUDA(s->qcand_win.reserve(cap * warps, st));
        ACG_CUDA(s->qwarp_n.reserve(warps, st));
        a.qcands = s->qcands.p;
        a.qcand_win = s->qcand_win.p;
        a.pat_code = dd.pat_code.p;
        a.qwarp_n = s->qwarp_n.p;
        a.qwarps = static_cast<std::uint32_t>(warps);
        a.qwords = static_cast<std::uint32_t>(d.qbloom.size());
        a.qbm = d.qbm ? 1u : 0u;
        a.qbloom2 = d.qbloom2.empty() ? nullptr : dd.qbloom2.p;
        a.qwords2 = static_cast<std::uint32_t>(d.qbloom2.size());
        a.qcand_cap = static_cast<std::uint32_t>(cap);
        a.qcand_n = s->scalars32.p + 3;
        a.qcand_max = s->scalars64.p + 6;
        zero_later(s, s->scalars32.p + 3, sizeof(std::uint32_t));
        zero_later(s, s->scalars64.p + 6, sizeof(unsigned long long));
        zero_later(s, s->qwarp_n.p, warps * sizeof(std::uint32_t));
        if (!s->qlegacy) {  // region pipeline: KQ -> V1 -> ORDER
            const std::uint32_t W = static_cast<std::uint32_t>(s->n_chunks);
            const std::uint32_t mcap = std::max<std::uint32_t>(64, s->min_mcap);
            s->last_mcap = mcap;
            ACG_CUDA(s->qscratch.reserve(static_cast<std::size_t>(W) * mcap, st));
            ACG_CUDA(s->qreg_n.reserve(std::max<unsigned long long>(W, warps), st));  // (KQ warps past the last region touch nothing)
            ACG_CUDA(s->qscal.reserve(2, st));
            zero_later(s, s->qscal.p, 2 * sizeof(std::uint32_t));
            a.qscratch = s->qscratch.p;
            a.mcap = mcap;
            a.qreg = static_cast<long long>(s->chunk);
            a.reg_n = s->qreg_n.p;
            a.qscal = s->qscal.p;
            if ((qfilter_fused(a) && !a.qbm) || qfilter_post(a)) {  // V1 runs inside KQ: its region counters start at zero
                zero_later(s, s->qreg_n.p, W * sizeof(std::uint32_t));
                ACG_CUDA(flush_zeros(s, st));
                ACG_CUDA(launch_qfilter(a, dd.num_sms, st));
                if (prof) ACG_CUDA(cudaEventRecord(s->ev[1], st));
            } else {
                ACG_CUDA(flush_zeros(s, st));
                ACG_CUDA(launch_qfilter(a, dd.num_sms, st));
                if (prof) ACG_CUDA(cudaEventRecord(s->ev[1], st));
                static const unsigned v1_ctas = [] {  // CTAs per SM (ACG_V1_CTAS: experiments)
                    const char* e = std::getenv("ACG_V1_CTAS");
                    const int v = e ? std::atoi(e) : 0;
                    return v > 0 && v <= 64 ? static_cast<unsigned>(v) : 16u;  // (r02: 16 -> V1 20.5 us vs 24 at 8)
                }();
                static const int v1_form = [] {  // ACG_V1_FORM=0: the slot-strided kernel
                    const char* e = std::getenv("ACG_V1_FORM");
                    return e ? std::atoi(e) : 1;
                }();
                if (v1_form == 0) ACG_CUDA(launch_pdl(qconfirm_region_kernel, v1_ctas * dd.num_sms, 256, st, a));
                else ACG_CUDA(launch_pdl(qconfirm_cta_kernel, a.qwarps, v1_form == 2 ? 128 : 256, st, a));
            }
            if (prof) ACG_CUDA(cudaEventRecord(s->ev[2], st));
            ScanArgs oa = a;
            oa.records = want_list ? s->records.p : nullptr;
            oa.rec_cap = want_list ? s->records.n : 0;
            ACG_CUDA(launch_pdl(qorder_region_kernel, (W + kQOrderWarps - 1) / kQOrderWarps, 32 * kQOrderWarps, st, oa,
                                s->chunk_offs.p));
            if (prof) ACG_CUDA(cudaEventRecord(s->ev[5], st));
            s->ev_mask = 0x27;  // events 0, 1, 2, 5 (stages KQ, V1, ORDER)
            s->launches += 3;
            s->have_run = true;
            return ACG_OK;
        }
        ACG_CUDA(flush_zeros(s, st));
        ACG_CUDA(launch_qfilter(a, dd.num_sms, st));
        ++s->launches;
        if (prof) ACG_CUDA(cudaEventRecord(s->ev[1], st));
        qconfirm_kernel<kCount><<<8 * dd.num_sms, 256, 0, st>>>(a);
        ACG_CUDA(cudaGetLastError());
        ++s->launches;
    } else if (mode == ACG_MODE_SPARSE) {
        // per K1s warp: one 16-byte event per flagged (block, stream) -> no overflow
        const unsigned long long walk = s->chunk + d.halo;
        const unsigned long long per_warp = 32ull * s->U_run;
        const unsigned long long n_warps = (s->n_chunks + per_warp - 1) / per_warp;
        s->ev_cap = static_cast<std::uint32_t>(per_warp * (walk / 16));
        ACG_CUDA(s->events.reserve(n_warps * s->ev_cap * 4ull, st));
        ACG_CUDA(s->ev_count.reserve(n_warps, st));
        ACG_CUDA(s->cands.reserve(s->n_chunks * acg::kern::kExport * 4ull, st));
        ACG_CUDA(s->cand_n.reserve(s->n_chunks, st));
        ACG_CUDA(s->cand_list.reserve(n_warps * acg::kern::kCandList * 2ull, st));
        ACG_CUDA(s->cand_cnt.reserve(n_warps, st));
        zero_later(s, s->cand_cnt.p, n_warps * sizeof(std::uint32_t));
        a.cand_list = s->cand_list.p;
        a.cand_cnt = s->cand_cnt.p;
        // excursion tasks: one region per fix-up warp; sized from the previous run's event
        // rate with headroom (1 per 16 walked bytes at first); overflow re-runs at sync
        const unsigned long long walked = s->n_chunks * walk;
        const double rate = s->last_event_rate > 0 ? s->last_event_rate : 1.0 / 16;
        const unsigned long long regions = fixup_rewalk_grid(n_warps, dd.num_sms) * 32ull;
        s->task_regions = regions;
        unsigned long long rcap = static_cast<unsigned long long>(walked * std::min(1.0, rate * 3.0) / regions) + 1024;
        rcap = std::max(rcap, s->min_task_cap);
        rcap = std::min<unsigned long long>(rcap, 0x7FFFFFFFull);
        ACG_CUDA(s->tasks.reserve(regions * rcap * 4ull, st));
        ACG_CUDA(s->task_cnt.reserve(regions, st));
        a.tasks = s->tasks.p;
        a.task_cnt = s->task_cnt.p;
        a.task_max = s->scalars32.p + 1;
        a.task_cap = static_cast<std::uint32_t>(rcap);
        zero_later(s, s->scalars32.p + 1, sizeof(std::uint32_t));
        a.events = s->events.p;
        a.cands = s->cands.p;
        a.cand_n = s->cand_n.p;
        a.ev_count = s->ev_count.p;
        a.ev_cap = s->ev_cap;
        a.ev_total = s->scalars64.p + 4;
        ACG_CUDA(flush_zeros(s, st));
        ACG_CUDA(launch_sparse_u(s->U_run, a, s->grid, s->tpb_run, smem_sparse(dd), st));
        ++s->launches;
        if (prof) ACG_CUDA(cudaEventRecord(s->ev[1], st));
        ACG_CUDA(launch_fixup(s->U_run, a, smem_sparse(dd), dd.num_sms, st));
        s->launches += 3;
    } else if (event_slots_ok(s, n_out_states, stats)) {
        // event pipeline (exact_kernels.cuh): KE walk logs output visits, E1
        // counts records per chunk + visits, K2 prefix, E2 expands (enqueue_write)
        s->g_run = sparseg_ok(s, n_out_states);
        s->c_run = !s->g_run && ctab_ok(s, n_out_states);
        ACG_CUDA(plan_events(s, s->g_run ? n_out_states + d.H : n_out_states, st));
        acg::kern::CtabArgs& ct = s->cargs;
        ct = acg::kern::CtabArgs{};
        if (s->c_run) {  // event payloads are state-word values: ids, or slots + rank
            s->eargs.ob = bits_for(d.ct_slots + n_out_states);
            ct.image = dd.ctab.p;
            ct.image_bytes = dd.ctab_bytes;
            ct.slots = d.ct_slots;
            ct.next = dd.ct_next.p;
            ct.rank = dd.ct_rank.p;
            ct.info = dd.ct_info.p;
            ct.pay_mask = d.ct_cnt ? acg::kCtPayMask : acg::kCtValMask;
            // list scans of counted words skip E1 (bins of the visit histogram must fit E2's shared memory)
            ct.counted = d.ct_cnt && want_list && static_cast<std::size_t>(n_out_states) * 4 <= 96 * 1024;
            ct.deep = d.ct_deep;
            ct.cold = d.ct_hot < d.S;
        }
        s->walk_pool_blocks = s->eargs.pool_blocks;
        zero_later(s, s->xev_pool.p, sizeof(std::uint32_t));
        zero_later(s, s->scalars64.p + 8, sizeof(unsigned long long));
        zero_later(s, s->scalars64.p + 9, sizeof(unsigned long long));
        // KE strides chunks over the CTAs (exact_kernels.cuh): a full one-per-SM grid
        // whenever there are enough chunks, whatever the per-block rounding
        const unsigned g_ev = static_cast<unsigned>(std::max<unsigned long long>(
            s->grid, std::min<unsigned long long>(dd.num_sms, (s->n_chunks + s->U_run - 1) / s->U_run)));
        if (s->g_run) {
            // SPARSE-G: walk the truncated automaton (shared memory only), then replay
            // the excursions exactly into the final events E1/E2 take
            const unsigned long long ecap = s->chunk + 1;
            ACG_CUDA(s->gfin.reserve(ecap * s->n_chunks, st));
            ACG_CUDA(s->gfin_count.reserve(s->n_chunks, st));
            ACG_CUDA(s->gfin_pool.reserve(1, st));
            zero_later(s, s->gfin_pool.p, sizeof(std::uint32_t));
            ACG_CUDA(flush_zeros(s, st));
            acg::kern::EventArgs ew = s->eargs;
            acg::kern::EventArgs ef{};
            ef.ev = s->gfin.p;
            ef.ecap = static_cast<std::uint32_t>(ecap);
            ef.ev_count = s->gfin_count.p;
            ef.pool_used = s->gfin_pool.p;
            ef.pool_base = static_cast<std::uint32_t>(ecap * s->n_chunks);
            ef.pool_blocks = 0;
            ef.ob = bits_for(n_out_states);
            ef.n_out = n_out_states;
            ef.ev_total = s->scalars64.p + 9;
            ScanArgs ga = a;
            ga.hotH = dd.hotG.p;
            ga.smem_table_bytes = dd.hotG_bytes;
            ACG_CUDA(launch_sparseg_walk(s->U_run, ga, ew, n_out_states, g_ev, s->tpb_run, dd.hotG_bytes + 256, st));
            if (prof) ACG_CUDA(cudaEventRecord(s->ev[1], st));
            const unsigned gx = static_cast<unsigned>(
                std::max<unsigned long long>(1, std::min<unsigned long long>((s->n_chunks + 255) / 256, 64ull * dd.num_sms)));
            acg::kern::sparseg_fix_kernel<<<gx, 256, 0, st>>>(ga, ew, ef, n_out_states);
            ACG_CUDA(cudaGetLastError());
            s->eargs = ef;  // E1 / E2 (and a regrowth's re-expansion) read the final events
            s->launches += 2;
        } else if (s->c_run) {
            ACG_CUDA(flush_zeros(s, st));
            const unsigned g_kc = static_cast<unsigned>(std::min<unsigned long long>(dd.num_sms, s->grid));  // rounds
            ACG_CUDA(launch_ctab_walk(s->U_run, d.ct_D, a, s->eargs, ct, g_kc, s->tpb_run, dd.ctab_bytes + 256, st));
            ++s->launches;
            if (prof) ACG_CUDA(cudaEventRecord(s->ev[1], st));
        } else {
            ACG_CUDA(flush_zeros(s, st));
            ACG_CUDA(launch_event_walk(d.mode, s->U_run, a, s->eargs, g_ev, s->tpb_run, smem_bytes(dd), st));
            ++s->launches;
            if (prof) ACG_CUDA(cudaEventRecord(s->ev[1], st));
        }
        s->ev_run = true;
        if (!(s->c_run && ct.counted)) {
        const std::size_t nb4 = static_cast<std::size_t>(n_out_states) * 4, nb1 = (n_out_states + 15u) & ~15u;
        const bool smem_bins = want_counts && nb4 <= kEventBinsMax;
        const bool smem_nout = (smem_bins ? nb4 : 0) + nb1 <= kEventBinsMax;
        const std::size_t xl_bytes = s->c_run ? static_cast<std::size_t>(d.ct_slots) * 2 : 0;
        // (the id -> rank table in shared memory only while two blocks still fit an SM;
        // otherwise through L1: it is read-only and mostly resident)
        const bool xl_smem = s->c_run && smem_nout && (smem_bins ? nb4 : 0) + nb1 + xl_bytes <= 100 * 1024;
        const std::size_t e1_smem = (smem_bins ? nb4 : 0) + (smem_nout ? nb1 : 0) + (xl_smem ? xl_bytes : 0);
        const unsigned g1 = static_cast<unsigned>(
            std::max<unsigned long long>(1, std::min<unsigned long long>((s->n_chunks + 15) / 16, 2ull * dd.num_sms)));
        auto e1 = [&](auto k) -> cudaError_t {
            if (cudaError_t err = prepare_smem(k, e1_smem)) return err;
            k<<<g1, 512, e1_smem, st>>>(a, s->eargs, ct, xl_smem);
            return cudaGetLastError();
        };
        if (s->c_run) {
            if (smem_bins && smem_nout) ACG_CUDA(e1(acg::kern::event_count_kernel<true, true, true>));
            else if (smem_bins) ACG_CUDA(e1(acg::kern::event_count_kernel<true, false, true>));
            else if (smem_nout) ACG_CUDA(e1(acg::kern::event_count_kernel<false, true, true>));
            else ACG_CUDA(e1(acg::kern::event_count_kernel<false, false, true>));
        } else if (smem_bins && smem_nout) ACG_CUDA(e1(acg::kern::event_count_kernel<true, true, false>));
        else if (smem_bins) ACG_CUDA(e1(acg::kern::event_count_kernel<true, false, false>));
        else if (smem_nout) ACG_CUDA(e1(acg::kern::event_count_kernel<false, true, false>));
        else ACG_CUDA(e1(acg::kern::event_count_kernel<false, false, false>));
        ACG_CUDA(cudaGetLastError());
        ++s->launches;
        }
    } else {
        // single pass (count + per-chunk slabs) once the previous run told the
        // record density and the slabs fit the budget; count + write otherwise
        // per-pattern counts from the written records when the list is produced
        // (the walk then issues no per-state visit atomics)
        s->hist_run = want_list && want_counts && s->a->nfa.n_patterns <= kHistMaxPatterns;
        if (s->hist_run) a.visits = nullptr;
        a.chunk_max = s->scalars64.p + 7;
        zero_later(s, s->scalars64.p + 7, sizeof(unsigned long long));
        // slabs sized chunk by chunk from the previous run's counts when it had the
        // same geometry (its counts are still in chunk_counts): total ~1.125 x its matches
        const double budget = scratch_budget(s->scratch.n * 8.0);
        const bool per_chunk = want_list && !stats && s->exact_chunk == s->chunk && s->exact_chunks == s->n_chunks &&
                               s->exact_density >= 0 &&
                               (1.125 * static_cast<double>(s->m_total) + 16.0 * s->n_chunks + 1) * 8.0 <= budget;
        ACG_CUDA(flush_zeros(s, st));
        if (per_chunk) {
            const unsigned long long cap = s->m_total + s->m_total / 8 + 16ull * s->n_chunks + 1;
            ACG_CUDA(s->scratch.reserve(cap, st));
            ACG_CUDA(s->slab_size.reserve(s->n_chunks + 1, st));
            ACG_CUDA(s->slab_off.reserve(s->n_chunks + 1, st));
            const unsigned g = static_cast<unsigned>(std::min<unsigned long long>((s->n_chunks + 255) / 256, 8ull * dd.num_sms));
            slab_sizes_kernel<<<std::max(g, 1u), 256, 0, st>>>(s->chunk_counts.p, static_cast<long long>(s->n_chunks),
                                                                s->slab_size.p);
            ACG_CUDA(cudaGetLastError());
            ACG_CUDA(cudaMemsetAsync(s->slab_off.p, 0, sizeof(unsigned long long), st));
            std::size_t tmp2 = s->cub_tmp.n;
            ACG_CUDA(cub::DeviceScan::InclusiveSum(s->cub_tmp.p, tmp2, s->slab_size.p + 1, s->slab_off.p + 1,
                                                   static_cast<int>(s->n_chunks), st));
            a.scratch = s->scratch.p;
            a.slab_off = s->slab_off.p;
            s->scratch_run = true;
        } else if (want_list && !stats && s->exact_density >= 0) {
            // slab = the larger of 1.25 x the mean and 1.1 x the largest chunk of the last run
            const double mean = s->exact_density * static_cast<double>(s->chunk);
            const double big = s->exact_chunk > 0 ? 1.1 * static_cast<double>(s->exact_max) *
                                                        static_cast<double>(s->chunk) / static_cast<double>(s->exact_chunk)
                                                  : 0.0;
            unsigned long long scap = static_cast<unsigned long long>(std::max(1.25 * mean, big)) + 32;
            if (static_cast<double>(scap) * s->n_chunks * 8.0 > budget)
                scap = static_cast<unsigned long long>(1.25 * mean) + 32;
            if (static_cast<double>(scap) * s->n_chunks * 8.0 <= budget) {
                ACG_CUDA(s->scratch.reserve(scap * s->n_chunks, st));
                a.scratch = s->scratch.p;
                a.scap = scap;
                s->scratch_run = true;
            }
        }
        ACG_CUDA(launch_exact_pass(d.mode, s->scratch_run ? kScratch : kCount, stats, s->U_run, a, s->grid, s->tpb_run,
                                   smem_bytes(dd), st));
        ++s->launches;
        if (prof) ACG_CUDA(cudaEventRecord(s->ev[1], st));
    }
    if (prof) ACG_CUDA(cudaEventRecord(s->ev[2], st));
    // K2: record slots = inclusive prefix of the chunk counts, shifted by one (CUB, not counted in launches)
    std::size_t tmp = s->cub_tmp.n;
    ACG_CUDA(cub::DeviceScan::InclusiveSum(s->cub_tmp.p, tmp, in_it, s->chunk_offs.p + 1,
                                           static_cast<int>(s->n_chunks), st));
    if (prof) ACG_CUDA(cudaEventRecord(s->ev[3], st));
    // K3: ordered records
    if (want_list) {
        const int rc = enqueue_write(s, st);
        if (rc) return rc;
    }
    if (prof) ACG_CUDA(cudaEventRecord(s->ev[4], st));
    // K4: per-pattern counts
    if (want_counts && n_out_states && mode != ACG_MODE_FILTER && (!s->hist_run || s->hist_fused)) {
        const unsigned tb = 256;
        const unsigned g = std::min<unsigned>((n_out_states + tb - 1) / tb, 8 * dd.num_sms);
        pattern_counts_kernel<<<g, tb, 0, st>>>(s->visits.p, dd.out_off.p, dd.out_ids.p, d.Hn, d.H, d.Cn, d.S,
                                                s->counts.p);
        ACG_CUDA(cudaGetLastError());
        ++s->launches;
    }
    if (prof) ACG_CUDA(cudaEventRecord(s->ev[5], st));
    s->have_run = true;
    return ACG_OK;
}

int scanner_sync(acg_scanner* s) {
    if (!s->have_run) return fail(ACG_ERR_INVALID, "no scan has been run");
    if (s->synced) return ACG_OK;
    ACG_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = s->last;
    ACG_CUDA(cudaMemcpyAsync(s->pinned, s->chunk_offs.p + s->n_chunks, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, st));
    ACG_CUDA(cudaMemcpyAsync(s->pinned + 5, s->scalars64.p + 4, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             st));
    ACG_CUDA(cudaMemcpyAsync(s->pinned + 6, s->scalars32.p, 4 * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, st));
    if (s->mode_run == ACG_MODE_FILTER)
        ACG_CUDA(cudaMemcpyAsync(s->pinned + 4, s->scalars64.p + 6, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    ACG_CUDA(cudaStreamSynchronize(st));
    if (s->mode_run == ACG_MODE_SPARSE && s->n_chunks) {
        const std::uint32_t ntask = reinterpret_cast<const std::uint32_t*>(s->pinned + 6)[1];
        if (ntask > s->args.task_cap) {  // a task region overflowed: grow and run again
            s->min_task_cap = ntask + ntask / 4 + 1024;
            // excursions this frequent make the exact walk the better mode; it
            // also needs no task memory (which would be regions x the worst
            // region's tasks): re-run exactly instead of growing past a budget
            const double need = static_cast<double>(s->task_regions) * s->min_task_cap * 16.0;
            const bool go_exact = need > static_cast<double>(kTaskBudget);
            const int req = s->mode_req;
            s->mode_req = go_exact ? ACG_MODE_EXACT : ACG_MODE_SPARSE;
            if (go_exact) {
                s->min_task_cap = 0;
                s->last_event_rate = 1.0;  // AUTO: exact from now on
            }
            ++s->replays;
            const int rc = scanner_run(s, s->run_text, s->run_n, s->run_emit, s->run_base, st);
            s->mode_req = req;
            if (rc) return rc;
            return scanner_sync(s);
        }
    }
    if (s->mode_run == ACG_MODE_FILTER && s->n_chunks && !s->qlegacy) {
        ACG_CUDA(cudaMemcpyAsync(s->pinned + 1, s->qscal.p, 2 * sizeof(std::uint32_t), cudaMemcpyDeviceToHost, st));
        ACG_CUDA(cudaStreamSynchronize(st));
        const std::uint32_t* qs = reinterpret_cast<const std::uint32_t*>(s->pinned + 1);
        const std::uint32_t slab_max = qs[0], too_big = qs[1];
        if (g_debug)
            std::fprintf(stderr, "[acg] filter region run: survivors max %llu cap %u slab_max %u mcap %u too_big %u\n",
                         s->pinned[4], s->args.qcand_cap, slab_max, s->last_mcap, too_big);
        if (s->pinned[4] <= s->args.qcand_cap && (slab_max > s->last_mcap || too_big)) {
            // a region's slab overflowed (grow it) or held more than ORDER sorts
            // (replay through the per-chunk pipeline from now on): run again
            if (too_big) s->qlegacy = true;
            else s->min_mcap = slab_max + slab_max / 4 + 32;
            const int req = s->mode_req;
            s->mode_req = ACG_MODE_FILTER;
            ++s->replays;
            const int rc = scanner_run(s, s->run_text, s->run_n, s->run_emit, s->run_base, st);
            s->mode_req = req;
            if (rc) return rc;
            return scanner_sync(s);
        }
    }
    if (s->mode_run == ACG_MODE_FILTER && s->n_chunks) {
        const unsigned long long worst = s->pinned[4];
        if (g_debug) {
            std::fprintf(stderr, "[acg] filter run (legacy %d): survivors max %llu cap %u chunks %llu matches %llu records %zu\n",
                         s->qlegacy ? 1 : 0, worst, s->args.qcand_cap, s->n_chunks, s->pinned[0], s->records.n);
            if (s->qlegacy && worst <= s->args.qcand_cap) {  // survivor sanity: duplicates, out-of-region positions
                const std::size_t W = s->args.qwarps, cap = s->args.qcand_cap;
                std::vector<std::uint32_t> wn(W);
                std::vector<unsigned long long> qc(W * cap), cc(s->n_chunks);
                cudaMemcpy(wn.data(), s->qwarp_n.p, W * 4, cudaMemcpyDeviceToHost);
                cudaMemcpy(qc.data(), s->qcands.p, W * cap * 8, cudaMemcpyDeviceToHost);
                cudaMemcpy(cc.data(), s->chunk_counts.p, s->n_chunks * 8, cudaMemcpyDeviceToHost);
                std::vector<unsigned long long> all;
                unsigned long long bad = 0;
                const unsigned long long nb = (s->run_n + 2047) / 2048, per = (nb + W - 1) / W;
                for (std::size_t w = 0; w < W; ++w)
                    for (std::size_t k = 0; k < wn[w]; ++k) {
                        const unsigned long long pos = qc[w * cap + k];
                        all.push_back(pos);
                        if (pos / 2048 < w * per || pos / 2048 >= (w + 1) * per) ++bad;
                    }
                std::sort(all.begin(), all.end());
                unsigned long long dups = 0;
                for (std::size_t i = 1; i < all.size(); ++i) dups += all[i] == all[i - 1];
                unsigned long long sum = 0, mx = 0, arg = 0;
                for (std::size_t c = 0; c < cc.size(); ++c) {
                    sum += cc[c];
                    if (cc[c] > mx) mx = cc[c], arg = c;
                }
                std::fprintf(stderr, "[acg]   survivors %zu dups %llu out-of-region %llu; chunk counts sum %llu max %llu at %llu\n",
                             all.size(), dups, bad, sum, mx, arg);
            }
        }
        if (worst > s->args.qcand_cap) {  // a survivor region overflowed: grow and run again
            s->min_task_cap = worst + worst / 4 + 64;
            const int req = s->mode_req;
            s->mode_req = ACG_MODE_FILTER;
            ++s->replays;
            const int rc = scanner_run(s, s->run_text, s->run_n, s->run_emit, s->run_base, st);
            s->mode_req = req;
            if (rc) return rc;
            return scanner_sync(s);
        }
    }
    if (s->ev_run && s->n_chunks) {
        ACG_CUDA(cudaMemcpyAsync(s->pinned + 1, s->xev_pool.p, sizeof(std::uint32_t), cudaMemcpyDeviceToHost, st));
        ACG_CUDA(cudaMemcpyAsync(s->pinned + 2, s->scalars64.p + 8, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        ACG_CUDA(cudaStreamSynchronize(st));
        const std::uint32_t used = static_cast<std::uint32_t>(s->pinned[1]);
        if (used > s->walk_pool_blocks) {  // the walk's event pool overflowed: grow it and run again
            s->xev_min_pool = used + used / 4 + 1024;
            s->xev_n = 0;  // (no valid counts from this run: uniform slabs)
            ++s->replays;
            const int rc = scanner_run(s, s->run_text, s->run_n, s->run_emit, s->run_base, st);
            if (rc) return rc;
            return scanner_sync(s);
        }
        s->xev_total = s->pinned[2];
        s->xev_chunk = s->chunk;
        s->xev_chunks = s->n_chunks;
        s->xev_n = s->run_n - s->run_emit;
    }
    s->m_total = s->n_chunks ? s->pinned[0] : 0;
    if (s->mode_run == ACG_MODE_EXACT && !s->ev_run && s->run_n > s->run_emit) {
        if (g_debug) {
            const std::uint32_t over = reinterpret_cast<const std::uint32_t*>(s->pinned + 6)[0];
            std::fprintf(stderr, "[acg] exact run: scratch %d per_chunk %d scap %llu chunks %llu matches %llu overflowed %u\n",
                         s->scratch_run ? 1 : 0, s->args.slab_off ? 1 : 0, s->args.scap, s->n_chunks, s->m_total, over);
        }
        s->exact_density = static_cast<double>(s->m_total) / static_cast<double>(s->run_n - s->run_emit);
        ACG_CUDA(cudaMemcpyAsync(s->pinned + 1, s->scalars64.p + 7, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        ACG_CUDA(cudaStreamSynchronize(st));
        s->exact_max = s->pinned[1];
        s->exact_chunk = s->chunk;
        s->exact_chunks = s->n_chunks;
    }
    if (s->mode_run == ACG_MODE_FILTER && s->run_n) {
        s->last_filter_rate = static_cast<double>(reinterpret_cast<const std::uint32_t*>(s->pinned + 6)[3]) /
                              static_cast<double>(s->run_n);
        s->last_filter_max = s->pinned[4];
        s->last_filter_n = s->run_n;
    }
    if (s->mode_run == ACG_MODE_SPARSE && s->n_chunks) {
        const double walked = static_cast<double>(s->n_chunks) * static_cast<double>(s->chunk + s->dd->dfa->halo);
        s->last_event_rate = static_cast<double>(s->pinned[5]) / walked;
    }
    if ((s->flags & ACG_SCAN_LIST) && s->m_total > s->records.n) {
        // record buffer overflowed: grow and re-emit (chunk counts and offsets are final)
        ACG_CUDA(s->records.reserve(s->m_total + s->m_total / 4, st));
        ++s->replays;
        s->regrow = true;
        const int rc = enqueue_write(s, st);
        s->regrow = false;
        if (rc) return rc;
        ACG_CUDA(cudaStreamSynchronize(st));
    }
    if ((s->flags & ACG_SCAN_PROFILE) && s->n_chunks) {
        // stage i-1 = time from the previous recorded event to event i
        int prev = 0;
        for (int i = 1; i < 6; ++i) {
            s->kernel_ms[i - 1] = 0.f;
            if (!(s->ev_mask >> i & 1)) continue;
            ACG_CUDA(cudaEventElapsedTime(&s->kernel_ms[i - 1], s->ev[prev], s->ev[i]));
            prev = i;
        }
    }
    s->synced = true;
    return ACG_OK;
}

int make_scanner(const acg_automaton* a, int device, std::uint32_t flags, acg_scanner** out) {
    auto s = std::make_unique<acg_scanner>();
    s->a = a;
    s->device = device;
    s->flags = flags;
    if (const int rc = get_device_dfa(a, device, &s->dd)) return rc;
    ACG_CUDA(cudaSetDevice(device));
    ACG_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    s->pinned = pinned_take();
    if (!s->pinned) return fail(ACG_ERR_OUT_OF_MEMORY, "pinned host allocation failed");
    ACG_CUDA(cudaEventCreateWithFlags(&s->order_ev, cudaEventDisableTiming));
    ACG_CUDA(s->scalars32.reserve(4, s->stream));
    ACG_CUDA(s->scalars64.reserve(10, s->stream));  // [8] = events of the last event-pipeline run
    ACG_CUDA(cudaMemsetAsync(s->scalars64.p, 0, 10 * sizeof(unsigned long long), s->stream));
    s->last = s->stream;
    if (flags & ACG_SCAN_PROFILE)
        for (auto& e : s->ev) ACG_CUDA(cudaEventCreate(&e));
    *out = s.release();
    return ACG_OK;
}

void free_scanner(acg_scanner* s) {
    if (!s) return;
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    if (s->last) cudaStreamSynchronize(s->last);
    if (s->stream) cudaStreamDestroy(s->stream);
    if (s->pinned) pinned_give(s->pinned);
    if (s->order_ev) cudaEventDestroy(s->order_ev);
    for (auto& e : s->ev)
        if (e) cudaEventDestroy(e);
    delete s;
}

// Scanner pool per automaton for the one-shot acg_scan (keeps device
// workspace across calls; one scanner per concurrent caller).
struct PoolKey {
    const acg_automaton* a;
    int device;
    std::uint32_t flags;
    bool operator<(const PoolKey& o) const {
        if (a != o.a) return a < o.a;
        if (device != o.device) return device < o.device;
        return flags < o.flags;
    }
};
std::mutex g_pool_mu;
std::map<PoolKey, std::vector<acg_scanner*>> g_pool;

acg_scanner* pool_take(const acg_automaton* a, int device, std::uint32_t flags) {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    auto& v = g_pool[PoolKey{a, device, flags}];
    if (v.empty()) return nullptr;
    acg_scanner* s = v.back();
    v.pop_back();
    return s;
}
void pool_give(acg_scanner* s) {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    auto& v = g_pool[PoolKey{s->a, s->device, s->flags}];
    if (v.size() < 8) v.push_back(s);
    else free_scanner(s);
}
void pool_drop(const acg_automaton* a) {
    std::vector<acg_scanner*> dead;
    {
        std::lock_guard<std::mutex> lock(g_pool_mu);
        for (auto it = g_pool.begin(); it != g_pool.end();) {
            if (it->first.a == a) {
                dead.insert(dead.end(), it->second.begin(), it->second.end());
                it = g_pool.erase(it);
            } else {
                ++it;
            }
        }
    }
    for (acg_scanner* s : dead) free_scanner(s);
}

int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return d;
}

void warm_up_device(int device) {
    using namespace acg::kern;
    if (cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) return;
    cudaFuncAttributes fa;
    auto load = [&](const void* k) { (void)cudaFuncGetAttributes(&fa, k); };
    // generic alphabets (exact mode) and DNA (sparse / exact / filter)
    load(reinterpret_cast<const void*>(exact_scan_kernel<2, 1, kCount, false>));
    load(reinterpret_cast<const void*>(exact_scan_kernel<2, 1, kWrite, false>));
    load(reinterpret_cast<const void*>(exact_scan_kernel<2, 1, kCount, true>));
    load(reinterpret_cast<const void*>(exact_scan_kernel<4, 0, kCount, false>));
    load(reinterpret_cast<const void*>(exact_scan_kernel<4, 0, kWrite, false>));
    load(reinterpret_cast<const void*>(exact_scan_kernel<2, 0, kCount, true>));
    load(reinterpret_cast<const void*>(sparse_scan_kernel<1, 4, sparse_tpb(1)>));
    load(reinterpret_cast<const void*>(fixup_rewalk_kernel<1>));
    load(reinterpret_cast<const void*>(fixup_walk_kernel<1>));
    load(reinterpret_cast<const void*>(fixup_resolve_kernel<1>));
    load(reinterpret_cast<const void*>(sparse_emit_kernel));
    load(reinterpret_cast<const void*>(compact_active_kernel));
    load(reinterpret_cast<const void*>(pattern_counts_kernel));
    load(reinterpret_cast<const void*>(zero_regions_kernel));
    load(reinterpret_cast<const void*>(scratch_copy_kernel<false>));
    load(reinterpret_cast<const void*>(scratch_copy_kernel<true>));
    load(reinterpret_cast<const void*>(qfilter_ldg_kernel<16, 2, false, false>));
    load(reinterpret_cast<const void*>(qconfirm_region_kernel));
    load(reinterpret_cast<const void*>(qconfirm_cta_kernel));
    load(reinterpret_cast<const void*>(qorder_region_kernel));
    // CUB's scan kernels and the pinned scalar slab, by one tiny use
    unsigned long long* d = nullptr;
    if (cudaMalloc(&d, 2 * sizeof(unsigned long long)) == cudaSuccess) {
        std::size_t tmp = 0;
        cub::DeviceScan::InclusiveSum(nullptr, tmp, d, d + 1, 1);
        void* t = nullptr;
        if (cudaMalloc(&t, std::max<std::size_t>(tmp, 16)) == cudaSuccess) {
            cub::DeviceScan::InclusiveSum(t, tmp, d, d + 1, 1);
            cudaDeviceSynchronize();
            cudaFree(t);
        }
        cudaFree(d);
    }
    if (unsigned long long* p = pinned_take()) pinned_give(p);
    (void)cudaGetLastError();
}

EagerDriverInit g_eager_driver_init;

// JSON string body of pattern bytes as nlohmann::json::dump(-1, ' ', false,
// error_handler_t::replace) writes it (the reference's cmd_match,
// proj/include/acmatch/cli.hpp:63-69): '"' '\\' and \b \f \n \r \t escaped,
// other bytes < 0x20 as \u00xx (lower-case hex), valid UTF-8 passed through,
// each invalid UTF-8 sequence replaced by U+FFFD (the byte that broke a
// sequence is read again as a possible start of the next one).
void json_escape(const std::uint8_t* b, std::size_t n, std::vector<std::uint8_t>& out) {
    auto fffd = [&] {
        out.push_back(0xEF);
        out.push_back(0xBF);
        out.push_back(0xBD);
    };
    std::size_t i = 0;
    while (i < n) {
        const std::uint8_t c = b[i];
        if (c < 0x80) {
            switch (c) {
                case '"': out.push_back('\\'); out.push_back('"'); break;
                case '\\': out.push_back('\\'); out.push_back('\\'); break;
                case '\b': out.push_back('\\'); out.push_back('b'); break;
                case '\f': out.push_back('\\'); out.push_back('f'); break;
                case '\n': out.push_back('\\'); out.push_back('n'); break;
                case '\r': out.push_back('\\'); out.push_back('r'); break;
                case '\t': out.push_back('\\'); out.push_back('t'); break;
                default:
                    if (c < 0x20) {
                        static const char hex[] = "0123456789abcdef";
                        const std::uint8_t esc[6] = {'\\', 'u', '0', '0', static_cast<std::uint8_t>(hex[c >> 4]),
                                                     static_cast<std::uint8_t>(hex[c & 15])};
                        out.insert(out.end(), esc, esc + 6);
                    } else {
                        out.push_back(c);
                    }
            }
            ++i;
            continue;
        }
        // UTF-8 sequence: lead byte ranges and the first continuation's range (RFC 3629)
        std::size_t need = 0;
        std::uint8_t lo = 0x80, hi = 0xBF;
        if (c >= 0xC2 && c <= 0xDF) need = 1;
        else if (c == 0xE0) need = 2, lo = 0xA0;
        else if ((c >= 0xE1 && c <= 0xEC) || c == 0xEE || c == 0xEF) need = 2;
        else if (c == 0xED) need = 2, hi = 0x9F;
        else if (c == 0xF0) need = 3, lo = 0x90;
        else if (c >= 0xF1 && c <= 0xF3) need = 3;
        else if (c == 0xF4) need = 3, hi = 0x8F;
        if (need == 0) {  // not a lead byte
            fffd();
            ++i;
            continue;
        }
        std::size_t k = 1;
        for (; k <= need && i + k < n; ++k) {
            const std::uint8_t d = b[i + k];
            const bool ok = k == 1 ? (d >= lo && d <= hi) : (d >= 0x80 && d <= 0xBF);
            if (!ok) break;
        }
        if (k == need + 1) {
            out.insert(out.end(), b + i, b + i + need + 1);
            i += need + 1;
        } else {
            fffd();  // the valid prefix is dropped; the breaking byte (if any) starts over
            i += k;
        }
    }
}

cudaError_t format_tables(const acg_automaton* a, DeviceDfa& dd, int json, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(dd.fmt_mu);
    if (dd.fmt_off[json].p) return cudaSuccess;
    const acg::Nfa& nfa = a->nfa;
    std::vector<std::uint8_t> bytes;
    std::vector<unsigned long long> offs(nfa.n_patterns + 1, 0);
    for (std::uint32_t p = 0; p < nfa.n_patterns; ++p) {
        const std::uint8_t* b = nfa.pat_bytes.data() + nfa.pat_off[p];
        const std::size_t len = nfa.pat_off[p + 1] - nfa.pat_off[p];
        if (json) json_escape(b, len, bytes);
        else bytes.insert(bytes.end(), b, b + len);
        offs[p + 1] = bytes.size();
    }
    if (bytes.empty()) bytes.push_back(0);
    cudaError_t e = upload(dd.fmt_str[json], bytes.data(), bytes.size(), st);
    if (e == cudaSuccess) e = upload(dd.fmt_off[json], offs.data(), offs.size(), st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // (host vectors die here)
    return e;
}

// Formats records [first, first + count) of the synced list into s->fmt_out
// (device); *bytes = their text size. JSON framing: "[" before the window's
// first record when open, "]\n" after its last when close (else ","); by
// default (open/close < 0) the window's place in this scanner's list decides.
int format_window(acg_scanner* s, int json, std::uint64_t first, std::uint64_t count, std::uint64_t* bytes,
                  int open = -1, int close = -1) {
    using namespace acg::kern;
    DeviceDfa& dd = *s->dd;
    cudaStream_t st = s->last;
    *bytes = 0;
    if (json && s->m_total == 0 && open < 0) {
        ACG_CUDA(s->fmt_out.reserve(3, st));
        ACG_CUDA(cudaMemcpyAsync(s->fmt_out.p, "[]\n", 3, cudaMemcpyHostToDevice, st));
        ACG_CUDA(cudaStreamSynchronize(st));
        *bytes = 3;
        return ACG_OK;
    }
    if (count == 0) return ACG_OK;
    ACG_CUDA(format_tables(s->a, dd, json, st));
    const std::uint64_t tiles = (count + kFmtTile - 1) / kFmtTile;
    ACG_CUDA(s->fmt_tiles.reserve(2 * tiles + 1, st));
    FmtArgs f{};
    f.rec = s->records.p + first;
    f.m = count;
    f.id_bits = dd.dfa->id_bits;
    f.str = dd.fmt_str[json].p;
    f.str_off = dd.fmt_off[json].p;
    f.json = json;
    f.open = open >= 0 ? open : first == 0;
    f.close = close >= 0 ? close : first + count == s->m_total;
    f.tile_sum = s->fmt_tiles.p;
    f.tile_off = s->fmt_tiles.p + tiles;
    const unsigned g = static_cast<unsigned>(std::min<std::uint64_t>(tiles, 16ull * dd.num_sms));
    format_len_kernel<<<g, kFmtTile, 0, st>>>(f);
    ACG_CUDA(cudaGetLastError());
    ACG_CUDA(cudaMemsetAsync(s->fmt_tiles.p + tiles, 0, sizeof(unsigned long long), st));
    std::size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, f.tile_sum, s->fmt_tiles.p + tiles + 1, static_cast<int>(tiles), st);
    ACG_CUDA(s->cub_tmp.reserve(std::max(tmp, s->cub_tmp.n), st));
    tmp = s->cub_tmp.n;
    ACG_CUDA(cub::DeviceScan::InclusiveSum(s->cub_tmp.p, tmp, f.tile_sum, s->fmt_tiles.p + tiles + 1,
                                           static_cast<int>(tiles), st));
    unsigned long long total = 0;
    ACG_CUDA(cudaMemcpyAsync(&total, s->fmt_tiles.p + 2 * tiles, sizeof total, cudaMemcpyDeviceToHost, st));
    ACG_CUDA(cudaStreamSynchronize(st));
    ACG_CUDA(s->fmt_out.reserve(std::max<std::uint64_t>(total, 1), st));
    f.out = s->fmt_out.p;
    format_write_kernel<<<g, kFmtTile, 0, st>>>(f);
    ACG_CUDA(cudaGetLastError());
    *bytes = total;
    return ACG_OK;
}

// Visit counts per NFA state of the reference walk over a text sample (the
// dense rows built with the automaton: one table lookup per byte).
std::vector<std::uint64_t> sample_visits(const acg::Nfa& nfa, const std::uint8_t* sample, std::uint64_t n) {
    std::vector<std::uint64_t> visits(nfa.state_count(), 0);
    const std::uint32_t K = nfa.K;
    bool in_alpha[256];
    for (int b = 0; b < 256; ++b)
        in_alpha[b] = nfa.mode == acg::kAlphaGeneric || b == 'A' || b == 'C' || b == 'G' || b == 'T';
    std::uint32_t s = 0;
    for (std::uint64_t i = 0; i < n; ++i) {
        const std::uint8_t b = sample[i];
        s = in_alpha[b] ? nfa.delta[static_cast<std::size_t>(s) * K + nfa.symmap[b]] : 0u;  // (escape: root)
        ++visits[s];
    }
    return visits;
}

constexpr std::uint64_t kAutoLayoutSample = 1ull << 20;

}  // namespace

extern "C" {

// A first host scan of a generic-alphabet automaton whose hot rows do not
// cover all states picks the profile-guided hot set from its own text (the
// first kAutoLayoutSample bytes) before the tables go to the device: results
// are unaffected, cfg3's walk runs 0.99 -> 0.65 ms per 256 MiB. ACG_AUTO_LAYOUT=0 turns it off.
__attribute__((visibility("hidden"))) void acg_internal_auto_layout(acg_automaton* a, const std::uint8_t* text,
                                                                    std::uint64_t n) {
    static const bool on = [] {
        const char* e = std::getenv("ACG_AUTO_LAYOUT");
        return !(e && e[0] == '0');
    }();
    if (!on || !a || !text || n < 4096) return;
    {
        std::lock_guard<std::mutex> lock(a->mu);
        if (!a->dev.empty() || !a->profile.empty() || a->hot_limit) return;
        const auto d = host_dfa_locked(a, kSm100SmemOptin);
        if (d->mode != acg::kAlphaGeneric || d->H >= d->S) return;
    }
    std::vector<std::uint64_t> visits = sample_visits(a->nfa, text, std::min<std::uint64_t>(n, kAutoLayoutSample));
    std::lock_guard<std::mutex> lock(a->mu);
    if (!a->dev.empty() || !a->profile.empty()) return;  // (another thread got there first)
    a->profile = std::move(visits);
    a->dfa.reset();
}

// Pooled scanners for the pipelined host scan (host_io.cpp); not part of include/acg.h.
__attribute__((visibility("hidden"))) int acg_internal_scanner_take(const acg_automaton* a, int device,
                                                                    std::uint32_t flags, acg_scanner** out) {
    acg_scanner* s = pool_take(a, device, flags);
    if (!s) {
        if (const int rc = make_scanner(a, device, flags, &s)) return rc;
    }
    *out = s;
    return ACG_OK;
}
__attribute__((visibility("hidden"))) void acg_internal_scanner_give(acg_scanner* s) { pool_give(s); }
__attribute__((visibility("hidden"))) void* acg_internal_scanner_stream(acg_scanner* s) { return s->stream; }
// records [first, first+count) of the synced list formatted with explicit JSON
// framing, copied to host (host_io.cpp's streamed scan)
__attribute__((visibility("hidden"))) int acg_internal_format(acg_scanner* s, int json, std::uint64_t first,
                                                              std::uint64_t count, int open, int close,
                                                              std::uint8_t* host, std::uint64_t cap,
                                                              std::uint64_t* bytes) {
    if (const int rc = scanner_sync(s)) return rc;
    if (const int rc = format_window(s, json, first, count, bytes, open, close)) return rc;
    if (!host) return ACG_OK;  // the text stays in the scanner's output buffer (acg_internal_fetch)
    if (*bytes > cap) return fail(ACG_ERR_INVALID, "output staging smaller than the formatted window");
    if (*bytes) {
        ACG_CUDA(cudaMemcpyAsync(host, s->fmt_out.p, *bytes, cudaMemcpyDeviceToHost, s->last));
        ACG_CUDA(cudaStreamSynchronize(s->last));
    }
    return ACG_OK;
}
// the last acg_internal_format's text (bytes of it) to host
__attribute__((visibility("hidden"))) int acg_internal_fetch(acg_scanner* s, std::uint8_t* host, std::uint64_t bytes) {
    if (bytes > s->fmt_out.n) return fail(ACG_ERR_INVALID, "nothing formatted");
    if (bytes) {
        ACG_CUDA(cudaMemcpyAsync(host, s->fmt_out.p, bytes, cudaMemcpyDeviceToHost, s->last));
        ACG_CUDA(cudaStreamSynchronize(s->last));
    }
    return ACG_OK;
}

// (host_io.cpp reports its errors through this; not part of include/acg.h)
__attribute__((visibility("hidden"))) int acg_internal_set_error(int code, const char* msg) { return fail(code, msg); }

const char* acg_last_error(void) { return g_last_error.c_str(); }
const char* acg_version(void) { return "acg 0.1 (sm_100a)"; }

int acg_build(const std::uint8_t* concat, const std::uint64_t* offsets, std::uint32_t n_patterns, acg_automaton** out) {
    if (!out) return fail(ACG_ERR_INVALID, "null output handle");
    *out = nullptr;
    if (n_patterns == 0) return fail(ACG_ERR_EMPTY_DICTIONARY, "dictionary is empty");
    if (!offsets || (!concat && offsets[n_patterns] != 0)) return fail(ACG_ERR_INVALID, "null pattern buffers");
    for (std::uint32_t i = 0; i < n_patterns; ++i)
        if (offsets[i + 1] < offsets[i]) return fail(ACG_ERR_INVALID, "pattern offsets must be non-decreasing");
    auto a = std::make_unique<acg_automaton>();
    try {
        const auto t0 = std::chrono::steady_clock::now();
        const int rc = acg::build_nfa(concat, offsets, n_patterns, a->nfa);
        const auto t1 = std::chrono::steady_clock::now();
        if (rc == acg::kErrEmptyPattern) {
            std::uint32_t i = 0;
            while (offsets[i + 1] != offsets[i]) ++i;
            return fail(rc, "pattern " + std::to_string(i) + " is empty");
        }
        if (rc == acg::kErrEmptyDictionary) return fail(rc, "dictionary is empty");
        if (rc == acg::kErrTooLarge)
            return fail(ACG_ERR_INVALID, "dictionary of 4 GiB or more: its trie would exceed 32-bit state ids");
        if (rc != acg::kOk) return fail(rc, "invalid dictionary");
        std::lock_guard<std::mutex> lock(a->mu);
        host_dfa_locked(a.get(), kSm100SmemOptin);
        if (g_debug)
            std::fprintf(stderr, "[acg] build: nfa %.3f s, dfa+filter %.3f s (%u states)\n",
                         std::chrono::duration<double>(t1 - t0).count(),
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count(),
                         a->nfa.state_count());
    } catch (const std::bad_alloc&) {
        return fail(ACG_ERR_OUT_OF_MEMORY, "host allocation failed while building the automaton");
    }
    *out = a.release();
    return ACG_OK;
}

void acg_automaton_destroy(acg_automaton* a) {
    if (!a) return;
    pool_drop(a);
    delete a;
}

std::uint32_t acg_state_count(const acg_automaton* a) { return a->nfa.state_count(); }
std::uint32_t acg_pattern_count(const acg_automaton* a) { return a->nfa.n_patterns; }
std::uint32_t acg_max_pattern_length(const acg_automaton* a) { return a->nfa.max_len; }
int acg_goto_transition(const acg_automaton* a, std::uint32_t s, std::uint8_t b, std::uint32_t* to) {
    std::uint32_t t = 0;
    const bool ok = a->nfa.goto_transition(s, b, &t);
    if (ok && to) *to = t;
    return ok ? 1 : 0;
}
std::uint32_t acg_transitions(const acg_automaton* a, std::uint32_t s, const std::uint8_t** bytes,
                              const std::uint32_t** targets) {
    const std::uint32_t lo = a->nfa.edge_off[s], hi = a->nfa.edge_off[s + 1];
    if (bytes) *bytes = a->nfa.edge_byte.data() + lo;
    if (targets) *targets = a->nfa.edge_to.data() + lo;
    return hi - lo;
}
std::uint32_t acg_failure(const acg_automaton* a, std::uint32_t s) { return a->nfa.fail[s]; }
std::uint32_t acg_outputs(const acg_automaton* a, std::uint32_t s, const std::uint32_t** ids) {
    const std::uint32_t lo = a->nfa.out_off[s], hi = a->nfa.out_off[s + 1];
    if (ids) *ids = a->nfa.out_ids.data() + lo;
    return hi - lo;
}
std::uint32_t acg_depth(const acg_automaton* a, std::uint32_t s) { return a->nfa.depth[s]; }

int acg_nfa_arrays(const acg_automaton* a, const std::uint32_t** fail_links, const std::uint32_t** depth,
                   const std::uint32_t** edge_off, const std::uint8_t** edge_byte, const std::uint32_t** edge_to,
                   const std::uint32_t** out_off, const std::uint32_t** out_ids) {
    if (!a) return fail(ACG_ERR_INVALID, "null automaton");
    if (fail_links) *fail_links = a->nfa.fail.data();
    if (depth) *depth = a->nfa.depth.data();
    if (edge_off) *edge_off = a->nfa.edge_off.data();
    if (edge_byte) *edge_byte = a->nfa.edge_byte.data();
    if (edge_to) *edge_to = a->nfa.edge_to.data();
    if (out_off) *out_off = a->nfa.out_off.data();
    if (out_ids) *out_ids = a->nfa.out_ids.data();
    return ACG_OK;
}
std::uint32_t acg_next_state(const acg_automaton* a, std::uint32_t s, std::uint8_t b) {
    return a->nfa.next_state(s, b);
}

int acg_optimize_layout(acg_automaton* a, const std::uint8_t* sample, std::uint64_t n) {
    if (!a || (!sample && n)) return fail(ACG_ERR_INVALID, "null argument");
    {
        std::lock_guard<std::mutex> lock(a->mu);
        if (!a->dev.empty()) return fail(ACG_ERR_INVALID, "layout is fixed once the automaton has been scanned");
    }
    std::vector<std::uint64_t> visits = sample_visits(a->nfa, sample, n);
    std::lock_guard<std::mutex> lock(a->mu);
    a->profile = std::move(visits);
    a->dfa.reset();
    return ACG_OK;
}

int acg_set_hot_limit(acg_automaton* a, std::uint32_t max_hot_rows) {
    if (!a) return fail(ACG_ERR_INVALID, "null automaton");
    std::lock_guard<std::mutex> lock(a->mu);
    if (!a->dev.empty()) return fail(ACG_ERR_INVALID, "layout is fixed once the automaton has been scanned");
    a->hot_limit = max_hot_rows;
    a->dfa.reset();
    return ACG_OK;
}

int acg_automaton_filter_info(const acg_automaton* a, std::uint32_t* q, double* pass_rate) {
    if (!a) return 0;
    std::shared_ptr<const acg::Dfa> dfa;
    {
        std::lock_guard<std::mutex> lock(a->mu);
        if (a->dev.empty()) dfa = host_dfa_locked(a, kSm100SmemOptin);
        else dfa = a->dev.begin()->second->dfa;
    }
    if (q) *q = dfa->q;
    if (pass_rate) *pass_rate = dfa->filter_fp;
    return dfa->filter_ok ? 1 : 0;
}

int acg_automaton_ctab_check(const acg_automaton* a, const std::uint8_t* text, std::uint64_t n, std::uint32_t* info,
                             std::uint64_t* mismatches, std::uint64_t* cold_steps) {
    using namespace acg;
    if (info) info[0] = info[1] = info[2] = info[3] = info[4] = 0;
    if (mismatches) *mismatches = 0;
    if (cold_steps) *cold_steps = 0;
    if (!a) return 0;
    std::shared_ptr<const acg::Dfa> dfa;
    {
        std::lock_guard<std::mutex> lock(a->mu);
        if (a->dev.empty()) dfa = host_dfa_locked(a, kSm100SmemOptin);
        else dfa = a->dev.begin()->second->dfa;
    }
    const acg::Dfa& d = *dfa;
    if (d.ctab.empty()) return 0;
    const std::uint32_t K = d.K, slots = d.ct_slots, D = d.ct_D, esc = K - 1;
    if (info) {
        info[0] = slots;
        info[1] = D;
        info[2] = d.ct_hot;
        std::uint32_t ents = 0;
        for (std::uint32_t i = 0; i < slots; ++i) ents += d.ctab[i] != kCtEmpty;
        info[3] = ents;
        info[4] = d.ct_deep ? 1u : 0u;
    }
    if (!text) return 1;
    // the device walk (exact_kernels.cuh: ctab_event_kernel), step for step
    std::uint64_t bad = 0, cold = 0;
    const std::uint32_t pay = d.ct_cnt ? kCtPayMask : kCtValMask;  // an id / payload without the count bits
    std::uint32_t c1 = esc, c2 = esc, s_dev = 0;
    std::uint32_t sw = d.ctab[slots + (D == 3 ? (K * K + K + 1) : (K + 1)) * esc];
    std::uint32_t xprev = sw;  // the previous position's T_D default (deep default)
    for (std::uint64_t i = 0; i < n; ++i) {
        const std::uint32_t c = d.symmap[text[i]];
        const std::uint32_t idx = D == 3 ? (c2 * K + c1) * K + c : c1 * K + c;
        std::uint32_t x = d.ctab[slots + idx];
        if (d.ct_deep) {
            const std::uint32_t e2 = d.ctab[(xprev & pay) + c] ^ (c << kCtColShift);
            xprev = x;
            if (!(e2 & kCtColMask)) x = e2;
        }
        c2 = c1;
        c1 = c;
        std::uint32_t nx;
        if (sw & kCtCold) {
            ++cold;
            const std::uint32_t s = (sw & kCtOut) ? (sw & pay) - slots + d.Hn : (sw & kCtValMask);
            nx = d.ct_next[static_cast<std::size_t>(s) * K + c];
        } else {
            const std::uint32_t ent = d.ctab[(sw & pay) + c];
            const std::uint32_t diff = ent ^ (c << kCtColShift);
            nx = (diff & kCtColMask) ? x : diff;
        }
        sw = nx;
        s_dev = d.next[static_cast<std::size_t>(s_dev) * K + c];
        if (sw != d.ct_sw[s_dev]) {
            ++bad;
            sw = d.ct_sw[s_dev];
        }
    }
    if (mismatches) *mismatches = bad;
    if (cold_steps) *cold_steps = cold;
    return 1;
}

int acg_automaton_layout(const acg_automaton* a, std::uint32_t* n_states, std::uint32_t* hot_rows,
                         std::uint32_t* columns, std::uint32_t* halo, int* alphabet_mode) {
    if (!a) return fail(ACG_ERR_INVALID, "null automaton");
    std::shared_ptr<const acg::Dfa> dfa;
    {
        std::lock_guard<std::mutex> lock(a->mu);
        if (a->dev.empty()) dfa = host_dfa_locked(a, kSm100SmemOptin);
        else dfa = a->dev.begin()->second->dfa;
    }
    const acg::Dfa& d = *dfa;
    if (n_states) *n_states = d.S;
    if (hot_rows) *hot_rows = d.H;
    if (columns) *columns = d.K;
    if (halo) *halo = d.halo;
    if (alphabet_mode) *alphabet_mode = d.mode;
    return ACG_OK;
}

int acg_scanner_create(const acg_automaton* a, int device, std::uint32_t flags, acg_scanner** out) {
    if (!a || !out) return fail(ACG_ERR_INVALID, "null argument");
    *out = nullptr;
    if (device < 0) device = current_device();
    if ((flags & ~ACG_SCAN_PROFILE) == 0) flags |= ACG_SCAN_LIST | ACG_SCAN_COUNTS;
    return make_scanner(a, device, flags, out);
}

void acg_scanner_destroy(acg_scanner* s) { free_scanner(s); }

int acg_scanner_set_geometry(acg_scanner* s, std::uint32_t streams_per_thread, std::uint32_t threads_per_block,
                             std::uint64_t chunk_bytes) {
    if (!s) return fail(ACG_ERR_INVALID, "null scanner");
    if (streams_per_thread) {
        if (streams_per_thread != 1 && streams_per_thread != 2 && streams_per_thread != 4 && streams_per_thread != 8)
            return fail(ACG_ERR_INVALID, "streams per thread must be 1, 2, 4 or 8");
        s->U = streams_per_thread;
    }
    if (threads_per_block) {
        if (threads_per_block % 32 || threads_per_block > 2u * acg::kern::kTPB)
            return fail(ACG_ERR_INVALID, "threads per block must be a multiple of 32, at most 1024 (512 above 2 streams per thread)");
        s->tpb = threads_per_block;
        s->tpb_set = true;
    }
    s->chunk_override = chunk_bytes;
    return ACG_OK;
}

int acg_scanner_run(acg_scanner* s, const std::uint8_t* d_text, std::uint64_t n, std::uint64_t emit_from,
                    std::uint64_t base_offset, void* stream) {
    if (!s || (!d_text && n)) return fail(ACG_ERR_INVALID, "null argument");
    return scanner_run(s, d_text, n, emit_from, base_offset, stream ? static_cast<cudaStream_t>(stream) : s->stream);
}

int acg_scanner_run_host(acg_scanner* s, const std::uint8_t* h_text, std::uint64_t n, void* stream) {
    if (!s || (!h_text && n)) return fail(ACG_ERR_INVALID, "null argument");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->stream;
    ACG_CUDA(cudaSetDevice(s->device));
    ACG_CUDA(adopt_stream(s, st));
    ACG_CUDA(s->text.reserve(std::max<std::uint64_t>(n, 16), st));
    if (n) ACG_CUDA(cudaMemcpyAsync(s->text.p, h_text, n, cudaMemcpyHostToDevice, st));
    return scanner_run(s, s->text.p, n, 0, 0, st);
}

int acg_scanner_sync(acg_scanner* s) {
    if (!s) return fail(ACG_ERR_INVALID, "null scanner");
    return scanner_sync(s);
}

std::uint64_t acg_scanner_match_count(acg_scanner* s) {
    if (!s || scanner_sync(s)) return 0;
    return s->m_total;
}

int acg_scanner_packed_records(acg_scanner* s, std::uint64_t* host, std::uint64_t cap, std::uint32_t* id_bits) {
    if (!s) return fail(ACG_ERR_INVALID, "null scanner");
    if (!(s->flags & ACG_SCAN_LIST)) return fail(ACG_ERR_INVALID, "scanner was created without ACG_SCAN_LIST");
    if (const int rc = scanner_sync(s)) return rc;
    if (id_bits) *id_bits = s->dd->dfa->id_bits;
    const std::uint64_t m = std::min<std::uint64_t>(cap, s->m_total);
    if (m) {
        ACG_CUDA(cudaMemcpyAsync(host, s->records.p, m * sizeof(std::uint64_t), cudaMemcpyDeviceToHost, s->last));
        ACG_CUDA(cudaStreamSynchronize(s->last));
    }
    return ACG_OK;
}

int acg_scanner_copy_records(acg_scanner* s, std::uint64_t first, std::uint64_t count, std::uint64_t* host) {
    if (!s || (!host && count)) return fail(ACG_ERR_INVALID, "null argument");
    if (!(s->flags & ACG_SCAN_LIST)) return fail(ACG_ERR_INVALID, "scanner was created without ACG_SCAN_LIST");
    if (const int rc = scanner_sync(s)) return rc;
    if (first > s->m_total || count > s->m_total - first) return fail(ACG_ERR_INVALID, "record range beyond the match list");
    if (count) {
        ACG_CUDA(cudaMemcpyAsync(host, s->records.p + first, count * sizeof(std::uint64_t), cudaMemcpyDeviceToHost, s->last));
        ACG_CUDA(cudaStreamSynchronize(s->last));
    }
    return ACG_OK;
}

int acg_scanner_format(acg_scanner* s, int format, std::uint64_t first, std::uint64_t count, std::uint8_t* host_out,
                       std::uint64_t cap, std::uint64_t* bytes) {
    if (!s || !bytes) return fail(ACG_ERR_INVALID, "null argument");
    if (format != ACG_FORMAT_TSV && format != ACG_FORMAT_JSON) return fail(ACG_ERR_INVALID, "unknown output format");
    if (!(s->flags & ACG_SCAN_LIST)) return fail(ACG_ERR_INVALID, "scanner was created without ACG_SCAN_LIST");
    if (const int rc = scanner_sync(s)) return rc;
    if (first > s->m_total || count > s->m_total - first) return fail(ACG_ERR_INVALID, "record range beyond the match list");
    ACG_CUDA(cudaSetDevice(s->device));
    if (const int rc = format_window(s, format == ACG_FORMAT_JSON, first, count, bytes)) return rc;
    if (!host_out) return ACG_OK;
    if (cap < *bytes) return fail(ACG_ERR_INVALID, "output buffer smaller than the formatted text");
    if (*bytes) {
        ACG_CUDA(cudaMemcpyAsync(host_out, s->fmt_out.p, *bytes, cudaMemcpyDeviceToHost, s->last));
        ACG_CUDA(cudaStreamSynchronize(s->last));
    }
    return ACG_OK;
}

int acg_scanner_write_matches(acg_scanner* s, int format, int fd, std::uint64_t* bytes) {
    if (!s) return fail(ACG_ERR_INVALID, "null scanner");
    if (bytes) *bytes = 0;
    if (const int rc = scanner_sync(s)) return rc;
    constexpr std::uint64_t kWindow = 1ull << 24;  // records per formatted window
    std::uint64_t total = 0;
    unsigned char* stage = nullptr;
    std::uint64_t stage_n = 0;
    int rc = ACG_OK;
    const std::uint64_t m = s->m_total;
    const std::uint64_t windows = m ? (m + kWindow - 1) / kWindow : 1;
    for (std::uint64_t w = 0; w < windows && !rc; ++w) {
        const std::uint64_t first = w * kWindow, count = std::min(kWindow, m - std::min(m, first));
        std::uint64_t nb = 0;
        if ((rc = acg_scanner_format(s, format, first, count, nullptr, 0, &nb))) break;
        if (nb > stage_n) {
            if (stage) cudaFreeHost(stage);
            stage_n = nb + nb / 8;
            if (cudaHostAlloc(reinterpret_cast<void**>(&stage), stage_n, cudaHostAllocDefault) != cudaSuccess) {
                cudaGetLastError();
                stage = nullptr;
                rc = fail(ACG_ERR_OUT_OF_MEMORY, "pinned staging allocation failed");
                break;
            }
        }
        if (nb) {
            if (cudaMemcpyAsync(stage, s->fmt_out.p, nb, cudaMemcpyDeviceToHost, s->last) != cudaSuccess ||
                cudaStreamSynchronize(s->last) != cudaSuccess) {
                rc = fail(ACG_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
                break;
            }
        }
        for (std::uint64_t off = 0; off < nb;) {
            const ssize_t k = ::write(fd, stage + off, nb - off);
            if (k < 0 && errno == EINTR) continue;
            if (k <= 0) {
                rc = fail(ACG_ERR_IO, "write failed");
                break;
            }
            off += static_cast<std::uint64_t>(k);
        }
        total += nb;
    }
    if (stage) cudaFreeHost(stage);
    if (!rc && bytes) *bytes = total;
    return rc;
}

int acg_scanner_records(acg_scanner* s, std::uint32_t* ids, std::uint64_t* ends, std::uint64_t cap) {
    if (!s) return fail(ACG_ERR_INVALID, "null scanner");
    if (const int rc = scanner_sync(s)) return rc;
    const std::uint64_t m = std::min<std::uint64_t>(cap, s->m_total);
    std::vector<std::uint64_t> packed(m);
    std::uint32_t bits = 0;
    if (const int rc = acg_scanner_packed_records(s, packed.data(), m, &bits)) return rc;
    const std::uint64_t mask = (1ull << bits) - 1;
    for (std::uint64_t i = 0; i < m; ++i) {
        ids[i] = static_cast<std::uint32_t>(packed[i] & mask);
        ends[i] = packed[i] >> bits;
    }
    return ACG_OK;
}

int acg_scanner_pattern_counts(acg_scanner* s, std::uint64_t* host_counts) {
    if (!s) return fail(ACG_ERR_INVALID, "null scanner");
    if (!(s->flags & ACG_SCAN_COUNTS)) return fail(ACG_ERR_INVALID, "scanner was created without ACG_SCAN_COUNTS");
    if (const int rc = scanner_sync(s)) return rc;
    ACG_CUDA(cudaMemcpyAsync(host_counts, s->counts.p, s->a->nfa.n_patterns * sizeof(std::uint64_t),
                             cudaMemcpyDeviceToHost, s->last));
    ACG_CUDA(cudaStreamSynchronize(s->last));
    return ACG_OK;
}

const std::uint64_t* acg_scanner_device_pattern_counts(acg_scanner* s) {
    return s ? reinterpret_cast<const std::uint64_t*>(s->counts.p) : nullptr;
}

const std::uint64_t* acg_scanner_device_records(acg_scanner* s, std::uint32_t* id_bits) {
    if (!s) return nullptr;
    if (id_bits) *id_bits = s->dd->dfa->id_bits;
    return reinterpret_cast<const std::uint64_t*>(s->records.p);
}

std::uint64_t acg_scanner_failure_follows(acg_scanner* s) {
    if (!s || scanner_sync(s)) return 0;
    if (cudaMemcpyAsync(s->pinned + 4, s->scalars64.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s->last) !=
            cudaSuccess ||
        cudaStreamSynchronize(s->last) != cudaSuccess)
        return 0;
    return s->pinned[4];
}

int acg_scanner_digest(acg_scanner* s, std::uint64_t* dsum, std::uint64_t* dxor, std::uint64_t* unsorted_pairs) {
    if (!s) return fail(ACG_ERR_INVALID, "null scanner");
    if (const int rc = scanner_sync(s)) return rc;
    ACG_CUDA(cudaMemsetAsync(s->scalars64.p + 1, 0, 3 * sizeof(unsigned long long), s->last));
    if (s->m_total) {
        const unsigned g = std::min<unsigned long long>((s->m_total + 255) / 256, 4096ull);
        acg::kern::digest_kernel<<<g, 256, 0, s->last>>>(s->records.p, s->m_total, s->dd->dfa->id_bits,
                                                          s->scalars64.p + 1);
        ACG_CUDA(cudaGetLastError());
    }
    ACG_CUDA(cudaMemcpyAsync(s->pinned + 1, s->scalars64.p + 1, 3 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s->last));
    ACG_CUDA(cudaStreamSynchronize(s->last));
    if (dsum) *dsum = s->pinned[1];
    if (dxor) *dxor = s->pinned[2];
    if (unsorted_pairs) *unsorted_pairs = s->pinned[3];
    return ACG_OK;
}

int acg_scanner_kernel_ms(acg_scanner* s, float* ms5) {
    if (!s || !ms5) return fail(ACG_ERR_INVALID, "null argument");
    if (!(s->flags & ACG_SCAN_PROFILE)) return fail(ACG_ERR_INVALID, "scanner was created without ACG_SCAN_PROFILE");
    if (const int rc = scanner_sync(s)) return rc;
    for (int i = 0; i < 5; ++i) ms5[i] = s->kernel_ms[i];
    return ACG_OK;
}

int acg_scanner_set_profiling(acg_scanner* s, int on) {
    if (!s) return fail(ACG_ERR_INVALID, "null scanner");
    if (on) {
        ACG_CUDA(cudaSetDevice(s->device));
        for (auto& e : s->ev)
            if (!e) ACG_CUDA(cudaEventCreate(&e));
        s->flags |= ACG_SCAN_PROFILE;
    } else {
        s->flags &= ~static_cast<std::uint32_t>(ACG_SCAN_PROFILE);
    }
    return ACG_OK;
}

int acg_scanner_set_mode(acg_scanner* s, int mode) {
    if (!s) return fail(ACG_ERR_INVALID, "null scanner");
    if (mode < ACG_MODE_AUTO || mode > ACG_MODE_FILTER) return fail(ACG_ERR_INVALID, "unknown mode");
    s->mode_req = mode;
    return ACG_OK;
}

int acg_scanner_last_mode(acg_scanner* s, double* event_rate) {
    if (!s) return -1;
    if (event_rate) *event_rate = s->mode_run == ACG_MODE_FILTER ? s->last_filter_rate : s->last_event_rate;
    return s->mode_run;
}

int acg_scanner_last_walk(const acg_scanner* s) {
    if (!s) return -1;
    return s->c_run ? 1 : s->g_run ? 2 : 0;
}

int acg_scanner_copy_pattern_counts(acg_scanner* s, void* d_dst, void* stream) {
    if (!s || !d_dst) return fail(ACG_ERR_INVALID, "null argument");
    if (!(s->flags & ACG_SCAN_COUNTS)) return fail(ACG_ERR_INVALID, "scanner was created without ACG_SCAN_COUNTS");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->last;
    ACG_CUDA(cudaMemcpyAsync(d_dst, s->counts.p, s->a->nfa.n_patterns * sizeof(std::uint64_t),
                             cudaMemcpyDeviceToDevice, st));
    return ACG_OK;
}

std::uint64_t acg_scanner_replays(const acg_scanner* s) { return s ? s->replays : 0; }

int acg_scanner_last_geometry(acg_scanner* s, std::uint64_t* n_chunks, std::uint64_t* chunk_bytes,
                              std::uint32_t* launches) {
    if (!s) return fail(ACG_ERR_INVALID, "null scanner");
    if (n_chunks) *n_chunks = s->n_chunks;
    if (chunk_bytes) *chunk_bytes = s->chunk;
    if (launches) *launches = s->launches;
    return ACG_OK;
}

int acg_scan(const acg_automaton* a, const std::uint8_t* text, std::uint64_t n, std::uint32_t flags,
             acg_result** out) {
    if (!a || !out || (!text && n)) return fail(ACG_ERR_INVALID, "null argument");
    *out = nullptr;
    if (!flags) flags = ACG_SCAN_LIST;
    const int device = current_device();
    acg_internal_auto_layout(const_cast<acg_automaton*>(a), text, n);
    acg_scanner* s = pool_take(a, device, flags);
    if (!s) {
        if (const int rc = make_scanner(a, device, flags, &s)) return rc;
    }
    auto res = std::make_unique<acg_result>();
    int rc = acg_scanner_run_host(s, text, n, nullptr);
    if (!rc) rc = scanner_sync(s);
    if (!rc && (flags & ACG_SCAN_LIST)) {
        res->ids.resize(s->m_total);
        res->ends.resize(s->m_total);
        rc = acg_scanner_records(s, res->ids.data(), res->ends.data(), s->m_total);
    }
    if (!rc && (flags & ACG_SCAN_COUNTS)) {
        res->counts.resize(a->nfa.n_patterns);
        rc = acg_scanner_pattern_counts(s, res->counts.data());
    }
    if (!rc && (flags & ACG_SCAN_STATS)) res->follows = acg_scanner_failure_follows(s);
    if (rc) {
        free_scanner(s);
        return rc;
    }
    pool_give(s);
    *out = res.release();
    return ACG_OK;
}

std::uint64_t acg_result_match_count(const acg_result* r) { return r ? r->ids.size() : 0; }
const std::uint32_t* acg_result_ids(const acg_result* r) { return r ? r->ids.data() : nullptr; }
const std::uint64_t* acg_result_ends(const acg_result* r) { return r ? r->ends.data() : nullptr; }
const std::uint64_t* acg_result_pattern_counts(const acg_result* r) {
    return r && !r->counts.empty() ? r->counts.data() : nullptr;
}
std::uint64_t acg_result_failure_follows(const acg_result* r) { return r ? r->follows : 0; }
void acg_result_destroy(acg_result* r) { delete r; }

}  // extern "C"

// the GPU-native dictionary-partitioned run (its own C-ABI entry points)
#include "partition.cuh"
