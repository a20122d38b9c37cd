// Input path and pipelined host scan.
//
// The reference reads files through istreambuf_iterator into a std::string
// (proj/include/acmatch/io.hpp:25-31; patterns :37-65) and scans a host
// string_view (aho_corasick.hpp:250-277). Here:
//  * acg_load_input reads the file with parallel pread()s straight into
//    page-locked memory, so the H2D copy runs at full PCIe rate;
//  * acg_load_patterns applies load_patterns' line rules (LF split, one
//    trailing CR stripped, empty lines skipped, first occurrence kept, dense
//    ids in load order) and returns the dictionary in the C ABI's layout;
//  * acg_scan_pipelined scans a host text of any size in pieces on two
//    scanners / two streams: piece k+1's H2D copy and scan run while piece
//    k's packed records come back (PCIe is full duplex). Pieces are text
//    windows with maxlen-1 bytes of warm-up context, so each
//    piece's list is canonical and the pieces concatenate in text order.
// Everything here is written against the public C ABI plus the CUDA runtime.
#include "acg.h"

#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_set>
#include <vector>

// sets the thread-local acg_last_error text; returns code (acg_device.cu; not exported)
extern "C" __attribute__((visibility("hidden"))) int acg_internal_set_error(int code, const char* msg);
// the library's per-automaton scanner pool (kept across calls: adaptive workspace sizes persist)
extern "C" __attribute__((visibility("hidden"))) int acg_internal_scanner_take(const acg_automaton* a, int device,
                                                                               uint32_t flags, acg_scanner** out);
extern "C" __attribute__((visibility("hidden"))) void acg_internal_scanner_give(acg_scanner* s);
extern "C" __attribute__((visibility("hidden"))) void* acg_internal_scanner_stream(acg_scanner* s);  // its own stream
// GPU-formatted window with explicit JSON framing, copied to host (acg_device.cu)
extern "C" __attribute__((visibility("hidden"))) int acg_internal_format(acg_scanner* s, int json, uint64_t first,
                                                                         uint64_t count, int open, int close,
                                                                         uint8_t* host, uint64_t cap, uint64_t* bytes);
extern "C" __attribute__((visibility("hidden"))) int acg_internal_fetch(acg_scanner* s, uint8_t* host, uint64_t bytes);
// profile-guided hot rows from the text on a generic-alphabet automaton's first scan (acg_device.cu)
extern "C" __attribute__((visibility("hidden"))) void acg_internal_auto_layout(acg_automaton* a, const uint8_t* text,
                                                                               uint64_t n);
constexpr uint32_t kPipelineTag = 0x100u;  // pool key bit: pipeline lanes keep their own adaptive state

namespace {

int io_fail(const std::string& msg) { return acg_internal_set_error(ACG_ERR_IO, msg.c_str()); }

// Whole file into page-locked memory (falls back to pageable if pinning fails).
int read_file(const char* path, std::uint8_t** data, std::uint64_t* n, bool pin) {
    *data = nullptr;
    *n = 0;
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) return io_fail(std::string("cannot open ") + path);
    struct stat sb {};
    if (::fstat(fd, &sb) != 0) {
        ::close(fd);
        return io_fail(std::string("read failed: ") + path);
    }
    const std::uint64_t size = static_cast<std::uint64_t>(sb.st_size);
    void* buf = nullptr;
    const std::size_t alloc = static_cast<std::size_t>(std::max<std::uint64_t>(size, 16));
    if (!pin || cudaHostAlloc(&buf, alloc, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        buf = std::malloc(alloc);
        if (!buf) {
            ::close(fd);
            return acg_internal_set_error(ACG_ERR_OUT_OF_MEMORY, "host allocation failed");
        }
        pin = false;
    }
    // parallel preads of 64 MiB pieces (a page-cache-resident file reads at memcpy speed)
    constexpr std::uint64_t kPiece = 64ull << 20;
    const std::uint64_t pieces = (size + kPiece - 1) / kPiece;
    const unsigned threads = static_cast<unsigned>(
        std::max<std::uint64_t>(1, std::min<std::uint64_t>(pieces, std::max(1u, std::thread::hardware_concurrency()))));
    std::atomic<std::uint64_t> next{0};
    std::atomic<bool> bad{false};
    auto worker = [&] {
        for (;;) {
            const std::uint64_t k = next.fetch_add(1);
            if (k >= pieces || bad) return;
            std::uint64_t off = k * kPiece;
            const std::uint64_t end = std::min(size, off + kPiece);
            while (off < end) {
                const ssize_t r = ::pread(fd, static_cast<char*>(buf) + off, end - off, static_cast<off_t>(off));
                if (r < 0 && errno == EINTR) continue;
                if (r <= 0) {
                    bad = true;
                    return;
                }
                off += static_cast<std::uint64_t>(r);
            }
        }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    ::close(fd);
    if (bad) {
        if (pin) cudaFreeHost(buf);
        else std::free(buf);
        return io_fail(std::string("read failed: ") + path);
    }
    *data = static_cast<std::uint8_t*>(buf);
    *n = size;
    return ACG_OK;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

}  // namespace

extern "C" {

int acg_load_input(const char* path, uint8_t** data, uint64_t* n) {
    if (!path || !data || !n) return acg_internal_set_error(ACG_ERR_INVALID, "null argument");
    return read_file(path, data, n, true);
}

void acg_host_free(void* p) {
    if (!p) return;
    if (is_pinned(p)) cudaFreeHost(p);
    else std::free(p);
}

int acg_load_patterns(const char* path, uint8_t** concat, uint64_t** offsets, uint32_t* count, uint64_t* duplicates,
                      uint64_t* skipped_empty) {
    if (!path || !concat || !offsets || !count) return acg_internal_set_error(ACG_ERR_INVALID, "null argument");
    *concat = nullptr;
    *offsets = nullptr;
    *count = 0;
    std::uint8_t* raw = nullptr;
    std::uint64_t n = 0;
    if (const int rc = read_file(path, &raw, &n, false)) return rc;
    const std::string_view text(reinterpret_cast<const char*>(raw), n);
    std::unordered_set<std::string_view> seen;
    std::vector<std::uint64_t> offs{0};
    std::vector<std::uint8_t> bytes;
    std::uint64_t dups = 0, empty = 0;
    std::size_t start = 0;
    while (start < text.size()) {
        const std::size_t nl = text.find('\n', start);
        std::string_view line = nl == std::string_view::npos ? text.substr(start) : text.substr(start, nl - start);
        start = nl == std::string_view::npos ? text.size() : nl + 1;
        if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
        if (line.empty()) {
            ++empty;
            continue;
        }
        if (!seen.insert(line).second) {
            ++dups;
            continue;
        }
        bytes.insert(bytes.end(), line.begin(), line.end());
        offs.push_back(bytes.size());
    }
    const std::size_t P = offs.size() - 1;
    if (P == 0) {
        std::free(raw);
        return acg_internal_set_error(ACG_ERR_EMPTY_DICTIONARY, (std::string("no patterns in ") + path).c_str());
    }
    if (P >= 0xFFFFFFFFull) {
        std::free(raw);
        return acg_internal_set_error(ACG_ERR_INVALID, "too many patterns");
    }
    *concat = static_cast<std::uint8_t*>(std::malloc(std::max<std::size_t>(bytes.size(), 1)));
    *offsets = static_cast<std::uint64_t*>(std::malloc(offs.size() * sizeof(std::uint64_t)));
    if (!*concat || !*offsets) {
        std::free(*concat);
        std::free(*offsets);
        std::free(raw);
        *concat = nullptr;
        *offsets = nullptr;
        return acg_internal_set_error(ACG_ERR_OUT_OF_MEMORY, "host allocation failed");
    }
    if (!bytes.empty()) std::memcpy(*concat, bytes.data(), bytes.size());
    std::memcpy(*offsets, offs.data(), offs.size() * sizeof(std::uint64_t));
    *count = static_cast<std::uint32_t>(P);
    if (duplicates) *duplicates = dups;
    if (skipped_empty) *skipped_empty = empty;
    std::free(raw);
    return ACG_OK;
}

}  // extern "C"

namespace {

// The pipeline of acg_scan_pipelined / acg_scan_stream: pieces alternate
// between two pooled scanners; on_piece(scanner, piece matches, matches
// before the piece) consumes each synced piece in text order.
int run_pipeline(const acg_automaton* a, int device, const uint8_t* h_text, uint64_t n, uint64_t emit_from,
                 uint64_t base_offset, uint64_t piece_bytes, uint32_t flags, bool want_list, uint64_t* h_counts,
                 uint64_t* failure_follows, const std::function<int(acg_scanner*, uint64_t, uint64_t)>& on_piece,
                 uint64_t* m_out) {
    if (!a || (!h_text && n) || !m_out) return acg_internal_set_error(ACG_ERR_INVALID, "null argument");
    if (emit_from > n || (emit_from & 15)) return acg_internal_set_error(ACG_ERR_INVALID, "emit_from must be a multiple of 16 inside the text");
    *m_out = 0;
    if (failure_follows) *failure_follows = 0;
    const std::uint32_t P = acg_pattern_count(a);
    if (h_counts) std::fill(h_counts, h_counts + P, 0ull);
    std::uint32_t halo = 0;
    if (const int rc = acg_automaton_layout(a, nullptr, nullptr, nullptr, &halo, nullptr)) return rc;
    const std::uint64_t ctx_max = (static_cast<std::uint64_t>(halo) + 15) & ~15ull;
    if (piece_bytes == 0) piece_bytes = 256ull << 20;
    piece_bytes = std::max<std::uint64_t>((piece_bytes + 15) & ~15ull, std::max<std::uint64_t>(16, 4 * ctx_max));
    const std::uint64_t owned = n - emit_from;
    const std::uint64_t pieces = owned ? (owned + piece_bytes - 1) / piece_bytes : 0;
    const std::uint32_t sflags = (want_list ? ACG_SCAN_LIST : 0u) | (h_counts ? ACG_SCAN_COUNTS : 0u) |
                                 (flags & ACG_SCAN_STATS);
    int rc = cudaSetDevice(device) == cudaSuccess ? ACG_OK : acg_internal_set_error(ACG_ERR_NO_DEVICE, "bad device");
    if (rc) return rc;
    const bool pinned = owned && is_pinned(h_text);
    acg_internal_auto_layout(const_cast<acg_automaton*>(a), h_text + emit_from, owned);

    struct Lane {
        acg_scanner* s = nullptr;
        cudaStream_t st = nullptr;
        std::uint8_t* d = nullptr;
        std::uint8_t* stage = nullptr;  // pinned staging (pageable input)
        std::uint64_t lo = 0, hi = 0;   // owned text range of the piece in flight
    } lane[2];
    std::vector<std::uint64_t> piece_counts(h_counts ? P : 0);
    std::uint64_t m = 0;
    const std::uint64_t dev_bytes = piece_bytes + ctx_max + 16;
    auto cleanup = [&] {
        for (auto& l : lane) {
            if (l.d) cudaFreeAsync(l.d, l.st);
            if (l.st) cudaStreamSynchronize(l.st);  // (the scanner's own stream: it stays with the scanner)
            if (l.stage) cudaFreeHost(l.stage);
            if (l.s) {
                if (rc == ACG_OK) acg_internal_scanner_give(l.s);
                else acg_scanner_destroy(l.s);
            }
        }
    };
    auto cuda_fail = [&](cudaError_t e) {
        cudaGetLastError();
        return acg_internal_set_error(e == cudaErrorMemoryAllocation ? ACG_ERR_OUT_OF_MEMORY : ACG_ERR_CUDA,
                                      cudaGetErrorString(e));
    };
    for (int i = 0; i < 2 && i < static_cast<int>(pieces); ++i) {
        auto& l = lane[i];
        if ((rc = acg_internal_scanner_take(a, device, sflags | kPipelineTag, &l.s))) break;
        l.st = static_cast<cudaStream_t>(acg_internal_scanner_stream(l.s));
        if (cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&l.d), dev_bytes, l.st)) {
            rc = cuda_fail(e);
            break;
        }
        if (!pinned) {
            if (cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&l.stage), dev_bytes, cudaHostAllocDefault)) {
                rc = cuda_fail(e);
                break;
            }
        }
    }
    // enqueue piece k on lane k % 2: H2D of [lo - ctx, hi), scan with emit_from = ctx
    auto enqueue = [&](std::uint64_t k) -> int {
        auto& l = lane[k % 2];
        l.lo = emit_from + k * piece_bytes;
        l.hi = std::min(n, l.lo + piece_bytes);
        const std::uint64_t ctx = std::min(l.lo, ctx_max);
        const std::uint64_t len = l.hi - l.lo + ctx;
        const std::uint8_t* src = h_text + (l.lo - ctx);
        if (!pinned) {
            std::memcpy(l.stage, src, len);  // (after this lane's previous copy completed: drained below)
            src = l.stage;
        }
        if (cudaError_t e = cudaMemcpyAsync(l.d, src, len, cudaMemcpyHostToDevice, l.st)) return cuda_fail(e);
        return acg_scanner_run(l.s, l.d, len, ctx, base_offset + (l.lo - ctx), l.st);
    };
    // drain the piece a lane holds: its records (on_piece), counts, follows
    auto drain = [&](Lane& l) -> int {
        if (int r = acg_scanner_sync(l.s)) return r;
        const std::uint64_t pm = acg_scanner_match_count(l.s);
        if (int r = on_piece(l.s, pm, m)) return r;
        if (h_counts) {
            if (int r = acg_scanner_pattern_counts(l.s, piece_counts.data())) return r;
            for (std::uint32_t p = 0; p < P; ++p) h_counts[p] += piece_counts[p];
        }
        if (failure_follows && (flags & ACG_SCAN_STATS)) *failure_follows += acg_scanner_failure_follows(l.s);
        m += pm;
        if (!pinned) cudaStreamSynchronize(l.st);  // the staging buffer is free again
        return ACG_OK;
    };
    for (std::uint64_t k = 0; !rc && k < std::min<std::uint64_t>(pieces, 2); ++k) rc = enqueue(k);
    for (std::uint64_t k = 0; !rc && k < pieces; ++k) {
        rc = drain(lane[k % 2]);
        if (!rc && k + 2 < pieces) rc = enqueue(k + 2);
    }
    cleanup();
    if (!rc) *m_out = m;
    return rc;
}

std::uint32_t id_bits_of(const acg_automaton* a) {  // (automaton.cpp: compile_dfa)
    const std::uint32_t P = acg_pattern_count(a);
    std::uint32_t ib = 1;
    while ((1ull << ib) < P) ++ib;
    return ib;
}

}  // namespace

extern "C" {

int acg_scan_pipelined(const acg_automaton* a, int device, const uint8_t* h_text, uint64_t n, uint64_t emit_from,
                       uint64_t base_offset, uint64_t piece_bytes, uint32_t flags, uint64_t* h_packed, uint64_t cap,
                       uint64_t* h_counts, uint64_t* m_out, uint32_t* id_bits, uint64_t* failure_follows) {
    const bool want_list = h_packed != nullptr;
    const int rc = run_pipeline(
        a, device, h_text, n, emit_from, base_offset, piece_bytes, flags, want_list, h_counts, failure_follows,
        [&](acg_scanner* s, std::uint64_t pm, std::uint64_t m) -> int {
            if (!want_list || m >= cap || !pm) return ACG_OK;
            return acg_scanner_copy_records(s, 0, std::min(pm, cap - m), h_packed + m);
        },
        m_out);
    if (!rc && id_bits) *id_bits = id_bits_of(a);
    return rc;
}

int acg_scan_stream(const acg_automaton* a, int device, const uint8_t* h_text, uint64_t n, uint64_t piece_bytes,
                    int format, acg_sink sink, void* user, uint64_t* h_counts, uint64_t* m_out, uint32_t* id_bits) {
    if (!sink) return acg_internal_set_error(ACG_ERR_INVALID, "null sink");
    if (format != -1 && format != ACG_FORMAT_TSV && format != ACG_FORMAT_JSON)
        return acg_internal_set_error(ACG_ERR_INVALID, "unknown output format");
    constexpr std::uint64_t kWindow = 1ull << 24;  // records per window handed to the sink
    const bool json = format == ACG_FORMAT_JSON;
    // page-locked staging: two windows (JSON holds the last one back: its final
    // "," becomes "]" once the stream's end is known)
    std::uint8_t* buf[2] = {nullptr, nullptr};
    std::uint64_t cap[2] = {0, 0}, held = 0;
    int hb = -1;  // buffer holding a window not yet handed over (JSON)
    auto grow = [&](int i, std::uint64_t need) -> int {
        if (need <= cap[i]) return ACG_OK;
        if (buf[i]) cudaFreeHost(buf[i]);
        cap[i] = need + need / 8 + 16;  // (+16: the held JSON window's closing "]\n" always fits in place)
        if (cudaHostAlloc(reinterpret_cast<void**>(&buf[i]), cap[i], cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            buf[i] = nullptr;
            cap[i] = 0;
            return acg_internal_set_error(ACG_ERR_OUT_OF_MEMORY, "pinned staging allocation failed");
        }
        return ACG_OK;
    };
    int next = 0;
    const int rc = run_pipeline(
        a, device, h_text, n, 0, 0, piece_bytes, 0, true, h_counts, nullptr,
        [&](acg_scanner* s, std::uint64_t pm, std::uint64_t m) -> int {
            for (std::uint64_t first = 0; first < pm; first += kWindow) {
                const std::uint64_t count = std::min(kWindow, pm - first);
                if (format < 0) {
                    if (int r = grow(0, count * 8)) return r;
                    if (int r = acg_scanner_copy_records(s, first, count, reinterpret_cast<std::uint64_t*>(buf[0])))
                        return r;
                    if (sink(user, buf[0], count)) return acg_internal_set_error(ACG_ERR_INVALID, "sink stopped the scan");
                    continue;
                }
                std::uint64_t nb = 0;
                const int open = json && m + first == 0;
                if (int r = acg_internal_format(s, json, first, count, open, 0, nullptr, 0, &nb)) return r;
                if (int r = grow(next, nb)) return r;
                if (int r = acg_internal_fetch(s, buf[next], nb)) return r;
                if (!json) {
                    if (nb && sink(user, buf[next], nb)) return acg_internal_set_error(ACG_ERR_INVALID, "sink stopped the scan");
                    continue;
                }
                if (hb >= 0 && sink(user, buf[hb], held)) return acg_internal_set_error(ACG_ERR_INVALID, "sink stopped the scan");
                hb = next;
                held = nb;
                next ^= 1;
            }
            return ACG_OK;
        },
        m_out);
    int out = rc;
    if (!out && json) {
        if (hb < 0) {
            static const std::uint8_t empty[] = {'[', ']', '\n'};
            if (sink(user, empty, 3)) out = acg_internal_set_error(ACG_ERR_INVALID, "sink stopped the scan");
        } else {
            // the last record's "," closes the list (cap >= held + 16: room for the "\n")
            buf[hb][held - 1] = ']';
            buf[hb][held] = '\n';
            if (sink(user, buf[hb], held + 1)) out = acg_internal_set_error(ACG_ERR_INVALID, "sink stopped the scan");
        }
    }
    for (auto* b : buf)
        if (b) cudaFreeHost(b);
    if (!out && id_bits) *id_bits = id_bits_of(a);
    return out;
}

}  // extern "C"
