// Filter-mode kernels (sampled q-gram prefilter + exact block walks; the
// scheme and its exactness argument are in qfilter.hpp).
//
//  * qfilter_kernel (KQ) streams the text once at HBM rate. Each lane owns a
//    16-byte word; 32 lanes cover 512 contiguous bytes (coalesced), a warp
//    takes D such segments per batch, double-buffered one batch ahead. The
//    word's 2-bit codes are packed into 32 bits; the next word's codes come
//    from the neighbour lane (shuffle), so the q-grams at the word's four
//    samples (offsets 0, 4, 8, 12) are funnel shifts of one 64-bit value.
//    Each q-gram probes Bloom stage 0 in shared memory (one LDS per 4 text
//    bytes); the rare survivors probe stages 1 and 2 and, if they pass, set
//    the dirty bits of the 64-byte blocks their matches could end in.
//    Non-ACGT bytes need no check: no occurrence contains one, so a q-gram
//    over them can only cause a (harmless) extra walk.
//  * qverify_count_kernel (V1): per dirty-bitmap word, every dirty block is
//    walked with the exact DFA from `halo` bytes before it (root start, so
//    the state is exact inside the block); matches ending in the block are
//    counted (per block, per 8 KiB chunk, per output state for K4).
//  * qverify_write_kernel (V2): one warp per chunk with matches; lanes take
//    the chunk's dirty blocks in order, a warp scan of the block counts gives
//    each block its slot range, and the block is walked again to write its
//    records — so records come out in (end, id) order with no sort.
#pragma once

#include "qfilter.hpp"
#include "scan_kernels.cuh"

namespace acg {
namespace kern {

__device__ __forceinline__ bool qpass(const std::uint32_t* tab, std::uint32_t c) {
    std::uint32_t h = qhash0(c);
    if (!((tab[h >> 5] >> (h & 31u)) & 1u)) return false;
    h = qhash1(c);
    if (!((tab[kQOff1 + (h >> 5)] >> (h & 31u)) & 1u)) return false;
    h = qhash2(c);
    return (tab[kQOff2 + (h >> 5)] >> (h & 31u)) & 1u;
}

// Sample j passed: mark the blocks of [emit_from, n) holding the ends its
// matches could have, [j+q-1, j+maxlen-1]. (Scalars by value: a reference to
// the kernel parameter block would force a per-thread local copy of it.)
__device__ __noinline__ void qmark(long long j, long long q, long long max_len, long long emit_from, long long n,
                                   std::uint32_t* dirty, unsigned long long* ev_total) {
    long long lo = j + q - 1, hi = j + max_len - 1;
    if (lo < emit_from) lo = emit_from;
    if (hi > n - 1) hi = n - 1;
    if (lo > hi) return;
    const unsigned long long b0 = static_cast<unsigned long long>(lo - emit_from) >> 6;
    const unsigned long long b1 = static_cast<unsigned long long>(hi - emit_from) >> 6;
    for (unsigned long long b = b0; b <= b1; ++b) atomicOr(dirty + (b >> 5), 1u << (b & 31u));
    if (ev_total) atomicAdd(ev_total, 1ull);
}

// 16 text bytes -> 16 2-bit codes (byte k at bits 2k); no validation.
__device__ __forceinline__ std::uint32_t qcodes(const uint4& w) {
    const std::uint32_t m0 = ((w.x >> 1) & 0x03030303u) * 0x01041040u, m1 = ((w.y >> 1) & 0x03030303u) * 0x01041040u;
    const std::uint32_t m2 = ((w.z >> 1) & 0x03030303u) * 0x01041040u, m3 = ((w.w >> 1) & 0x03030303u) * 0x01041040u;
    return __byte_perm(__byte_perm(m0, m1, 0x0073u), __byte_perm(m2, m3, 0x7300u), 0x7610u);
}

__device__ __forceinline__ uint4 qload(const std::uint8_t* text, long long wi, long long W) {
    return wi < W ? ldg_text(text + 16 * wi) : make_uint4(0, 0, 0, 0);
}

template <int D>
__global__ void __launch_bounds__(512, 1) qfilter_kernel(const ScanArgs a) {
    std::uint32_t* tab = reinterpret_cast<std::uint32_t*>(acg_hot_smem);
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.qbloom);
        uint4* dst = reinterpret_cast<uint4*>(tab);
        for (std::uint32_t i = threadIdx.x; i < kQWords / 4; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long W = (a.n + 15) >> 4;
    const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    const long long wid = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const std::uint32_t qm = a.q >= 16 ? 0xFFFFFFFFu : (1u << (2 * a.q)) - 1u;
    constexpr long long kBatch = 32LL * D;  // words per warp batch
    const long long stride = warps * kBatch;

    // buffers: D words per lane + the word after the batch (lane 31 only)
    auto load = [&](uint4 (&w)[D], uint4& x, long long b0) {
#pragma unroll
        for (int d = 0; d < D; ++d) w[d] = qload(a.text, b0 + 32 * d + lane, W);
        x = lane == 31 ? qload(a.text, b0 + kBatch, W) : make_uint4(0, 0, 0, 0);
    };
    auto process = [&](const uint4 (&w)[D], const uint4& x, long long b0) {
        std::uint32_t code[D + 1];
#pragma unroll
        for (int d = 0; d < D; ++d) code[d] = qcodes(w[d]);
        code[D] = qcodes(x);
#pragma unroll
        for (int d = 0; d < D; ++d) {
            std::uint32_t nc = __shfl_down_sync(0xFFFFFFFFu, code[d], 1);
            const std::uint32_t first_next = d + 1 < D ? __shfl_sync(0xFFFFFFFFu, code[d + 1 < D ? d + 1 : d], 0)
                                                       : code[D];
            if (lane == 31) nc = first_next;
            const long long P = 16 * (b0 + 32 * d + lane);
            if (P >= a.n) continue;
            const unsigned long long comb = static_cast<unsigned long long>(nc) << 32 | code[d];
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                const std::uint32_t c = static_cast<std::uint32_t>(comb >> (8 * o)) & qm;
                if (qpass(tab, c)) qmark(P + 4 * o, a.q, a.max_len, a.emit_from, a.n, a.dirty, a.ev_total);
            }
        }
    };

    long long b0 = wid * kBatch;
    if (b0 >= W) return;
    uint4 wa[D], wb[D], xa, xb;
    load(wa, xa, b0);
    for (;;) {
        const long long b1 = b0 + stride;
        if (b1 < W) load(wb, xb, b1);
        process(wa, xa, b0);
        if (b1 >= W) break;
        const long long b2 = b1 + stride;
        if (b2 < W) load(wa, xa, b2);
        process(wb, xb, b1);
        if (b2 >= W) break;
        b0 = b2;
    }
}

// Exact walk of dirty block b (bytes [emit_from + 64b, +64)): from the root
// `halo` bytes earlier; hot rows [0, hot_rows) from shared memory (`tab`),
// the rest from the L2-resident table.
template <int PASS>
__device__ __forceinline__ void qwalk_block(long long b, std::uint32_t tab, unsigned long long& cnt,
                                         unsigned long long& wr, const ScanArgs& a) {
    const long long pb = a.emit_from + b * static_cast<long long>(kQBlock);
    const long long pe = min(pb + static_cast<long long>(kQBlock), a.n);
    long long p = pb - a.halo;
    if (p < 0) p = 0;
    std::uint32_t s = 0;
    for (; p < pe; ++p) {
        const int col = text_col(a, p);
        if (col < 0) {
            s = 0;
            continue;
        }
        std::uint32_t v = s < a.hot_rows ? lds_u16(tab + 2u * (s * 4u + static_cast<std::uint32_t>(col))) : kEsc16;
        if (v == kEsc16) v = __ldg(a.next + s * 4u + static_cast<std::uint32_t>(col));
        s = v;
        if (p >= pb && s >= a.Hn && has_out(s, a)) emit<PASS>(s, p, cnt, wr, a);
    }
}

__device__ __forceinline__ std::uint32_t stage_hot_rows(const ScanArgs& a) {
    extern __shared__ __align__(16) std::uint8_t smem[];
    const std::uint32_t bytes = a.hot_rows * 8u;  // 4 columns of u16
    const uint4* src = reinterpret_cast<const uint4*>(a.hot16);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (std::uint32_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
    return smem_u32(smem);
}

// V1: count walks of every dirty block (thread per dirty-bitmap word).
__global__ void __launch_bounds__(256) qverify_count_kernel(const ScanArgs a, long long n_dwords) {
    const std::uint32_t tab = stage_hot_rows(a);
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_dwords; i += stride) {
        std::uint32_t bits = a.dirty[i];
        while (bits) {
            const long long b = i * 32 + (__ffs(bits) - 1);
            bits &= bits - 1;
            unsigned long long cnt = 0, wr = 0;
            qwalk_block<kCount>(b, tab, cnt, wr, a);
            a.block_count[b] = static_cast<std::uint32_t>(cnt);
            if (cnt) atomicAdd(a.chunk_counts + (b / kQChunkBlocks), cnt);
        }
    }
}

// V2: ordered record writes, one warp per chunk with matches.
__global__ void __launch_bounds__(256) qverify_write_kernel(const ScanArgs a) {
    const long long n_work = static_cast<long long>(*a.active_count);
    const long long warps_per_block = blockDim.x >> 5;
    if (static_cast<long long>(blockIdx.x) * warps_per_block >= n_work) return;
    const std::uint32_t tab = stage_hot_rows(a);
    const int lane = threadIdx.x & 31;
    const long long stride = static_cast<long long>(gridDim.x) * warps_per_block;
    for (long long t = static_cast<long long>(blockIdx.x) * warps_per_block + (threadIdx.x >> 5); t < n_work;
         t += stride) {
        const long long c = a.active_list[t];
        unsigned long long base = a.chunk_offs[c];
#pragma unroll 1
        for (int w = 0; w < static_cast<int>(kQChunkBlocks / 32); ++w) {
            const long long wi = c * (kQChunkBlocks / 32) + w;
            const std::uint32_t bits = a.dirty[wi];
            const long long b = wi * 32 + lane;
            const std::uint32_t cnt = ((bits >> lane) & 1u) ? a.block_count[b] : 0u;
            std::uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const std::uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += v;
            }
            if (cnt) {
                unsigned long long wr = base + incl - cnt, dummy = 0;
                qwalk_block<kWrite>(b, tab, dummy, wr, a);
            }
            base += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
    }
}

}  // namespace kern
}  // namespace acg
