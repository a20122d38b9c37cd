// Filter-mode kernels (sampled q-gram prefilter; the scheme and its
// exactness argument are in qfilter.hpp).
//
//  * qfilter_kernel (KQ) streams the text once at HBM rate. Each lane owns
//    32 bytes (one 256-bit load); 32 lanes cover 1 KiB contiguous (coalesced),
//    a warp streams its own contiguous region in batches of D such segments,
//    double-buffered one batch ahead. Each 16-byte half's 2-bit codes are
//    packed into 32 bits; the next lane's first half comes by shuffle, so the
//    q-grams at the eight samples (offsets 0, 4, .., 28) are funnel shifts of
//    two 64-bit values. Each q-gram costs one shared-memory probe of the
//    blocked Bloom filter (one 32-bit word, four bits), branch-free; survivors (rare) are
//    appended to a candidate list with one warp-aggregated atomic (a full
//    list is detected at sync and the scan re-run with a larger one).
//    Non-ACGT bytes need no check here: no occurrence contains one, so a
//    q-gram over them can only make a (harmless) extra candidate.
//  * qconfirm_kernel (V0) confirms each survivor exactly — the q-gram's
//    (pattern, offset) list from a hash table, then a byte compare at
//    i = j - offset — and so enumerates every occurrence exactly once (by
//    its owned sample). Count pass: per-chunk and per-pattern counts, the
//    packed records into a scratch list; write pass (record-buffer regrowth
//    only): records straight into their chunk's slot range.
//  * qscatter_kernel moves the scratch records into their chunk's slot range
//    (K2 prefix) and qsort_chunks_kernel orders each chunk's records (warp
//    bitonic sort of up to 32); a chunk with more records is replayed by
//    qheavy_kernel with the exact chunk walk, which writes them in order.
#pragma once

#include "qfilter.hpp"
#include "scan_kernels.cuh"

namespace acg {
namespace kern {

// 16 text bytes -> 16 2-bit codes (byte k at bits 2k); no validation.
__device__ __forceinline__ std::uint32_t qcodes(const uint4& w) {
    const std::uint32_t m0 = ((w.x >> 1) & 0x03030303u) * 0x01041040u, m1 = ((w.y >> 1) & 0x03030303u) * 0x01041040u;
    const std::uint32_t m2 = ((w.z >> 1) & 0x03030303u) * 0x01041040u, m3 = ((w.w >> 1) & 0x03030303u) * 0x01041040u;
    return __byte_perm(__byte_perm(m0, m1, 0x0073u), __byte_perm(m2, m3, 0x7300u), 0x7610u);
}

// KQ geometry: lane = 32 text bytes (two 16-byte words); segment = 32 lanes
// = 1 KiB; batch = D contiguous segments. Each warp streams its own
// contiguous region of batches, double-buffered one batch ahead.
template <int D, int TPB>
__global__ void __launch_bounds__(TPB, 1) qfilter_kernel(const ScanArgs a) {
    std::uint32_t* tab = reinterpret_cast<std::uint32_t*>(acg_hot_smem);
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.qbloom);
        uint4* dst = reinterpret_cast<uint4*>(tab);
        for (std::uint32_t i = threadIdx.x; i < kQWords / 4; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    constexpr long long kSeg = 1024, kBatch = kSeg * D;  // bytes
    const long long n = a.n;
    const long long n_batches = (n + kBatch - 1) / kBatch;
    const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    const long long wid = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long per = (n_batches + warps - 1) / warps;
    const long long bat0 = wid * per, bat1 = min(bat0 + per, n_batches);
    if (bat0 >= bat1) return;
    const std::uint32_t qm = a.q >= 16 ? 0xFFFFFFFFu : (1u << (2 * a.q)) - 1u;
    const std::uint8_t* text = a.text;
    const bool al32 = (reinterpret_cast<std::uintptr_t>(text) & 31u) == 0;  // 256-bit loads need 32-byte alignment

    // 0 iff the q-gram passes the Bloom filter
    auto probe = [&](std::uint32_t c) -> std::uint32_t { return qmask(c) & ~tab[qword(c)]; };
    auto gram = [&](std::uint32_t lo, std::uint32_t hi, int o) -> std::uint32_t {
        return (o == 0 ? lo : __funnelshift_r(lo, hi, 8 * o)) & qm;
    };
    struct Lane {
        uint4 lo, hi;
    };
    auto load = [&](Lane (&w)[D], long long base) {
        if (al32 && base + kBatch <= n) {  // interior batch: unchecked 256-bit loads
#pragma unroll
            for (int d = 0; d < D; ++d) ldg_text32(text + base + kSeg * d + 32 * lane, w[d].lo, w[d].hi);
        } else {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const long long p = base + kSeg * d + 32 * lane;
                w[d].lo = p < n ? ldg_text(text + p) : make_uint4(0, 0, 0, 0);
                w[d].hi = p + 16 < n ? ldg_text(text + p + 16) : make_uint4(0, 0, 0, 0);
            }
        }
    };
    auto process = [&](const Lane (&w)[D], long long base) {
        const long long after = base + kBatch;  // the word after the batch (lane 31 of the last segment)
        const uint4 xw = (lane == 31 && after < n) ? ldg_text(text + after) : make_uint4(0, 0, 0, 0);
        std::uint32_t c0[D + 1], c1[D], z[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            c0[d] = qcodes(w[d].lo);
            c1[d] = qcodes(w[d].hi);
        }
        c0[D] = qcodes(xw);
#pragma unroll
        for (int d = 0; d < D; ++d) {
            std::uint32_t nc = __shfl_down_sync(0xFFFFFFFFu, c0[d], 1);
            const std::uint32_t first_next = __shfl_sync(0xFFFFFFFFu, c0[d + 1], 0);
            if (lane == 31) nc = d + 1 < D ? first_next : c0[D];
            std::uint32_t t = probe(gram(c0[d], c1[d], 0));
#pragma unroll
            for (int o = 1; o < 4; ++o) t = min(t, probe(gram(c0[d], c1[d], o)));
#pragma unroll
            for (int o = 0; o < 4; ++o) t = min(t, probe(gram(c1[d], nc, o)));
            z[d] = base + kSeg * d + 32 * lane < n ? t : 1u;
            c1[d] = nc;  // keep the neighbour code for the rare path (c1 is recomputed there)
        }
        // survivors -> the candidate list (warp-aggregated; rare)
#pragma unroll
        for (int d = 0; d < D; ++d) {
            if (!__ballot_sync(0xFFFFFFFFu, z[d] == 0u)) continue;
            std::uint32_t pm = 0;
            if (z[d] == 0u) {
                const std::uint32_t h1 = qcodes(w[d].hi);
#pragma unroll
                for (int o = 0; o < 4; ++o) pm |= (probe(gram(c0[d], h1, o)) == 0u ? 1u : 0u) << o;
#pragma unroll
                for (int o = 0; o < 4; ++o) pm |= (probe(gram(h1, c1[d], o)) == 0u ? 1u : 0u) << (4 + o);
            }
            const std::uint32_t k = __popc(pm);
            std::uint32_t incl = k;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const std::uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += v;
            }
            std::uint32_t slot = 0;
            if (lane == 31) slot = atomicAdd(a.qcand_n, incl);
            slot = __shfl_sync(0xFFFFFFFFu, slot, 31) + incl - k;
            const long long P = base + kSeg * d + 32 * lane;
            for (std::uint32_t m = pm; m; m &= m - 1, ++slot) {
                const long long j = P + 4 * (__ffs(m) - 1);
                if (slot < a.qcand_cap) a.qcands[slot] = static_cast<unsigned long long>(j);
            }
        }
    };

    long long b = bat0;
    Lane wa[D], wb[D];
    load(wa, b * kBatch);
    for (;;) {
        const bool more1 = b + 1 < bat1;
        if (more1) load(wb, (b + 1) * kBatch);
        process(wa, b * kBatch);
        if (!more1) break;
        const bool more2 = b + 2 < bat1;
        if (more2) load(wa, (b + 2) * kBatch);
        process(wb, (b + 1) * kBatch);
        if (!more2) break;
        b += 2;
    }
}

// V0: exact confirmation of the survivors (see the header comment).
template <int PASS>
__global__ void __launch_bounds__(256) qconfirm_kernel(const ScanArgs a) {
    const long long n_c = min(static_cast<long long>(*a.qcand_n), static_cast<long long>(a.qcand_cap));
    const std::uint32_t tmask = (1u << a.qtab_bits) - 1u;
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n_c;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long j = static_cast<long long>(a.qcands[t]);
        if (j + static_cast<long long>(a.q) > a.n) continue;
        std::uint32_t code = 0;
        bool ok = true;
        for (std::uint32_t k = 0; k < a.q; ++k) {
            const std::uint32_t b = a.text[j + k];
            ok = ok && (b == 'A' || b == 'C' || b == 'G' || b == 'T');
            code |= ((b >> 1) & 3u) << (2 * k);
        }
        if (!ok) continue;
        std::uint32_t slot = qslot(code, a.qtab_bits), bucket = kQEmpty;
        for (;;) {
            const uint2 e = *reinterpret_cast<const uint2*>(a.qtab + 2 * slot);
            if (e.y == kQEmpty) break;
            if (e.x == code) {
                bucket = e.y;
                break;
            }
            slot = (slot + 1) & tmask;
        }
        if (bucket == kQEmpty) continue;
        for (std::uint32_t e = a.qb_off[bucket]; e < a.qb_off[bucket + 1]; ++e) {
            const std::uint32_t ent = a.qb_ent[e];
            const long long i = j - static_cast<long long>(ent & 3u);
            const std::uint32_t p = ent >> 2;
            const std::uint32_t lo = a.pat_off[p], len = a.pat_off[p + 1] - lo;
            if (i < 0 || i + len > a.n) continue;
            const long long end = i + len - 1;
            if (end < a.emit_from) continue;
            bool eq = true;
            for (std::uint32_t k = 0; k < len && eq; ++k) eq = a.text[i + k] == a.pat_bytes[lo + k];
            if (!eq) continue;
            const long long c = (end - a.emit_from) / a.chunk;
            const unsigned long long key = ((a.base + static_cast<unsigned long long>(end)) << a.id_bits) | p;
            if (PASS == kCount) {
                atomicAdd(a.chunk_counts + c, 1ull);
                if (a.pcounts) atomicAdd(a.pcounts + p, 1ull);
                if (a.qscratch) {
                    const unsigned long long w = atomicAdd(a.qscratch_n, 1ull);
                    if (w < a.rec_cap) a.qscratch[w] = key;
                }
            } else {
                const unsigned long long w = a.chunk_offs[c] + atomicAdd(a.qfill + c, 1u);
                if (w < a.rec_cap) a.records[w] = key;
            }
        }
    }
}

// Scratch records -> their chunk's slot range (unordered within the chunk).
__global__ void __launch_bounds__(256) qscatter_kernel(const ScanArgs a) {
    const unsigned long long n = min(*a.qscratch_n, a.rec_cap);
    for (unsigned long long t = blockIdx.x * 256ull + threadIdx.x; t < n; t += gridDim.x * 256ull) {
        const unsigned long long key = a.qscratch[t];
        const long long end = static_cast<long long>((key >> a.id_bits) - a.base);
        const long long c = (end - a.emit_from) / a.chunk;
        const unsigned long long w = a.chunk_offs[c] + atomicAdd(a.qfill + c, 1u);
        if (w < a.rec_cap) a.records[w] = key;
    }
}

// Orders each chunk's records: warp bitonic sort when the chunk has <= 32;
// bigger chunks go to the heavy list (qheavy_kernel).
__global__ void __launch_bounds__(256) qsort_chunks_kernel(const ScanArgs a, std::uint32_t* heavy,
                                                           std::uint32_t* n_heavy) {
    const long long n_work = static_cast<long long>(*a.active_count);
    const int lane = threadIdx.x & 31;
    const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    for (long long t = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); t < n_work;
         t += warps) {
        const long long c = a.active_list[t];
        const unsigned long long lo = a.chunk_offs[c], k = a.chunk_offs[c + 1] - lo;
        if (k <= 1) continue;
        if (k > 32) {
            if (lane == 0) heavy[atomicAdd(n_heavy, 1u)] = static_cast<std::uint32_t>(c);
            continue;
        }
        if (lo + k > a.rec_cap) continue;  // record buffer overflowed: re-emitted after regrowth
        unsigned long long v = lane < static_cast<int>(k) ? a.records[lo + lane] : ~0ull;
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                const unsigned long long o = __shfl_xor_sync(0xFFFFFFFFu, v, stride);
                const bool up = (lane & size) == 0;     // this lane's run ascends
                const bool low = (lane & stride) == 0;  // lower element of its pair
                v = (low == up) ? min(v, o) : max(v, o);
            }
        }
        if (lane < static_cast<int>(k)) a.records[lo + lane] = v;
    }
}

// Chunks with more than 32 records: the exact chunk walk (A_H in shared
// memory) re-emits them in order over their slot range.
__global__ void __launch_bounds__(256, 1) qheavy_kernel(const ScanArgs a, const std::uint32_t* heavy,
                                                        const std::uint32_t* n_heavy) {
    const long long n = static_cast<long long>(*n_heavy);
    if (static_cast<long long>(blockIdx.x) * blockDim.x >= n) return;
    extern __shared__ __align__(16) std::uint8_t smem[];
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.hotH);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (std::uint32_t i = threadIdx.x; i < a.smem_table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const std::uint32_t tab = smem_u32(smem);
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x)
        exact_chunk_walk<kWrite>(heavy[t], tab, a);
}

}  // namespace kern
}  // namespace acg
