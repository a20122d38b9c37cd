// Filter-mode kernels (sampled q-gram prefilter; the scheme and its
// exactness argument are in qfilter.hpp).
//
//  * qfilter_kernel (KQ) streams the text once at HBM rate: a producer warp
//    moves the CTA's contiguous region through a ring of shared-memory stages
//    with TMA bulk copies (mbarrier full/empty pipeline, L2 evict-first);
//    consumer lanes take 32 bytes each. Each 16-byte half's 2-bit codes are
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
// (bits 1-2 of each byte gathered into the top byte by one multiply: the
// partial products of the other bytes land in disjoint bits below 24 or
// overflow, so no carries reach the top byte)
__device__ __forceinline__ std::uint32_t qcodes(const uint4& w) {
    const std::uint32_t m0 = (w.x & 0x06060606u) * 0x00820820u, m1 = (w.y & 0x06060606u) * 0x00820820u;
    const std::uint32_t m2 = (w.z & 0x06060606u) * 0x00820820u, m3 = (w.w & 0x06060606u) * 0x00820820u;
    return __byte_perm(__byte_perm(m0, m1, 0x0073u), __byte_perm(m2, m3, 0x7300u), 0x7610u);
}

// ---- bulk-copy (TMA) ring primitives --------------------------------------
__device__ __forceinline__ void mbar_init(std::uint32_t bar, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint32_t bar, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint32_t bar, std::uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// Global -> shared bulk copy (TMA engine), completion counted on `bar`; the
// text is streamed once, so it is marked evict-first in L2.
__device__ __forceinline__ void bulk_load(std::uint32_t dst, const void* src, std::uint32_t bytes, std::uint32_t bar,
                                          unsigned long long policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint4 lds128(std::uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

// KQ. Warp 0 is the producer: one lane streams the CTA's contiguous region
// of the text into a ring of NST shared-memory stages with bulk copies
// (full/empty mbarriers). Warps 1..NC consume one 1 KiB block of each stage
// (a stage = NC KiB, plus the next 16 bytes so the last word sees its
// neighbour).
template <int NC, int NST>
__global__ void __launch_bounds__(32 * (NC + 1), 1) qfilter_kernel(const ScanArgs a) {
    constexpr std::uint32_t kUnits = NC * 32, kStage = kUnits * 32, kSlot = kStage + 16;
    const std::uint32_t bloom_bytes = a.qwords * 4u;
    const std::uint32_t* tab = reinterpret_cast<const std::uint32_t*>(acg_hot_smem);
    const std::uint32_t ring = smem_u32(acg_hot_smem) + bloom_bytes;  // 16-byte aligned (qwords % 4 == 0)
    const std::uint32_t bars = ring + NST * kSlot;                     // full[NST], empty[NST]
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.qbloom);
        uint4* dst = reinterpret_cast<uint4*>(acg_hot_smem);
        for (std::uint32_t i = threadIdx.x; i < bloom_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
        if (threadIdx.x == 0) {
            for (int k = 0; k < NST; ++k) {
                mbar_init(bars + 8 * k, 1);
                mbar_init(bars + 8 * (NST + k), NC);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
    }
    __syncthreads();
    const long long n = a.n;
    const long long n_stages = (n + kStage - 1) / kStage;
    const long long per = (n_stages + gridDim.x - 1) / gridDim.x;
    const long long st0 = static_cast<long long>(blockIdx.x) * per;
    const long long its = max(0LL, min(st0 + per, n_stages) - st0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0) {  // producer
        if (lane == 0) {
            unsigned long long policy;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
            for (long long it = 0; it < its; ++it) {
                const std::uint32_t k = static_cast<std::uint32_t>(it % NST);
                if (it >= NST) mbar_wait(bars + 8 * (NST + k), static_cast<std::uint32_t>((it / NST - 1) & 1));
                const long long off = (st0 + it) * kStage;
                const std::uint32_t bytes =
                    static_cast<std::uint32_t>((min(static_cast<long long>(kSlot), n - off) + 15) & ~15LL);
                mbar_expect_tx(bars + 8 * k, bytes);
                bulk_load(ring + k * kSlot, a.text + off, bytes, bars + 8 * k, policy);
            }
        }
        return;
    }

    const std::uint32_t qsh = a.qsh;
    const std::uint32_t words = a.qwords;
#ifdef ACG_QABL_NOPROBE  // ablation: no shared-memory probe
    auto probe = [&](std::uint32_t y) -> std::uint32_t { return (qmask(y) & ~(y * 0x9E3779B1u)) | 1u; };
#else
    auto probe = [&](std::uint32_t y) -> std::uint32_t { return qmask(y) & ~tab[qword(y, words)]; };
#endif
    auto gram = [&](std::uint32_t lo, std::uint32_t hi, int o) -> std::uint32_t {
        return (o == 0 ? lo : __funnelshift_r(lo, hi, 8 * o)) * qsh;
    };
    // lane l of consumer warp w reads words l and 32+l of the warp's 1 KiB
    // block (16-byte strides: conflict-free LDS.128); word 31's neighbour is
    // word 32 (lane 0's second word), word 63's is the next block's word 0.
    const std::uint32_t blk = static_cast<std::uint32_t>(warp - 1) * 1024u;
    // survivors go to this warp's own region (no atomics on the hot path)
    const unsigned long long region = (static_cast<unsigned long long>(blockIdx.x) * NC + (warp - 1)) * a.qcand_cap;
    std::uint32_t found = 0;  // warp-uniform
    for (long long it = 0; it < its; ++it) {
        const std::uint32_t k = static_cast<std::uint32_t>(it % NST);
        mbar_wait(bars + 8 * k, static_cast<std::uint32_t>((it / NST) & 1));
#ifdef ACG_QABL_STREAM  // ablation: stream only
        __syncwarp();
        if (lane == 0) mbar_arrive(bars + 8 * (NST + k));
        continue;
#endif
        const std::uint32_t at = ring + k * kSlot + blk + 16 * lane;
        const uint4 w0 = lds128(at), w1 = lds128(at + 512);
        const uint4 nx = lane == 31 ? lds128(at + 528) : make_uint4(0, 0, 0, 0);
        const std::uint32_t c0 = qcodes(w0), c1 = qcodes(w1), cx = qcodes(nx);
        __syncwarp();
        if (lane == 0) mbar_arrive(bars + 8 * (NST + k));  // this warp is done with the slot
        std::uint32_t n0 = __shfl_down_sync(0xFFFFFFFFu, c0, 1), n1 = __shfl_down_sync(0xFFFFFFFFu, c1, 1);
        const std::uint32_t first1 = __shfl_sync(0xFFFFFFFFu, c1, 0);
        if (lane == 31) {
            n0 = first1;
            n1 = cx;
        }
        std::uint32_t t[8];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            t[o] = probe(gram(c0, n0, o));
            t[4 + o] = probe(gram(c1, n1, o));
        }
        const std::uint32_t z = min(min(min(t[0], t[1]), min(t[2], t[3])), min(min(t[4], t[5]), min(t[6], t[7])));
        const long long P0 = (st0 + it) * kStage + blk + 16 * lane, P1 = P0 + 512;
        const bool hit = z == 0u && P0 < n;
        if (!__ballot_sync(0xFFFFFFFFu, hit)) continue;
        // survivors -> the candidate list (warp-aggregated; rare)
        std::uint32_t pm = 0;
        if (hit) {
#pragma unroll
            for (int o = 0; o < 8; ++o) pm |= (t[o] == 0u ? 1u : 0u) << o;
            if (P1 >= n) pm &= 0xFu;
        }
        const std::uint32_t cnt = __popc(pm);
        std::uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += v;
        }
        std::uint32_t slot = found + incl - cnt;
        found += __shfl_sync(0xFFFFFFFFu, incl, 31);
        for (std::uint32_t m = pm; m; m &= m - 1, ++slot) {
            const int o = __ffs(m) - 1;
            if (slot < a.qcand_cap) {
                a.qcands[region + slot] = static_cast<unsigned long long>(o < 4 ? P0 + 4 * o : P1 + 4 * (o - 4));
                a.qcand_code[region + slot] = o < 4 ? gram(c0, n0, o) : gram(c1, n1, o - 4);
            }
        }
    }
    if (lane == 0) {
        a.qwarp_n[blockIdx.x * NC + (warp - 1)] = found;
        atomicAdd(a.qcand_n, found);
        atomicMax(a.qcand_max, static_cast<unsigned long long>(found));
    }
}

// V0: exact confirmation of the survivors (see the header comment).
template <int PASS>
__global__ void __launch_bounds__(256) qconfirm_kernel(const ScanArgs a) {
    const std::uint32_t tmask = (1u << a.qtab_bits) - 1u;
    const long long total = static_cast<long long>(a.qwarps) * a.qcand_cap;
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        if (static_cast<std::uint32_t>(t % a.qcand_cap) >= a.qwarp_n[t / a.qcand_cap]) continue;
        const long long j = static_cast<long long>(a.qcands[t]);
        // the survivor's q-gram code, from KQ (y holds it in the top bits)
        const std::uint32_t code = a.q >= 16 ? a.qcand_code[t] : a.qcand_code[t] >> (32 - 2 * a.q);
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
        // (KQ read any bytes as codes; the pattern compare below checks the real bytes)
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
// bigger chunks go to the heavy list (qheavy_kernel). Warps sweep the chunk
// offsets directly (no compacted list: its single counter would serialise
// thousands of same-address atomics).
__device__ __forceinline__ unsigned long long bitonic32(unsigned long long v, int lane) {
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
    return v;
}

__global__ void __launch_bounds__(256) qsort_chunks_kernel(const ScanArgs a, std::uint32_t* heavy,
                                                           std::uint32_t* n_heavy) {
    const int lane = threadIdx.x & 31;
    const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    for (long long c0 = (static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
         c0 < a.n_chunks; c0 += warps * 32) {
        const long long c = c0 + lane;
        const unsigned long long lo = c < a.n_chunks ? a.chunk_offs[c] : 0ull;
        const unsigned long long k = c < a.n_chunks ? a.chunk_offs[c + 1] - lo : 0ull;
        unsigned todo = __ballot_sync(0xFFFFFFFFu, k >= 2);
        const unsigned big = __ballot_sync(0xFFFFFFFFu, k > 32);
        if (big & (1u << lane)) heavy[atomicAdd(n_heavy, 1u)] = static_cast<std::uint32_t>(c);
        todo &= ~big;
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const unsigned long long slo = __shfl_sync(0xFFFFFFFFu, lo, src);
            const unsigned long long sk = __shfl_sync(0xFFFFFFFFu, k, src);
            if (slo + sk > a.rec_cap) continue;  // record buffer overflowed: re-emitted after regrowth
            unsigned long long v = lane < static_cast<int>(sk) ? a.records[slo + lane] : ~0ull;
            v = bitonic32(v, lane);
            if (lane < static_cast<int>(sk)) a.records[slo + lane] = v;
        }
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
