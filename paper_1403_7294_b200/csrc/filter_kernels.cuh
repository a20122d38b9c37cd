// Filter-mode kernels (sampled q-gram prefilter; the scheme and its
// exactness argument are in qfilter.hpp).
//
//  * qfilter_ldg_kernel (KQ) streams the text once at HBM rate: every warp
//    walks its own contiguous region in 2 KiB blocks with 128-bit streaming
//    loads straight into registers (R blocks in flight per warp), so all of
//    shared memory holds the Bloom filter. Each 16-byte word's 2-bit codes
//    are packed into 32 bits; the next word's codes come by shuffle, so the
//    q-grams at the samples (offsets 0, 4, 8, 12) are funnel shifts of two
//    32-bit values. Each q-gram costs one shared-memory probe of the blocked
//    Bloom filter (one 32-bit word, four bits), branch-free; survivors (rare)
//    go to the warp's own candidate region (a full region is detected at
//    sync and the scan re-run with larger ones).
//    (A TMA bulk-copy ring with a producer warp was measured first: 0.356 ms
//    per GiB against 0.260 ms for this kernel at the same Bloom size — the
//    ring's shared memory came out of the Bloom filter and its 46 KiB in
//    flight per SM did not cover HBM latency.)
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

// The q-gram code of the sample at byte j of the survivor's 16-byte word
// (jw = j & 15) from its 32-base code window.
__device__ __forceinline__ std::uint32_t qwin_code(unsigned long long win, std::uint32_t jw, std::uint32_t q) {
    const unsigned long long c = win >> (2 * jw);
    return static_cast<std::uint32_t>(q >= 32 ? c : c & ((1ull << (2 * q)) - 1));
}

// Pre-check in code space: pattern p (2-bit codes pc0 = bases 0..31, pc1 =
// 32..63) placed at text byte i against the survivor's 32-base window that
// starts at byte wstart (d = i - wstart in [-3, 12]); compares every base
// both cover. A mismatch rejects the occurrence without reading the text.
__device__ __forceinline__ bool qwin_match(unsigned long long win, int d, std::uint32_t len, unsigned long long pc0,
                                           unsigned long long pc1) {
    unsigned long long al;  // pattern codes aligned to window bases
    if (d >= 0) al = pc0 << (2 * d);
    else al = (pc0 >> (-2 * d)) | (pc1 << (64 + 2 * d));
    const int kmin = d > 0 ? d : 0;
    const int kmax = min(32, d + static_cast<int>(min(len, 64u)));
    if (kmax <= kmin) return true;
    const unsigned long long hi = kmax >= 32 ? ~0ull : (1ull << (2 * kmax)) - 1;
    const unsigned long long mask = hi & ~((1ull << (2 * kmin)) - 1);
    return ((win ^ al) & mask) == 0;
}

// Exact check of pattern p (bytes [lo, lo+len) of the dictionary) against
// text[i, i+len): 16 independent byte pairs per round, so a match costs
// ceil(len/16) dependent memory round trips rather than len.
__device__ __forceinline__ bool qmatch(const ScanArgs& a, long long i, std::uint32_t lo, std::uint32_t len) {
    for (std::uint32_t k0 = 0; k0 < len; k0 += 16) {
        std::uint32_t diff = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k0 + k < len) diff |= static_cast<std::uint32_t>(__ldg(a.text + i + k0 + k) ^ __ldg(a.pat_bytes + lo + k0 + k));
        if (diff) return false;
    }
    return true;
}

// Confirms survivor slot t (found in region w) exactly and appends each match
// to the slab of the region its end lies in.
__device__ __forceinline__ void qconfirm_slot(const ScanArgs& a, long long w, unsigned long long t) {
    const std::uint32_t tmask = (1u << a.qtab_bits) - 1u;
    const long long j = static_cast<long long>(__ldcg(a.qcands + t));
    const unsigned long long win = __ldcg(a.qcand_win + t);
    const std::uint32_t code = qwin_code(win, static_cast<std::uint32_t>(j & 15), a.q);
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
    if (bucket == kQEmpty) return;
    const long long wlast = static_cast<long long>(a.qwarps) - 1;
    const bool single = bucket & kQSingle;
    const std::uint32_t e0 = single ? 0u : a.qb_off[bucket], e1 = single ? 1u : a.qb_off[bucket + 1];
    for (std::uint32_t e = e0; e < e1; ++e) {
        const std::uint32_t ent = single ? bucket & ~kQSingle : a.qb_ent[e];
        const long long i = j - static_cast<long long>(ent & 3u);
        const std::uint32_t p = ent >> 2;
        const std::uint32_t lo = a.pat_off[p], len = a.pat_off[p + 1] - lo;
        if (i < 0 || i + len > a.n) continue;
        const long long end = i + len - 1;
        if (end < a.emit_from) continue;
        // pre-check in code space against the survivor's window (no text read;
        // random text passes 4^-(bases compared beyond the q-gram)), then the
        // whole pattern byte by byte
        const ulonglong2 pc = *reinterpret_cast<const ulonglong2*>(a.pat_code + 2ull * p);
        if (!qwin_match(win, static_cast<int>(i - (j & ~15LL)), len, pc.x, pc.y) || !qmatch(a, i, lo, len)) continue;
        // filed under the region holding its END (any pattern length: a long
        // occurrence found from region w's survivors may end many regions on)
        const long long d = min(end / a.qreg, wlast);
        const std::uint32_t k = atomicAdd(a.reg_n + d, 1u);
        if (k < a.mcap)
            a.qscratch[static_cast<unsigned long long>(d) * a.mcap + k] =
                ((a.base + static_cast<unsigned long long>(end)) << a.id_bits) | p;
        if (a.pcounts) atomicAdd(a.pcounts + p, 1ull);
    }
}

// KQ. No text staging in shared memory (all of it is left to the Bloom
// filter): every warp streams its own contiguous
// region of 2 KiB blocks with 128-bit streaming loads straight into
// registers, R blocks in flight per warp (R*2 KiB*NW per SM). Lane l holds
// the 16-byte words l, 32+l, 64+l, 96+l of a block (rows of 512 bytes); the
// word after lane 31's row r is lane 0's row r+1, after row 3 it is lane 0's
// row 0 of the next block (whose codes are computed one step ahead). 16
// Bloom probes per lane and block; survivors go to the warp's region through
// a shared-memory counter (no warp scan).
template <int TLD = 0>  // text load flavour (TLD > 0: experiments)
__device__ __forceinline__ uint4 ldg_stream(const std::uint8_t* p) {
    uint4 v;
    if (TLD == 1) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (TLD == 2) asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else if (TLD == 3) asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// programmatic dependent launch (sm_90+): wait for / release the stream's neighbouring grids
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ const std::uint32_t* tab_of() { return reinterpret_cast<const std::uint32_t*>(acg_hot_smem); }

// Load flavours, LDV = 8 * (text load) + (level-2 probe load). Defaults: 24 for the
// single-level kernel (text L1::no_allocate), 25 with the level-2 filter (probes as
// ld.global.cg: a probe must not allocate a line in the 23 KB of L1 left beside the
// filter — with ld.global.nc every probe and every text line queued behind that
// allocation: cfg2 0.956 -> 0.814 ms per 2 GiB). The other values are the measured
// alternatives ("Measured and rejected").
template <int LDV>
__device__ __forceinline__ std::uint32_t q2_load(const std::uint32_t* p) {
    std::uint32_t v;
    if (LDV == 1) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if (LDV == 2) asm volatile("ld.global.cv.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if (LDV == 3) asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if (LDV == 4) asm volatile("atom.global.or.b32 %0, [%1], 0;" : "=r"(v) : "l"(p) : "memory");
    else v = __ldg(p);
    return v;
}

template <int NW, int R, bool L2F, bool FUSED, bool BM, bool POST, int LDV = 0>
__device__ __forceinline__ void qfilter_produce(const ScanArgs& a, const std::uint32_t* tab, std::uint32_t* wcnt,
                                                std::uint32_t* pub, std::uint32_t* nfin) {
    constexpr long long kBlk = 2048;
    const long long n = a.n;
    const long long nb = (n + kBlk - 1) / kBlk;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long gw = static_cast<long long>(blockIdx.x) * NW + warp;
    const long long tw = static_cast<long long>(gridDim.x) * NW;
    const long long per = (nb + tw - 1) / tw;
    const long long b0 = gw * per, b1 = min(b0 + per, nb);
    const std::uint32_t qsh = a.qsh, words = a.qwords;
    const unsigned long long region = static_cast<unsigned long long>(gw) * a.qcand_cap;

    uint4 buf[R][4];
    // blocks are loaded in order b0, b0+1, ...: a running pointer, and bounds
    // checks only for the text's last (partial) block
    const long long nfull = n / kBlk;
    const std::uint8_t* lp = a.text + b0 * kBlk + 16 * lane;
    long long lb = b0;
    auto load = [&](uint4 (&dst)[4]) {
        if (lb < nfull) {
#pragma unroll
            for (int r = 0; r < 4; ++r) dst[r] = ldg_stream<LDV / 8>(lp + 512 * r);
        } else {
            const long long off = lb * kBlk + 16 * lane;
#pragma unroll
            for (int r = 0; r < 4; ++r)
                dst[r] = (lb < nb && off + 512 * r < n) ? ldg_stream<LDV / 8>(lp + 512 * r) : make_uint4(0, 0, 0, 0);
        }
        lp += kBlk;
        ++lb;
    };
    const std::uint32_t qmul = qsh * kQMul0;  // window -> hash in one multiply (qfilter.hpp)
    const std::uint32_t qmul2 = qmul * kQMul3;  // window -> level-2 word hash qhash2(h)
#if !defined(ACG_KQ_NOPIN)
    // qmask's PRMT takes its first byte table from a register: as a literal the compiler
    // re-materialises it before nearly every probe (14 moves per block); a value it
    // cannot know at compile time (n >= 0, so the XOR is with 0) stays in one register
    const std::uint32_t bits_lo = 0x08040201u ^ static_cast<std::uint32_t>(static_cast<unsigned long long>(n) >> 63);
    auto probe = [&](std::uint32_t h) -> std::uint32_t {
        return __byte_perm(bits_lo, 0x80402010u, __umulhi(h, kQMul1) & 0x7777u) & ~tab[qword(h, words)];
    };
    auto mask_of = [&](std::uint32_t h) -> std::uint32_t {
        return __byte_perm(bits_lo, 0x80402010u, __umulhi(h, kQMul1) & 0x7777u);
    };
#else
    auto probe = [&](std::uint32_t h) -> std::uint32_t { return qmask(h) & ~tab[qword(h, words)]; };
    auto mask_of = [&](std::uint32_t h) -> std::uint32_t { return qmask(h); };
#endif
    auto window = [&](std::uint32_t lo, std::uint32_t hi, int o) -> std::uint32_t {
        return o == 0 ? lo : __funnelshift_r(lo, hi, 8 * o);
    };
    auto gram = [&](std::uint32_t lo, std::uint32_t hi, int o) -> std::uint32_t { return window(lo, hi, o) * qsh; };

    if (b0 < b1) {
#pragma unroll
        for (int k = 0; k < R; ++k) load(buf[k]);
        std::uint32_t cur[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) cur[r] = qcodes(buf[0][r]);
        load(buf[0]);
        for (long long bb = b0; bb < b1; bb += R) {
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const long long b = bb + k;
                if (b >= b1) break;
                const int sl = (k + 1) % R;  // slot holding block b+1
                std::uint32_t nxt[4];
                // lane 0 needs the next block's first word now (lane 31's last neighbour);
                // the rest of the next block is packed later (L2F: while level-2 probes fly)
                nxt[0] = qcodes(buf[sl][0]);
                if (!L2F) {
#pragma unroll
                    for (int r = 1; r < 4; ++r) nxt[r] = qcodes(buf[sl][r]);
                    load(buf[sl]);  // block b + 1 + R
                }
                // neighbour codes: lane+1's word of the same row; lane 31 gets lane 0's next row
                std::uint32_t nb_[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const std::uint32_t s = lane == 0 ? (r < 3 ? cur[r + 1] : nxt[0]) : cur[r];
                    nb_[r] = __shfl_sync(0xFFFFFFFFu, s, (lane + 1) & 31);
                }
                std::uint32_t t[16];
                std::uint32_t m1[L2F ? 16 : 1];  // L2F: level 1's masks, tested again at level 2
                std::uint32_t bm_hits = 0;  // BM: samples that pass both levels (bit 4r+o)
                if (BM) {
                    // level 1: bit (c & 0xFFFFF) of a 2^20-bit bitmap of the keys' 10-gram
                    // prefixes; the word's bit is rotated to position k and merged into
                    // the mask (SHF, LOP3, LDS, SHF.W, LOP3 per sample, no hashing)
                    std::uint32_t hm = 0;
#pragma unroll
                    for (int r = 0; r < 4; ++r)
#pragma unroll
                        for (int o = 0; o < 4; ++o) {
                            const std::uint32_t win = window(cur[r], nb_[r], o);
                            const std::uint32_t wd = tab[(win >> 5) & (kQBitmapWords - 1)];
                            hm |= __funnelshift_r(wd, wd, win - (4 * r + o)) & (1u << (4 * r + o));
                        }
                    // level 2, the lane's level-1 hits only: the blocked Bloom filter of
                    // the full q-grams after the bitmap
                    const std::uint32_t* bl = tab + kQBitmapWords;
                    const std::uint32_t w2 = words - kQBitmapWords;
                    for (std::uint32_t mm = hm; mm; mm &= mm - 1) {
                        const int k = __ffs(mm) - 1, r = k >> 2, o = k & 3;
                        const std::uint32_t lo = r == 0 ? cur[0] : r == 1 ? cur[1] : r == 2 ? cur[2] : cur[3];
                        const std::uint32_t hi = r == 0 ? nb_[0] : r == 1 ? nb_[1] : r == 2 ? nb_[2] : nb_[3];
                        const std::uint32_t h = (o == 0 ? lo : __funnelshift_r(lo, hi, 8 * o)) * qmul;
                        const std::uint32_t m = qmask(h);
                        if ((bl[qword(h, w2)] & m) == m) bm_hits |= 1u << k;
                    }
                } else {
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int o = 0; o < 4; ++o) {
                        if (L2F) {
                            const std::uint32_t h = window(cur[r], nb_[r], o) * qmul;
                            m1[4 * r + o] = mask_of(h);
                            t[4 * r + o] = m1[4 * r + o] & ~tab[qword(h, words)];
                        } else {
                            t[4 * r + o] = probe(window(cur[r], nb_[r], o) * qmul);
                        }
                    }
                }
                if (L2F) {
                    // level 2 for the samples level 1 passed: predicated L2-resident
                    // probes, issued together (one L2 latency per block)
                    std::uint32_t v2[16];
#pragma unroll
                    for (int r = 0; r < 4; ++r)
#pragma unroll
                        for (int o = 0; o < 4; ++o) {
                            const int i = 4 * r + o;
                            // word from h2 = window * (qmul * kQMul3) (= qhash2(h)), the mask is level 1's
                            const std::uint32_t h2 = window(cur[r], nb_[r], o) * qmul2;
                            v2[i] = t[i] == 0u ? q2_load<LDV % 8>(a.qbloom2 + qword(h2, a.qwords2)) : 0u;
                        }
                    // pack the next block and issue its load while the probes are in flight
#pragma unroll
                    for (int r = 1; r < 4; ++r) nxt[r] = qcodes(buf[sl][r]);
                    load(buf[sl]);  // block b + 1 + R
#pragma unroll
                    for (int i = 0; i < 16; ++i) t[i] = m1[i] & ~v2[i];
                }
                bool hit;
                if (BM) {
                    hit = bm_hits != 0u;
                } else {
                    std::uint32_t z = min(min(t[0], t[1]), t[2]);
                    z = min(min(z, t[3]), t[4]);
                    z = min(min(z, t[5]), t[6]);
                    z = min(min(z, t[7]), t[8]);
                    z = min(min(z, t[9]), t[10]);
                    z = min(min(z, t[11]), t[12]);
                    z = min(min(z, t[13]), t[14]);
                    z = min(z, t[15]);
                    hit = z == 0u;
                }
                const bool anyhit = __any_sync(0xFFFFFFFFu, hit);
                if (anyhit && hit) {
                    std::uint32_t pm = 0;
                    if (BM) {
                        pm = bm_hits;
                    } else {
#pragma unroll
                        for (int o = 0; o < 16; ++o) pm |= (t[o] == 0u ? 1u : 0u) << o;
                    }
                    const long long P = b * kBlk + 16 * lane;
                    if (b >= nfull) {  // the text's partial last block: samples past its end are not survivors
#pragma unroll
                        for (int o = 0; o < 16; ++o)
                            if (P + 512 * (o >> 2) + 4 * (o & 3) >= n) pm &= ~(1u << o);
                    }
                    std::uint32_t slot = atomicAdd(&wcnt[warp], static_cast<std::uint32_t>(__popc(pm)));
                    for (std::uint32_t m = pm; m; m &= m - 1, ++slot) {
                        const int i = __ffs(m) - 1, r = i >> 2, o = i & 3;
                        const long long pos = P + 512 * r + 4 * o;
                        if (slot < a.qcand_cap) {
                            std::uint32_t lo = cur[0], hi = nb_[0];
                            if (r == 1) lo = cur[1], hi = nb_[1];
                            if (r == 2) lo = cur[2], hi = nb_[2];
                            if (r == 3) lo = cur[3], hi = nb_[3];
                            a.qcands[region + slot] = static_cast<unsigned long long>(pos);
                            a.qcand_win[region + slot] = (static_cast<unsigned long long>(hi) << 32) | lo;
                        }
                    }
                }
                if (FUSED && anyhit) {  // publish this warp's survivors to the consumer warp
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence_block();
                        *static_cast<volatile std::uint32_t*>(&pub[warp]) = *static_cast<volatile std::uint32_t*>(&wcnt[warp]);
                    }
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) cur[r] = nxt[r];
            }
        }
    }
    __syncwarp();
    if (lane == 0) {
        const std::uint32_t found = *static_cast<volatile std::uint32_t*>(&wcnt[warp]);
        a.qwarp_n[gw] = found;
        // V1's per-region counters (one per chunk; zeroed by the host when V1 runs inside KQ)
        if (!FUSED && !POST && a.reg_n && gw < a.n_chunks) a.reg_n[gw] = 0u;
        atomicAdd(a.qcand_n, found);
        atomicMax(a.qcand_max, static_cast<unsigned long long>(found));
        if (FUSED) {
            __threadfence_block();
            *static_cast<volatile std::uint32_t*>(&pub[warp]) = found;
            __threadfence_block();
            atomicAdd(nfin, 1u);
        }
    }
}

// The consumer warp of the fused KQ: confirms the producers' published
// survivors while they stream (V1's work overlapped with the scan), until all
// producers have finished; what is left is drained by the whole CTA.
template <int NW>
__device__ __forceinline__ void qfilter_consume(const ScanArgs& a, const std::uint32_t* pub, std::uint32_t* done_sh,
                                                std::uint32_t* nfin) {
    const int lane = threadIdx.x & 31;
    std::uint32_t done[NW];
#pragma unroll
    for (int p = 0; p < NW; ++p) done[p] = 0;
    for (;;) {
        const bool fin = *static_cast<volatile std::uint32_t*>(nfin) == NW;
        if (fin) break;  // the rest goes to the cooperative drain
        bool any = false;
#pragma unroll
        for (int p = 0; p < NW; ++p) {
            const std::uint32_t avail = min(*static_cast<const volatile std::uint32_t*>(&pub[p]), a.qcand_cap);
            if (done[p] < avail) {
                __threadfence_block();
                const long long w = static_cast<long long>(blockIdx.x) * NW + p;
                const std::uint32_t k = done[p] + lane;
                if (k < avail) qconfirm_slot(a, w, static_cast<unsigned long long>(w) * a.qcand_cap + k);
                done[p] = min(avail, done[p] + 32u);
                any = true;
            }
        }
        if (!any) __nanosleep(256);
    }
    if (lane == 0)
#pragma unroll
        for (int p = 0; p < NW; ++p) done_sh[p] = done[p];
}

// After every producer finished: the whole CTA confirms the survivors the
// consumer warp had not reached.
template <int NW>
__device__ __forceinline__ void qfilter_drain(const ScanArgs& a, const std::uint32_t* pub, const std::uint32_t* done_sh) {
    std::uint32_t total = 0;
#pragma unroll
    for (int p = 0; p < NW; ++p) total += min(pub[p], a.qcand_cap) - done_sh[p];
    for (std::uint32_t f = threadIdx.x; f < total; f += blockDim.x) {
        std::uint32_t g = f;
        int p = 0;
        for (; p < NW; ++p) {
            const std::uint32_t len = min(pub[p], a.qcand_cap) - done_sh[p];
            if (g < len) break;
            g -= len;
        }
        const long long w = static_cast<long long>(blockIdx.x) * NW + p;
        qconfirm_slot(a, w, static_cast<unsigned long long>(w) * a.qcand_cap + done_sh[p] + g);
    }
}

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


// POST: the CTA confirms its own warps' survivors right after streaming (V1
// inside KQ, overlapping the other CTAs' streaming tails; no V1 launch).
template <int NW, int R, bool L2F, bool FUSED, bool BM = false, bool POST = false, int LDV = 0>
__global__ void __launch_bounds__(32 * (NW + (FUSED ? 1 : 0)), 1) qfilter_ldg_kernel(const ScanArgs a) {
    __shared__ std::uint32_t wcnt[NW], pub[NW], done_sh[NW], nfin;
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.qbloom);
        uint4* dst = reinterpret_cast<uint4*>(acg_hot_smem);
        for (std::uint32_t i = threadIdx.x; i < a.qwords / 4; i += blockDim.x) dst[i] = __ldg(src + i);
        if (threadIdx.x < NW) wcnt[threadIdx.x] = pub[threadIdx.x] = 0;
        if (threadIdx.x == 0) nfin = 0;
    }
    pdl_wait();  // (launched programmatically: the filter is staged; the workspace is ours from here)
    __syncthreads();
    if (FUSED && (threadIdx.x >> 5) == NW) {  // the consumer warp
        qfilter_consume<NW>(a, pub, done_sh, &nfin);
    } else {
        qfilter_produce<NW, R, L2F, FUSED, BM, POST, LDV>(a, tab_of(), wcnt, pub, &nfin);
    }
    if (!POST && !FUSED) pdl_trigger();  // V1 may be scheduled (it waits for this grid's results)
    if (POST) {
        __syncthreads();  // this CTA's survivors and their counts are written
        const unsigned long long cap = a.qcand_cap;
        const unsigned long long t0 = static_cast<unsigned long long>(blockIdx.x) * NW * cap;
        for (unsigned long long t = t0 + threadIdx.x; t < t0 + NW * cap; t += blockDim.x) {
            const long long w = static_cast<long long>(t / cap);
            if (t - static_cast<unsigned long long>(w) * cap < min(wcnt[w - static_cast<long long>(blockIdx.x) * NW],
                                                                   a.qcand_cap))
                qconfirm_slot(a, w, t);
        }
    }
    if (FUSED) {
        __syncthreads();
        qfilter_drain<NW>(a, pub, done_sh);
    }
}

// V1: confirms every survivor exactly (the q-gram's (pattern, offset)
// bucket, then a byte compare at i = j - offset); threads stride over the
// survivor regions' slots. Each match is appended to the slab of the region
// holding its end (reg_n[d], zeroed by KQ, counts them even past the
// capacity), so every slab holds exactly its region's matches whatever the
// pattern length.
__global__ void __launch_bounds__(256) qconfirm_region_kernel(const ScanArgs a) {
    pdl_wait();  // (launched programmatically after KQ: its survivors are complete past this point)
    const long long total = static_cast<long long>(a.qwarps) * a.qcand_cap;
    pdl_trigger();  // ORDER may be scheduled (it waits for this grid's results)
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long w = t / a.qcand_cap;
        if (static_cast<std::uint32_t>(t - w * a.qcand_cap) >= a.qwarp_n[w]) continue;
        qconfirm_slot(a, w, static_cast<unsigned long long>(t));
    }
}

// V1, one CTA per survivor region (the default): the region's survivors on
// consecutive threads — no slot -> region division, no lanes parked on empty
// slots (the strided form above ran 11.9 active threads per warp, and its
// instruction stream, not the lookups' latency, was V1's time).
__global__ void __launch_bounds__(256) qconfirm_cta_kernel(const ScanArgs a) {
    pdl_wait();  // (launched programmatically after KQ: its survivors are complete past this point)
    pdl_trigger();  // ORDER may be scheduled (it waits for this grid's results)
    for (long long w = blockIdx.x; w < static_cast<long long>(a.qwarps); w += gridDim.x) {
        const std::uint32_t nw = min(a.qwarp_n[w], a.qcand_cap);
        const unsigned long long t0 = static_cast<unsigned long long>(w) * a.qcand_cap;
        for (std::uint32_t k = threadIdx.x; k < nw; k += blockDim.x) qconfirm_slot(a, w, t0 + k);
    }
}

// ORDER: one warp per region. Its slot range starts at the sum of the
// matches owned by earlier regions (summed directly from reg_n: no separate
// scan pass); it reads its slab (every match ending in the region) and sorts
// it: one bitonic round in registers for <= 32, a warp bitonic sort in shared
// memory for <= kQOrderMax; a bigger region sets qscal[1] and the host replays
// the run through the per-chunk pipeline (V0/K2/K3).
constexpr int kQOrderMax = 1024;
constexpr int kQOrderWarps = 4;

__global__ void __launch_bounds__(32 * kQOrderWarps) qorder_region_kernel(const ScanArgs a, unsigned long long* offs) {
    pdl_wait();  // (after V1: its slabs and region counts are complete past this point)
    static_assert(kQOrderWarps == 4, "the CTA prefix below reads whole uint4 groups of regions");
    __shared__ unsigned long long buf[kQOrderWarps][kQOrderMax];
    __shared__ unsigned long long part[kQOrderWarps];
    const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long w0 = static_cast<long long>(blockIdx.x) * kQOrderWarps;
    const long long w = w0 + wl;
    const long long W = a.qwarps;
    {  // the CTA's prefix: sum of reg_n[0, w0) by all its threads (16-byte loads)
        const uint4* r4 = reinterpret_cast<const uint4*>(a.reg_n);
        unsigned long long ps = 0;
#pragma unroll 4
        for (long long v = threadIdx.x; v < (w0 >> 2); v += blockDim.x) {
            const uint4 q = r4[v];
            ps += static_cast<unsigned long long>(q.x) + q.y + q.z + q.w;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) ps += __shfl_xor_sync(0xFFFFFFFFu, ps, o);
        if (lane == 0) part[wl] = ps;
    }
    __syncthreads();
    if (w >= W) return;
    unsigned long long off = part[0] + part[1] + part[2] + part[3];
    for (long long v = w0; v < w; ++v) off += a.reg_n[v];  // this CTA's earlier regions (< 4)
    const std::uint32_t own = a.reg_n[w];
    if (lane == 0) {
        if (a.reg_n[w] > a.mcap) atomicMax(a.qscal, a.reg_n[w]);  // slab overflow: the host re-runs
        offs[w] = off;
        if (w == W - 1) offs[W] = off + own;
    }
    if (own == 0) return;
    if (own > static_cast<std::uint32_t>(kQOrderMax)) {
        if (lane == 0) atomicMax(a.qscal + 1, own);
        return;
    }
    if (own > a.mcap) return;  // slab overflowed: the host re-runs with larger slabs
    const unsigned long long* sw = a.qscratch + static_cast<unsigned long long>(w) * a.mcap;
    unsigned long long* b = buf[wl];
    const std::uint32_t k = own;
    if (k <= 32) {
        unsigned long long v = lane < static_cast<int>(k) ? sw[lane] : ~0ull;
        v = bitonic32(v, lane);
        if (lane < static_cast<int>(k) && off + lane < a.rec_cap) a.records[off + lane] = v;
        return;
    }
    for (std::uint32_t t = lane; t < k; t += 32) b[t] = sw[t];
    __syncwarp();
    std::uint32_t p2 = 64;
    while (p2 < k) p2 <<= 1;
    for (std::uint32_t t = k + lane; t < p2; t += 32) b[t] = ~0ull;
    __syncwarp();
    for (std::uint32_t size = 2; size <= p2; size <<= 1) {
        for (std::uint32_t stride = size >> 1; stride; stride >>= 1) {
            for (std::uint32_t t = lane; t < p2 / 2; t += 32) {
                const std::uint32_t i = 2 * t - (t & (stride - 1));  // lower index of the pair
                const std::uint32_t jj = i + stride;
                const bool up = (i & size) == 0;
                const unsigned long long x = b[i], y = b[jj];
                if ((x > y) == up) {
                    b[i] = y;
                    b[jj] = x;
                }
            }
            __syncwarp();
        }
    }
    for (std::uint32_t t = lane; t < k; t += 32)
        if (off + t < a.rec_cap) a.records[off + t] = b[t];
}

// V0: exact confirmation of the survivors (see the header comment).
template <int PASS>
__global__ void __launch_bounds__(256) qconfirm_kernel(const ScanArgs a) {
    const std::uint32_t tmask = (1u << a.qtab_bits) - 1u;
    const long long total = static_cast<long long>(a.qwarps) * a.qcand_cap;
    pdl_trigger();  // ORDER may be scheduled (it waits for this grid's results)
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        if (static_cast<std::uint32_t>(t % a.qcand_cap) >= a.qwarp_n[t / a.qcand_cap]) continue;
        const long long j = static_cast<long long>(a.qcands[t]);
        // the survivor's q-gram code, from KQ (y holds it in the top bits)
        const unsigned long long win = a.qcand_win[t];
        const std::uint32_t code = qwin_code(win, static_cast<std::uint32_t>(j & 15), a.q);
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
        const bool single = bucket & kQSingle;
        const std::uint32_t e0 = single ? 0u : a.qb_off[bucket], e1 = single ? 1u : a.qb_off[bucket + 1];
        for (std::uint32_t e = e0; e < e1; ++e) {
            const std::uint32_t ent = single ? bucket & ~kQSingle : a.qb_ent[e];
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
