// sm_100a Aho-Corasick DFA scan kernels.
//
// Replaces the reference's hot loop, acmatch::scan
// (proj/include/acmatch/aho_corasick.hpp:250-272), with chunked dense-DFA walks.
//
// Chunking. The owned text [emit_from, n) is cut into chunks of `chunk` bytes;
// the stream for chunk c starts `halo` (= round_up(maxlen,16)) bytes early from
// the root, so its state is exact from the first owned byte on (the DFA state
// at i depends only on text[i-maxlen+1 .. i]). Every thread
// walks U chunks in lockstep (U independent dependent-load chains).
//
// Device numbering. [0,Hn) hot non-output, [Hn,H) hot output, [H,Cn) cold
// output, [Cn,S) cold non-output; rows [0,H) are "hot" (shared memory); the
// output states [Hn,Cn) are contiguous, output rank = s - Hn.
//
// Count-pass kernels:
//
//  * sparse_scan_kernel (K1s) walks the TRUNCATED automaton A_H whose states
//    are the hot set H. H is a BFS prefix of the trie (all nodes of depth < D
//    plus some of depth D), hence closed under "longest suffix in H", and
//    A_H(s,c) = longest suffix of s.c in H is a self-contained DFA whose state
//    is always the longest hot suffix of the text — equal to the true state
//    whenever the true state is hot. Its table (u16, bit 15 = attention) lives
//    entirely in shared memory: no global lookups, no branches. A transition
//    is flagged when the TRUE next state is cold or has outputs; the stream
//    then logs an event (offset, exact previous state, packed symbols).
//    Events inside a cold excursion come from proxy states and are skipped.
//  * fixup_kernel (K1f) replays each chunk's events in order with the full
//    u32 DFA (L2-resident), walking every cold excursion until the true state
//    is hot again, and counts / writes the outputs. Used for both the count
//    pass and the ordered write pass of the sparse mode.
//  * exact_scan_kernel (K1x) walks the true DFA in lockstep: hot rows from
//    shared memory, cold rows with predicated L2 loads; used when excursions
//    are frequent (large or dense automata), for exact ScanStats, and for the
//    ordered write pass of that mode.
//
// Outputs. COUNT writes per-chunk record counts (u64) and per-output-state
// visit counts; an exclusive scan gives every chunk its canonical
// (end, id)-ordered slot range; WRITE stores packed records
// (end << id_bits | id), ascending.
#pragma once

#include <cstdint>

// Dynamic shared memory, named at global scope so inline PTX can address it
// as a symbol (ptxas folds the base into the LDS immediate/uniform operand).
extern __shared__ __align__(16) std::uint8_t acg_hot_smem[];

namespace acg {
namespace kern {

// kScratch: one exact walk that counts AND stores each chunk's records into
// its own scratch slab (scap per chunk; a fuller chunk keeps counting and is
// re-walked by a WRITE pass over the overflow list).
enum Pass : int { kCount = 0, kWrite = 1, kScratch = 2 };
#ifndef ACG_EXACT_UNROLL
#define ACG_EXACT_UNROLL 16  // steps of the exact walk's fast path unrolled (code size vs ILP)
#endif
#define ACG_PRAGMA(x) _Pragma(#x)
#define ACG_UNROLL(n) ACG_PRAGMA(unroll n)
constexpr int kTPB = 512;  // threads per block of the scan kernels
constexpr std::uint32_t kEsc16 = 0xFFFFu;

struct ScanArgs {
    const std::uint8_t* text;  // 16-byte aligned; byte i of this buffer = global byte base+i
    long long n;               // bytes in the buffer
    long long emit_from;       // first owned byte (multiple of 16)
    unsigned long long base;   // global offset of text[0] (added to record ends)
    long long chunk;           // owned bytes per chunk (multiple of 16)
    long long halo;            // warm-up bytes (multiple of 16)
    long long n_chunks;
    // DFA
    const std::uint32_t* next;     // S*K exact transitions (device ids)
    const std::uint16_t* hot16;    // (H+1)*K exact hot rows; 0xFFFF = consult `next`; row H = all 0xFFFF
    const std::uint16_t* hotH;     // H*K truncated-automaton rows: id | 0x8000 attention
    const std::uint32_t* out_off;  // S+1
    const std::uint32_t* out_ids;
    const unsigned long long* outinfo;  // S: out_off | count << 32 | first id << 40 (automaton.hpp)
    const std::uint32_t* depth;    // S: trie depth per device state (sparse-mode dedup)
    const std::uint16_t* follows;      // S*K (stats only)
    const std::uint16_t* follows_esc;  // S (stats only, dna4 mode)
    const std::uint8_t* symmap;        // 256 (generic mode)
    std::uint32_t K, H, Hn, Cn;
    std::uint32_t smem_table_bytes;    // bytes of the staged table (multiple of 16)
    // outputs
    unsigned long long* chunk_counts;       // COUNT: written (u64 so K2 scans it directly)
    const std::uint32_t* active_list;       // WRITE: chunk ids with matches (compacted)
    const std::uint32_t* active_count;      // WRITE: number of entries in active_list
    const unsigned long long* chunk_offs;   // WRITE: exclusive prefix of chunk_counts
    unsigned long long* visits;             // COUNT (optional): per output state (rank order)
    unsigned long long* records;            // WRITE
    unsigned long long rec_cap;
    std::uint32_t id_bits;
    unsigned long long* follows_total;      // COUNT with stats (optional)
    // sparse-mode event log: per K1s warp `ev_cap` 16-byte events (see K1s)
    std::uint32_t* events;
    std::uint32_t* ev_count;                // per K1s warp (may exceed ev_cap: overflow)
    std::uint32_t ev_cap;
    std::uint32_t* cands;                   // per chunk kExport exported candidates (uint4)
    std::uint32_t* cand_list;               // per K1s warp buffer: kCandList (key, state) pairs
    std::uint32_t* cand_cnt;                // per K1s warp buffer: candidates appended (zeroed per run)
    std::uint32_t* tasks;                   // excursion tasks (uint4): one region of task_cap per fix-up warp
    std::uint32_t* task_cnt;                // per region: tasks appended
    std::uint32_t* task_max;                // max over regions (overflow check at sync)
    std::uint32_t task_cap;
    std::uint32_t* cand_n;                  // per chunk: exported count, 0xFFFFFFFF = re-walk
    unsigned long long* ev_total;           // sum of events (mode heuristic)
    // filter mode (filter_kernels.cuh)
    const std::uint32_t* qbloom;            // kQWords blocked-Bloom words
    const std::uint32_t* qtab;              // exact q-gram table: 2^qtab_bits (code, bucket) slots
    std::uint32_t qtab_bits;
    const std::uint32_t* qb_off;            // bucket offsets
    const std::uint32_t* qb_ent;            // pattern id << 2 | offset
    const std::uint8_t* pat_bytes;          // the dictionary
    const std::uint32_t* pat_off;           // n_patterns + 1
    std::uint32_t qwords;                   // words of the staged level-1 image (Bloom, or bitmap + Bloom)
    std::uint32_t qbm;                      // 1: level 1 = 10-gram bitmap, then the Bloom filter (qfilter.hpp)
    const std::uint32_t* qbloom2;           // level-2 Bloom filter (L2-resident; null = single level)
    std::uint32_t qwords2;
    unsigned long long* qcands;             // KQ survivors (sample offsets): one region of qcand_cap per KQ warp
    unsigned long long* qcand_win;          // their text codes: 32 bases from the survivor's 16-byte word (2 bits each)
    const unsigned long long* pat_code;     // per pattern: 2-bit codes of its first 64 bytes (2 words)
    std::uint32_t* qwarp_n;                 // per KQ consumer warp: survivors found (may exceed qcand_cap)
    std::uint32_t qwarps;                   // KQ consumer warps (regions)
    std::uint32_t* qcand_n;                 // total survivors (rate heuristic)
    unsigned long long* qcand_max;          // max over regions (overflow check at sync)
    std::uint32_t qcand_cap;                // per-region capacity
    unsigned long long* pcounts;            // per-pattern counts (filter mode counts them directly)
    unsigned long long* qscratch;           // V0 count pass: packed records, unordered (rec_cap entries)
    unsigned long long* qscratch_n;
    std::uint32_t* qfill;                   // per chunk: records placed so far
    std::uint32_t q;                        // q-gram length
    std::uint32_t qsh;                      // 2^(32 - 2q): window * qsh puts the q-gram code in the top bits
    std::uint32_t max_len;                  // longest pattern
    // filter mode, region pipeline (V1 + ORDER): KQ warp w's region of the
    // buffer [w*qreg, (w+1)*qreg) owns the matches that END in it
    long long qreg;                         // region bytes (multiple of 2048)
    std::uint32_t* reg_n;                   // per region: confirmed matches that end in it
    std::uint32_t mcap;                     // per-region slab capacity (qscratch)
    std::uint32_t* qscal;                   // [0] max reg_n (overflow), [1] regions too big for ORDER
    // exact mode, single pass (kScratch): chunk c's slab is scratch[c*scap, (c+1)*scap),
    // or [slab_off[c], slab_off[c+1]) when sized from the previous run's chunk counts
    unsigned long long* scratch;
    unsigned long long scap;
    const unsigned long long* slab_off;
    unsigned long long* chunk_max;          // COUNT / kScratch: max over chunks of the record count
};

__device__ __forceinline__ uint4 ld_stream16(const std::uint8_t* p) {
    uint4 v;
// Each stream reads 16 bytes of its own chunk per 16 steps, so a warp's load
// touches 32 different sectors: the L2 prefetch hint makes the first load of
// a stream fetch the next 256 (or 128) bytes of it, which its next loads then
// hit (ncu, cfg3: evict-first streaming loads without the hint read the text
// 6.7x from DRAM).
#if defined(ACG_EXACT_TEXT_CS)  // experiment
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
#elif defined(ACG_EXACT_TEXT_128)
    asm volatile("ld.global.nc.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];"
#else
    asm volatile("ld.global.nc.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
#endif
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ std::uint32_t lds_u16(std::uint32_t saddr) {
    std::uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(saddr));
    return v;
}

// u16 from shared memory, zero-extended into a 32-bit register
__device__ __forceinline__ std::uint32_t lds_u16z(std::uint32_t saddr) {
    std::uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(saddr));
    return v;
}

__device__ __forceinline__ std::uint32_t lds_u32(std::uint32_t saddr) {
    std::uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
    return v;
}
__device__ __forceinline__ std::uint32_t lds_u8z(std::uint32_t saddr) {
    std::uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(saddr));
    return v;
}

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// DNA4: byte -> column (byte>>1)&3 (A0 C1 T2 G3). Packs 16 bytes into 16
// 2-bit columns (symbol k at bits 2k..2k+1); `bad` != 0 if any byte is not ACGT.
__device__ __forceinline__ std::uint32_t dna4_word(std::uint32_t w, std::uint32_t& bad) {
    const std::uint32_t s4 = (w >> 1) & 0x03030303u;
    const std::uint32_t t = (s4 | (s4 >> 4)) & 0x00FF00FFu;
    const std::uint32_t sel = t | (t >> 8);
    bad |= __byte_perm(0x47544341u, 0u, sel) ^ w;  // reconstruct 'A','C','T','G'
    return s4 * 0x01041040u;                        // packed byte in bits 24..31
}

__device__ __forceinline__ std::uint32_t dna4_pack(const uint4& w, std::uint32_t& bad) {
    const std::uint32_t m0 = dna4_word(w.x, bad), m1 = dna4_word(w.y, bad);
    const std::uint32_t m2 = dna4_word(w.z, bad), m3 = dna4_word(w.w, bad);
    const std::uint32_t lo = __byte_perm(m0, m1, 0x0073u);
    const std::uint32_t hi = __byte_perm(m2, m3, 0x7300u);
    return __byte_perm(lo, hi, 0x7610u);
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ std::uint32_t out_rank(std::uint32_t s, const ScanArgs& a) {
    return s - a.Hn;
}

__device__ __forceinline__ bool has_out(std::uint32_t s, const ScanArgs& a) {
    return s - a.Hn < a.Cn - a.Hn;
}

// Column of byte b (-1 = escape: every state goes to the root).
template <int MODE>
__device__ __forceinline__ int column_of(std::uint32_t b, const std::uint8_t* smap, const ScanArgs& a) {
    if (MODE == 0) return (b == 'A' || b == 'C' || b == 'G' || b == 'T') ? static_cast<int>((b >> 1) & 3u) : -1;
    const std::uint32_t c = smap ? smap[b] : a.symmap[b];
    return c == a.K - 1 ? -1 : static_cast<int>(c);
}

// Output handling at owned buffer position `pos` for state s (has outputs).
#ifdef ACG_EMIT_NOINLINE  // experiment: one out-of-line copy instead of one per unrolled step
#define ACG_EMIT_INLINE __noinline__
#else
#define ACG_EMIT_INLINE __forceinline__
#endif
template <int PASS>
__device__ ACG_EMIT_INLINE void emit(std::uint32_t s, long long pos, unsigned long long& cnt, unsigned long long& wr,
                                     const ScanArgs& a, unsigned long long slab_end = 0) {
    // one load: the state's output count, first id and list offset
    const unsigned long long info = __ldg(a.outinfo + s);
    std::uint32_t n = static_cast<std::uint32_t>(info >> 32) & 0xFFu;
    const std::uint32_t lo = static_cast<std::uint32_t>(info);
    if (n == 255u) n = __ldg(a.out_off + s + 1) - lo;
    // per-state visits are recorded by whichever pass the host enables them for
    if (a.visits) atomicAdd(a.visits + out_rank(s, a), 1ull);
    if (PASS == kCount) {
        cnt += n;
    } else {
        // kWrite: wr = global record slot; kScratch: wr = slot in scratch, below the chunk's slab end
        const unsigned long long endk = (a.base + static_cast<unsigned long long>(pos)) << a.id_bits;
        const unsigned long long lim = PASS == kWrite ? a.rec_cap : slab_end;
        unsigned long long* dst = PASS == kWrite ? a.records : a.scratch;
        const std::uint32_t first = static_cast<std::uint32_t>(info >> 40);
        for (std::uint32_t j = 0; j < n; ++j) {
            const std::uint32_t id = (j == 0 && (first || a.id_bits <= 24)) ? first : __ldg(a.out_ids + lo + j);
            if (wr < lim) dst[wr] = endk | id;
            ++wr;
            if (PASS == kScratch) ++cnt;
        }
    }
}

// ===================================================================== K1x ==
// Exact lockstep walk. One step of U streams: U shared loads issued together
// (cold source rows clamp to the all-escape row H), then U L2 loads for the
// escapes, so a warp waits for at most one L2 latency per step.
template <int U, int MODE, int PASS, bool STATS>
__global__ void __launch_bounds__(U <= 2 ? 2 * kTPB : kTPB, 1) exact_scan_kernel(const ScanArgs a) {
    extern __shared__ __align__(16) std::uint8_t smem[];
    const std::uint32_t hot_s = smem_u32(smem);
    const std::uint8_t* smap = smem + a.smem_table_bytes;

    const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long n_work = PASS == kWrite ? static_cast<long long>(*a.active_count) : a.n_chunks;
    if (static_cast<long long>(blockIdx.x) * blockDim.x * U >= n_work) return;  // whole block idle

    long long chunk_id[U];
    bool act[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const long long i = tid * U + u;
        act[u] = i < n_work;
        chunk_id[u] = act[u] ? (PASS == kWrite ? static_cast<long long>(a.active_list[i]) : i) : 0;
    }
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.hot16);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (std::uint32_t i = threadIdx.x; i < a.smem_table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
        if (MODE == 1)
            for (std::uint32_t i = threadIdx.x; i < 256; i += blockDim.x) smem[a.smem_table_bytes + i] = a.symmap[i];
    }
    __syncthreads();
    if (!act[0]) return;

    std::uint32_t st[U];
    unsigned long long cnt[U], wr[U], fol[U], send[U];
    long long pos0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        st[u] = 0;
        cnt[u] = 0;
        fol[u] = 0;
        wr[u] = (PASS == kWrite && act[u]) ? a.chunk_offs[chunk_id[u]]
                : PASS == kScratch             ? (a.slab_off ? (act[u] ? a.slab_off[chunk_id[u]] : 0ull)
                                                             : static_cast<unsigned long long>(chunk_id[u]) * a.scap)
                                               : 0ull;
        send[u] = PASS != kScratch ? 0ull
                  : a.slab_off     ? (act[u] ? a.slab_off[chunk_id[u] + 1] : 0ull)
                                   : static_cast<unsigned long long>(chunk_id[u] + 1) * a.scap;
        pos0[u] = a.emit_from + chunk_id[u] * a.chunk - a.halo;
    }
    const std::uint32_t K = a.K, H = a.H, Hn = a.Hn;
    const long long steps = a.halo + a.chunk;

    uint4 w[U];
    auto load = [&](long long off) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = pos0[u] + off;
            w[u] = (act[u] && p >= 0 && p < a.n) ? ld_stream16(a.text + p) : make_uint4(0, 0, 0, 0);
        }
    };
    load(0);
    for (long long off = 0; off < steps; off += 16) {
        uint4 cur[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cur[u] = w[u];
        if (off + 16 < steps) load(off + 16);
        const bool owned_blk = off >= a.halo;
        bool fast = true;
        std::uint32_t pk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = pos0[u] + off;
            const bool full = p >= 0 && p + 16 <= a.n;
            if (MODE == 0) {
                std::uint32_t bad = 0;
                pk[u] = dna4_pack(cur[u], bad);
                fast = fast && (!act[u] || (full && bad == 0));
            } else {
                pk[u] = 0;
                fast = fast && (!act[u] || full);
            }
        }
        if (fast) {
            ACG_UNROLL(ACG_EXACT_UNROLL)
            for (int k = 0; k < 16; ++k) {
                std::uint32_t col[U], v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (MODE == 0) {
                        col[u] = (pk[u] >> (2 * k)) & 3u;
                    } else {
                        const std::uint32_t word = k < 4 ? cur[u].x : k < 8 ? cur[u].y : k < 12 ? cur[u].z : cur[u].w;
                        col[u] = smap[(word >> ((k & 3) * 8)) & 0xFFu];
                    }
                    const std::uint32_t r = min(st[u], H);
                    v[u] = lds_u16(hot_s + 2u * (r * K + col[u]));
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (STATS && owned_blk) fol[u] += __ldg(a.follows + st[u] * K + col[u]);
                    if (v[u] == kEsc16) v[u] = __ldg(a.next + st[u] * K + col[u]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    st[u] = v[u];
                    if (owned_blk && st[u] >= Hn && act[u] && has_out(st[u], a))
                        emit<PASS>(st[u], pos0[u] + off + k, cnt[u], wr[u], a, send[u]);
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!act[u]) continue;
#pragma unroll 1
                for (int k = 0; k < 16; ++k) {
                    const long long p = pos0[u] + off + k;
                    const bool inside = p >= 0 && p < a.n;
                    const std::uint32_t word = k < 4 ? cur[u].x : k < 8 ? cur[u].y : k < 12 ? cur[u].z : cur[u].w;
                    const int c = inside ? column_of<MODE>((word >> (8 * (k & 3))) & 0xFFu, smap, a) : -1;
                    if (STATS && owned_blk && inside)
                        fol[u] += c < 0 ? (MODE == 0 ? __ldg(a.follows_esc + st[u])
                                                     : __ldg(a.follows + st[u] * K + (K - 1)))
                                        : __ldg(a.follows + st[u] * K + c);
                    std::uint32_t nx = 0;
                    if (c >= 0) {
                        nx = lds_u16(hot_s + 2u * (min(st[u], H) * K + c));
                        if (nx == kEsc16) nx = __ldg(a.next + st[u] * K + c);
                    }
                    st[u] = nx;
                    if (owned_blk && nx >= Hn && has_out(nx, a)) emit<PASS>(nx, p, cnt[u], wr[u], a, send[u]);
                }
            }
        }
    }
    if (PASS != kWrite) {
        unsigned long long f = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!act[u]) continue;
            a.chunk_counts[chunk_id[u]] = cnt[u];
            f += fol[u];
        }
        if (STATS && a.follows_total && f) atomicAdd(a.follows_total, f);
        if (a.chunk_max) {  // largest chunk count (sizes the next run's slabs)
            unsigned long long m = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) m = max(m, act[u] ? cnt[u] : 0ull);
            if (m > *static_cast<volatile unsigned long long*>(a.chunk_max)) atomicMax(a.chunk_max, m);
        }
    }
}

// ===================================================================== K1s ==
// Truncated-automaton fast pass (dna4 alphabet). Per step and stream:
//   c2 = PRMT(byte k of (word & 0x06060606))      column * 2
//   a  = (v * 8 + c2) & 0x3FFFF                    next row address (drops the flag bit)
//   v  = LDS.U16 [a + table]                       (table base folded into the LDS)
//   acc |= v                                       flag accumulator
// Interior threads (all U chunk windows inside the buffer) read text with
// unchecked 16*RB-byte refills per stream, double-buffered one refill ahead
// (256-bit loads when 32-byte aligned), validated with a 6-op SIMD test per
// word (exactly A,C,G,T pass). A block with any non-ACGT byte or past a text
// edge is walked per byte from the same registers. Every 4 steps the
// sub-block's flag bit and start state are folded into registers.
//
// Event log. After each 16-step block the warp ballots its flagged streams and
// writes their events to consecutive slots of a per-warp buffer (coalesced):
//   w0 = walk offset of the block | flag bits << 17 | stream slot (lane*U+u) << 21
//        | w2 valid << 28 | w3 valid << 29
//   w1 = A_H state at sub-blocks 0,1 (u16 each), w2 = sub-blocks 2,3
//   w3 = this block's 16 packed 2-bit columns (valid if w0 bit 28)
__device__ __forceinline__ std::uint32_t lds_hot(std::uint32_t off) {
    std::uint16_t v;
    asm volatile("{ .reg .u32 t; mov.u32 t, acg_hot_smem; add.u32 t, t, %1; ld.shared.u16 %0, [t]; }"
                 : "=h"(v)
                 : "r"(off));
    return v;
}

// 0 iff all 4 bytes of w are in {A,C,G,T}
__device__ __forceinline__ std::uint32_t acgt_bad(std::uint32_t w) {
    const std::uint32_t t = ((w >> 2) & ~(w >> 1)) & 0x01010101u;  // byte is T-like ((b & 6) == 4)
    const std::uint32_t z = (w ^ 0x41414141u) & 0xF9F9F9F9u;
    return z ^ (t * 0x11u);
}

// 16 columns packed 2 bits each (symbol k at bits 2k), for the event record
__device__ __forceinline__ std::uint32_t pack_cols(const uint4& w) {
    const std::uint32_t m0 = ((w.x >> 1) & 0x03030303u) * 0x01041040u, m1 = ((w.y >> 1) & 0x03030303u) * 0x01041040u;
    const std::uint32_t m2 = ((w.z >> 1) & 0x03030303u) * 0x01041040u, m3 = ((w.w >> 1) & 0x03030303u) * 0x01041040u;
    return __byte_perm(__byte_perm(m0, m1, 0x0073u), __byte_perm(m2, m3, 0x7300u), 0x7610u);
}

__device__ __forceinline__ uint4 ldg_text(const std::uint8_t* p) {
#ifdef ACG_ABLATE_TEXT
    const std::uint32_t h = static_cast<std::uint32_t>(reinterpret_cast<std::uintptr_t>(p)) * 2654435761u;
    const std::uint32_t m = 0x41414141u | ((h & 0x06060606u));
    return make_uint4(m, m ^ 0x02020202u, m ^ 0x04040404u, m ^ 0x06060606u);
#endif
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// 32 bytes (two blocks) with one 256-bit load (sm_100: LDG.E.ENL2.256); p 32-byte aligned
__device__ __forceinline__ void ldg_text32(const std::uint8_t* p, uint4& lo, uint4& hi) {
#ifdef ACG_ABLATE_TEXT
    lo = ldg_text(p);
    hi = ldg_text(p + 16);
    return;
#endif
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.L2::128B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p));
}

// 16 bytes at p (any byte of [p, p+16) inside [0, n)); bytes past n are masked by the caller
__device__ __forceinline__ uint4 ldg_block_checked(const std::uint8_t* text, long long p, long long n) {
    return (p >= 0 && p < n) ? ldg_text(text + p) : make_uint4(0, 0, 0, 0);
}

// One 16-step block of U streams from registers.
template <int U>
__device__ __forceinline__ void k1s_block(const uint4 (&wb)[U], std::uint32_t (&st)[U], std::uint32_t (&fl)[U],
                                          std::uint32_t (&s01)[U], std::uint32_t (&s23)[U]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        std::uint32_t acc[U], w6[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const std::uint32_t word = j == 0 ? wb[u].x : j == 1 ? wb[u].y : j == 2 ? wb[u].z : wb[u].w;
            w6[u] = word & 0x06060606u;
            if (j == 0) s01[u] = st[u];
            else if (j == 1) s01[u] |= st[u] << 16;
            else if (j == 2) s23[u] = st[u];
            else s23[u] |= st[u] << 16;
            acc[u] = 0;
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            std::uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = lds_hot((st[u] * 8u + __byte_perm(w6[u], 0u, 0x4440u + kk)) & 0x3FFFFu);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc[u] |= v[u];
                st[u] = v[u];  // flag bit stripped by the next address mask
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const std::uint32_t bit = (acc[u] >> (15 - j)) & (1u << j);
            fl[u] = j ? (fl[u] | bit) : bit;
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        st[u] &= 0x7FFFu;
        s01[u] &= 0x7FFF7FFFu;
        s23[u] &= 0x7FFF7FFFu;
    }
}

// One 16-step block of one stream, per byte from registers: bytes outside
// [0, n) and non-ACGT bytes are escapes (every state goes to the root).
__device__ __forceinline__ void k1s_block_slow(const uint4 wv, long long pb, long long n, std::uint32_t& st,
                                               std::uint32_t& fl, std::uint32_t& s01, std::uint32_t& s23) {
    fl = 0;
    s01 = 0;
    s23 = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if ((k & 3) == 0) {
            const int j = k >> 2;
            if (j < 2) s01 |= st << (16 * j);
            else s23 |= st << (16 * (j - 2));
        }
        const std::uint32_t word = k < 4 ? wv.x : k < 8 ? wv.y : k < 12 ? wv.z : wv.w;
        const std::uint32_t bb = (word >> (8 * (k & 3))) & 0xFFu;
        const long long p = pb + k;
        if (p < 0 || p >= n || !(bb == 'A' || bb == 'C' || bb == 'G' || bb == 'T')) {
            st = 0;
            continue;
        }
        const std::uint32_t v = lds_hot(st * 8u + (bb & 6u));
        if (v & 0x8000u) fl |= 1u << (k >> 2);
        st = v & 0x7FFFu;
    }
}

template <int U, int RB, int TPB>  // RB = 16-byte blocks per refill
__global__ void __launch_bounds__(TPB, 1) sparse_scan_kernel(const ScanArgs a) {
    const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (static_cast<long long>(blockIdx.x) * blockDim.x * U >= a.n_chunks) return;
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.hotH);
        uint4* dst = reinterpret_cast<uint4*>(acg_hot_smem);
        for (std::uint32_t i = threadIdx.x; i < a.smem_table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long wid = tid >> 5;
    if (wid * 32 * U >= a.n_chunks) return;  // whole warp idle (idle lanes of a live warp stay for the ballots)
    const long long c0 = tid * U;             // streams walk chunks c0 .. c0+U-1
    const int n_act = static_cast<int>(max(0ll, min(static_cast<long long>(U), a.n_chunks - c0)));
    const long long p0 = a.emit_from + c0 * a.chunk - a.halo;  // stream u starts at p0 + u*chunk
    const long long steps = a.halo + a.chunk;
    const std::uint32_t wcap = a.ev_cap;
    uint4* evw = reinterpret_cast<uint4*>(a.events) + static_cast<unsigned long long>(wid) * wcap;
    const unsigned lt_mask = (1u << lane) - 1u;
    std::uint32_t wn = 0;  // warp-uniform event count

    std::uint32_t st[U];
#pragma unroll
    for (int u = 0; u < U; ++u) st[u] = 0;

    // interior: every block of every stream lies inside [0, n) -> unchecked loads
    const bool interior = n_act == U && p0 >= 0 && p0 + (U - 1) * a.chunk + steps <= a.n;
    const std::uint8_t* ptr = a.text + p0;
    const long long cs = a.chunk;
    const std::uint32_t R = 16u * RB;
#ifdef ACG_NO_LDG256
    const bool al32 = false;
#else
    const bool al32 = ((reinterpret_cast<std::uintptr_t>(ptr) | static_cast<std::uintptr_t>(cs)) & 31u) == 0;
#endif
    uint4 wa[U][RB], wb[U][RB];
    auto load = [&](uint4 (&buf)[U][RB], std::uint32_t off0) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (interior && al32) {
#pragma unroll
                for (int b = 0; b + 1 < RB; b += 2) ldg_text32(ptr + u * cs + off0 + 16 * b, buf[u][b], buf[u][b + 1]);
                if (RB & 1) buf[u][RB - 1] = ldg_text(ptr + u * cs + off0 + 16 * (RB - 1));
            } else if (interior) {
#pragma unroll
                for (int b = 0; b < RB; ++b) buf[u][b] = ldg_text(ptr + u * cs + off0 + 16 * b);
            } else {
#pragma unroll
                for (int b = 0; b < RB; ++b) {
                    const long long o = u * cs + off0 + 16 * b;
                    buf[u][b] = (u < n_act && off0 + 16 * b < steps) ? ldg_block_checked(a.text, p0 + o, a.n)
                                                                    : make_uint4(0, 0, 0, 0);
                }
            }
        }
    };
    auto process = [&](const uint4 (&buf)[U][RB], std::uint32_t off0) {
#pragma unroll
        for (int b = 0; b < RB; ++b) {
            const std::uint32_t off = off0 + 16u * b;
            if (off >= steps) break;
            std::uint32_t bad = 0;
#ifndef ACG_ABLATE_VALIDATE
#pragma unroll
            for (int u = 0; u < U; ++u)
                bad |= acgt_bad(buf[u][b].x) | acgt_bad(buf[u][b].y) | acgt_bad(buf[u][b].z) | acgt_bad(buf[u][b].w);
#endif
            if (!interior) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const long long p = p0 + u * cs + off;
                    if (u < n_act && !(p >= 0 && p + 16 <= a.n)) bad = 1;
                }
            }
            std::uint32_t fl[U], s01[U], s23[U];
            const bool fast = bad == 0;
            if (fast) {
                uint4 wv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) wv[u] = buf[u][b];
                k1s_block<U>(wv, st, fl, s01, s23);
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    fl[u] = 0;
                    if (u >= n_act) continue;
                    k1s_block_slow(buf[u][b], p0 + u * cs + off, a.n, st[u], fl[u], s01[u], s23[u]);
                }
            }
            // warp-coalesced event log (converged here)
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (u >= n_act) fl[u] = 0;
#ifdef ACG_ABLATE_EVENTS
                wn ^= fl[u] ^ s01[u] ^ s23[u];
                continue;
#endif
                const unsigned m = __ballot_sync(0xffffffffu, fl[u] != 0);
                if (m) {
                    if (fl[u]) {
                        const std::uint32_t idx = min(wn + static_cast<std::uint32_t>(__popc(m & lt_mask)), wcap - 1);
                        evw[idx] = make_uint4(off | (fl[u] << 17) | (static_cast<std::uint32_t>(lane * U + u) << 21) |
                                                  (fast ? 1u << 28 : 0u),
                                              s01[u], s23[u], fast ? pack_cols(buf[u][b]) : 0u);
                    }
                    wn += static_cast<std::uint32_t>(__popc(m));
                }
            }
        }
    };
    load(wa, 0);
    for (std::uint32_t off0 = 0; off0 < steps; off0 += 2 * R) {
        if (off0 + R < steps) load(wb, off0 + R);
        process(wa, off0);
        if (off0 + R >= steps) break;
        if (off0 + 2 * R < steps) load(wa, off0 + 2 * R);
        process(wb, off0 + R);
    }
#ifdef ACG_ABLATE_EVENTS
    if (wn == 0x12345678u) a.ev_count[wid] = st[0];
    wn = 0;
#endif
    if (lane == 0) {
        a.ev_count[wid] = wn;
        if (a.ev_total && wn) atomicAdd(a.ev_total, static_cast<unsigned long long>(wn));
    }
}

// ===================================================================== K1f ==
// Event replay, one warp per K1s warp buffer (32*U chunks), lanes over its
// events (coalesced). Every flagged step is walked INDEPENDENTLY: re-walk A_H
// over each flagged 4-step sub-block from its recorded start state
// (reproducing the fast pass's states exactly), and from every flagged
// transition (s, c) walk the full DFA until the state is hot again,
// collecting candidate outputs (chunk slot, offset, state).
//
// Exactness without ordering: a flagged transition taken from a PROXY state
// (inside a true cold excursion) starts a walk whose state is, at every
// offset, a node-suffix of the text - a suffix of the true state - so its
// outputs are a subset of the true outputs there, and it only reaches offsets
// the true excursion covers (while its state is cold, the true state is at
// least as deep). Every true excursion starts with an exact flagged
// transition. Hence out(deepest candidate at each offset) is exactly the true
// output set: per chunk, keep for each offset the deepest candidate.
//
// The warp then writes every chunk's record count, adds per-state visits of
// the kept candidates, and exports them (offset order, with their record
// prefix inside the chunk) for the emit pass. Candidates are rare in sparse
// mode; a lane holding more than kCand of them makes the warp fall back to an
// exact replay of its chunks.
constexpr int kCand = 8;      // candidates per lane in the resolver (32*kCand per buffer)
constexpr int kCandList = 256;  // per-buffer candidate list in global memory
constexpr int kExport = 8;  // exported candidates per chunk (more: emit re-walks the chunk)

struct Cands {
    std::uint32_t key[kCand];  // slot << 24 | walk offset
    std::uint32_t st[kCand];
    int n;  // may exceed kCand (overflow)
};

__device__ __forceinline__ int text_col(const ScanArgs& a, long long p) {
    const std::uint32_t b = (p >= 0 && p < a.n) ? a.text[p] : 0u;
    return column_of<0>(b, nullptr, a);
}

// Full-DFA walk from (s, col) at walk offset i until the state is hot again;
// collects candidate outputs. Columns past the logged block come from the text.
__device__ __forceinline__ void excursion(std::uint32_t s, std::uint32_t col, long long i, long long boff,
                                          std::uint32_t win, bool wok, long long pos0, long long steps,
                                          std::uint32_t slot, Cands& cd, const ScanArgs& a) {
    std::uint32_t x = __ldg(a.next + s * 4u + col);
    for (;;) {
        if (i >= a.halo && has_out(x, a)) {
            if (cd.n < kCand) {
                cd.key[cd.n] = (slot << 24) | static_cast<std::uint32_t>(i);
                cd.st[cd.n] = x;
            }
            ++cd.n;
        }
        if (x < a.H || i + 1 >= steps) return;
        ++i;
        const long long d = i - boff;
        const int cc = (wok && d < 16) ? static_cast<int>((win >> (2 * d)) & 3u) : text_col(a, pos0 + i);
        x = cc < 0 ? 0u : __ldg(a.next + x * 4u + static_cast<std::uint32_t>(cc));
    }
}

__device__ __forceinline__ void walk_event(const uint4 e, long long chunk_base, std::uint32_t tab, Cands& cd,
                                           const ScanArgs& a) {
    const long long boff = e.x & 0x1FFFFu;
    const std::uint32_t fl = (e.x >> 17) & 0xFu;
    const std::uint32_t slot = (e.x >> 21) & 0x7Fu;
    const bool wok = (e.x >> 28) & 1u;
    const long long pos0 = a.emit_from + (chunk_base + slot) * a.chunk - a.halo;
    const long long steps = a.halo + a.chunk;
    // re-walk A_H from the first flagged sub-block to the end of the last one
    const int j0 = __ffs(fl) - 1, j1 = 31 - __clz(fl);
    std::uint32_t s = e.y;
    if (wok) {
        for (int d = 4 * j0; d < 4 * j1 + 4; ++d) {
            const std::uint32_t col = (e.z >> (2 * d)) & 3u;
            const std::uint32_t v = lds_u16(tab + (s << 3) + (col << 1));
#ifndef ACG_ABLATE_FIX_EXC
            if (v & 0x8000u) excursion(s, col, boff + d, boff, e.z, true, pos0, steps, slot, cd, a);
#else
            if (v == 0x12345u) cd.n = 99;
#endif
            s = v & 0x7FFFu;
        }
    } else {  // block with escapes / text edges: columns from the text
        for (int d = 4 * j0; d < 4 * j1 + 4; ++d) {
            const int col = text_col(a, pos0 + boff + d);
            if (col < 0) {
                s = 0;
                continue;
            }
            const std::uint32_t v = lds_u16(tab + (s << 3) + (static_cast<std::uint32_t>(col) << 1));
            if (v & 0x8000u)
                excursion(s, static_cast<std::uint32_t>(col), boff + d, boff, 0u, false, pos0, steps, slot, cd, a);
            s = v & 0x7FFFu;
        }
    }
}

// Exact sequential replay of one chunk window by one lane: walk A_H from shared
// memory, replaying each flagged transition's excursion exactly (no event log).
template <int PASS>
__device__ __noinline__ void exact_chunk_walk(long long c, std::uint32_t tab, const ScanArgs& a) {
    const long long pos0 = a.emit_from + c * a.chunk - a.halo;
    const long long steps = a.halo + a.chunk;
    unsigned long long cnt = 0, wr = PASS == kWrite ? a.chunk_offs[c] : 0ull;
    std::uint32_t s = 0;
    for (long long o = 0; o < steps; ++o) {
        const int col = text_col(a, pos0 + o);
        if (col < 0) {
            s = 0;
            continue;
        }
        const std::uint32_t v = lds_u16(tab + (s << 3) + (static_cast<std::uint32_t>(col) << 1));
        if (!(v & 0x8000u)) {
            s = v & 0x7FFFu;
            continue;
        }
        std::uint32_t x = __ldg(a.next + s * 4u + static_cast<std::uint32_t>(col));
        for (;;) {
            if (o >= a.halo && has_out(x, a)) emit<PASS>(x, pos0 + o, cnt, wr, a);
            if (x < a.H || o + 1 >= steps) break;
            ++o;
            const int cc = text_col(a, pos0 + o);
            x = cc < 0 ? 0u : __ldg(a.next + x * 4u + static_cast<std::uint32_t>(cc));
        }
        s = x < a.H ? x : 0u;
    }
    if (PASS == kCount) a.chunk_counts[c] = cnt;
}

__device__ __noinline__ void resolve_warp(Cands cd, long long chunk_base, int n_slots, int lane, const ScanArgs& a);

// F1: re-walk the flagged sub-blocks of one warp buffer (lanes over events,
// coalesced reads), appending one excursion task per flagged step:
//   w0 = chunk index, w1 = walk offset | A_H state before the step << 17,
//   w2 = column | block columns valid << 2, w3 = the block's packed columns.
template <int U>
__device__ void fixup_rewalk_warp(long long wid, std::uint32_t tab, int lane, uint4* region, std::uint32_t& nreg,
                                  const ScanArgs& a) {
    const long long chunk_base = wid * 32 * U;
    const std::uint32_t ne = a.ev_count[wid];
    if (ne > a.ev_cap) {  // cannot happen (one slot per block and stream); defensive
        if (lane == 0) a.cand_cnt[wid] = 0xFFFFFFFFu;
        return;
    }
    const uint4* ev = reinterpret_cast<const uint4*>(a.events) + static_cast<unsigned long long>(wid) * a.ev_cap;
    const unsigned lt = (1u << lane) - 1u;
    for (std::uint32_t base = 0; base < ne; base += 32) {
        const std::uint32_t j = base + lane;
        const bool have = j < ne;
        const uint4 e = have ? ev[j] : make_uint4(0, 0, 0, 0);
        const long long boff = e.x & 0x1FFFFu;
        std::uint32_t fl = have ? (e.x >> 17) & 0xFu : 0u;
        const std::uint32_t slot = (e.x >> 21) & 0x7Fu;
        const bool wok = (e.x >> 28) & 1u;
        const long long chunk = chunk_base + slot;
        const long long pos0 = a.emit_from + chunk * a.chunk - a.halo;
        // one round per flagged sub-block of the busiest lane (usually one)
        while (__any_sync(0xffffffffu, fl != 0)) {
            const bool act = fl != 0;
            const int jj = act ? __ffs(fl) - 1 : 0;
            fl &= fl - 1;
            std::uint32_t s = ((jj < 2 ? e.y : e.z) >> (16 * (jj & 1))) & 0x7FFFu;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int d = 4 * jj + kk;
                bool task = false;
                std::uint32_t col = 0;
                const std::uint32_t sprev = s;
                if (act) {
                    int c;
                    if (wok) c = static_cast<int>((e.w >> (2 * d)) & 3u);
                    else c = text_col(a, pos0 + boff + d);
                    if (c < 0) {
                        s = 0;
                    } else {
                        col = static_cast<std::uint32_t>(c);
                        const std::uint32_t v = lds_u16(tab + (s << 3) + (col << 1));
                        task = (v & 0x8000u) != 0;
                        s = v & 0x7FFFu;
                    }
                }
                const unsigned m = __ballot_sync(0xffffffffu, task);
                if (m) {
                    if (task) {
                        const std::uint32_t q = nreg + __popc(m & lt);
                        if (q < a.task_cap)
                            region[q] = make_uint4(static_cast<std::uint32_t>(chunk),
                                                   static_cast<std::uint32_t>(boff + d) | (sprev << 17),
                                                   col | (wok ? 4u : 0u), e.w);
                    }
                    nreg += static_cast<std::uint32_t>(__popc(m));
                }
            }
        }
    }
}

template <int U>
__global__ void __launch_bounds__(1024, 1) fixup_rewalk_kernel(const ScanArgs a) {
    extern __shared__ __align__(16) std::uint8_t smem[];
    const std::uint32_t tab = smem_u32(smem);
    const int lane = threadIdx.x & 31;
    const long long n_work = (a.n_chunks + 32 * U - 1) / (32 * U);
    const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    const long long w0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if ((static_cast<long long>(blockIdx.x) * blockDim.x >> 5) >= n_work) return;
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.hotH);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (std::uint32_t i = threadIdx.x; i < a.smem_table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    // each fix-up warp appends its tasks to its own region (task_cap tasks) with a register counter
    uint4* region = reinterpret_cast<uint4*>(a.tasks) + static_cast<unsigned long long>(w0) * a.task_cap;
    std::uint32_t nreg = 0;
    for (long long w = w0; w < n_work; w += warps) fixup_rewalk_warp<U>(w, tab, lane, region, nreg, a);
    if (lane == 0) {
        a.task_cnt[w0] = nreg;
        atomicMax(a.task_max, nreg);
    }
}

// F2: one thread per excursion task: walk the full DFA (L2) from the exact or
// proxy state until the state is hot again; candidates go to the task's
// buffer list.
constexpr int kWalkILP = 4;

template <int U>
__device__ __forceinline__ void record_cand(long long chunk, long long i, std::uint32_t x, const ScanArgs& a) {
    const long long wid = chunk / (32 * U);
    const std::uint32_t slot = static_cast<std::uint32_t>(chunk - wid * 32 * U);
    const std::uint32_t q = atomicAdd(a.cand_cnt + wid, 1u);
    if (q < kCandList)
        reinterpret_cast<uint2*>(a.cand_list)[static_cast<unsigned long long>(wid) * kCandList + q] =
            make_uint2((slot << 24) | static_cast<std::uint32_t>(i), x);
}

// F2: two warps per task region; every lane walks kWalkILP tasks at once
// (independent dependent-lookup chains interleaved).
template <int U>
__global__ void __launch_bounds__(256) fixup_walk_kernel(const ScanArgs a, std::uint32_t n_regions) {
    const long long steps = a.halo + a.chunk;
    const std::uint32_t H = a.H;
    const std::uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const std::uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (std::uint32_t rw = gw; rw < 2 * n_regions; rw += nw) {
        const std::uint32_t r = rw >> 1, half = rw & 1;
        const std::uint32_t nt = min(a.task_cnt[r], a.task_cap);
        const uint4* tks = reinterpret_cast<const uint4*>(a.tasks) + static_cast<unsigned long long>(r) * a.task_cap;
        // lanes of this warp take tasks half*32 + lane + 64*q (q = 0, 1, ...), kWalkILP at a time
        for (std::uint32_t t0 = half * 32 + lane; t0 < nt; t0 += 64 * kWalkILP) {
            std::uint32_t x[kWalkILP], pk[kWalkILP];
            long long i[kWalkILP], boff[kWalkILP], chunk[kWalkILP];
            bool live[kWalkILP], wok[kWalkILP];
#pragma unroll
            for (int c = 0; c < kWalkILP; ++c) {
                const std::uint32_t t = t0 + 64u * c;
                live[c] = t < nt;
                const uint4 tk = live[c] ? tks[t] : make_uint4(0, 0, 0, 0);
                chunk[c] = tk.x;
                i[c] = tk.y & 0x1FFFFu;
                boff[c] = i[c] & ~15ll;
                wok[c] = (tk.z >> 2) & 1u;
                pk[c] = tk.w;
                x[c] = live[c] ? __ldg(a.next + (tk.y >> 17) * 4u + (tk.z & 3u)) : 0u;
            }
            for (;;) {
                bool any = false;
#pragma unroll
                for (int c = 0; c < kWalkILP; ++c) {
                    if (!live[c]) continue;
                    if (i[c] >= a.halo && has_out(x[c], a)) record_cand<U>(chunk[c], i[c], x[c], a);
                    if (x[c] < H || i[c] + 1 >= steps) {
                        live[c] = false;
                        continue;
                    }
                    any = true;
                    ++i[c];
                    const long long d = i[c] - boff[c];
                    const long long pos0 = a.emit_from + chunk[c] * a.chunk - a.halo;
                    const int cc = (wok[c] && d < 16) ? static_cast<int>((pk[c] >> (2 * d)) & 3u) : text_col(a, pos0 + i[c]);
                    x[c] = cc < 0 ? 0u : __ldg(a.next + x[c] * 4u + static_cast<std::uint32_t>(cc));
                }
                if (!any) break;
            }
        }
    }
}

// F3: per warp buffer: counts (and, when candidates exist, dedup + export).
template <int U>
__device__ void fixup_resolve_warp(long long wid, std::uint32_t tab, int lane, const ScanArgs& a) {
    const long long chunk_base = wid * 32 * U;
    const int n_slots = static_cast<int>(min(static_cast<long long>(32 * U), a.n_chunks - chunk_base));
    const std::uint32_t nc = a.cand_cnt[wid];
    if (nc > 32u * kCand) {  // exact replay of every chunk of this buffer, one lane per chunk (practically never)
        for (int sl = lane; sl < n_slots; sl += 32) {
            a.cand_n[chunk_base + sl] = 0xFFFFFFFFu;  // emit pass re-walks
            exact_chunk_walk<kCount>(chunk_base + sl, tab, a);
        }
        return;
    }
    if (nc == 0) {
        for (int sl = lane; sl < n_slots; sl += 32) {
            a.chunk_counts[chunk_base + sl] = 0;
            a.cand_n[chunk_base + sl] = 0;
        }
        return;
    }
    Cands cd;
    cd.n = 0;
    const uint2* cl = reinterpret_cast<const uint2*>(a.cand_list) + static_cast<unsigned long long>(wid) * kCandList;
#pragma unroll
    for (int q = 0; q < kCand; ++q) {
        const std::uint32_t idx = static_cast<std::uint32_t>(lane) + 32u * q;
        if (idx < nc) {
            const uint2 v = cl[idx];
            cd.key[q] = v.x;
            cd.st[q] = v.y;
            cd.n = q + 1;
        }
    }
    resolve_warp(cd, chunk_base, n_slots, lane, a);
}

template <int U>
__global__ void __launch_bounds__(512, 1) fixup_resolve_kernel(const ScanArgs a) {
    extern __shared__ __align__(16) std::uint8_t smem[];
    const std::uint32_t tab = smem_u32(smem);
    const int lane = threadIdx.x & 31;
    const long long n_work = (a.n_chunks + 32 * U - 1) / (32 * U);
    const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    const long long w0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if ((static_cast<long long>(blockIdx.x) * blockDim.x >> 5) >= n_work) return;
    // the table is only needed by the exact fallback
    bool need = false;
    for (long long w = w0; w < n_work; w += warps) need |= a.cand_cnt[w] > 32u * kCand;
    if (__syncthreads_or(need)) {
        const uint4* src = reinterpret_cast<const uint4*>(a.hotH);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (std::uint32_t i = threadIdx.x; i < a.smem_table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
        __syncthreads();
    }
    for (long long w = w0; w < n_work; w += warps) fixup_resolve_warp<U>(w, tab, lane, a);
}

// Dedup, counts, visits and export of one warp buffer's candidates (rare path).
__device__ __noinline__ void resolve_warp(Cands cd, long long chunk_base, int n_slots, int lane, const ScanArgs& a) {
    // keep, per (slot, offset), the deepest candidate (ties: lowest (lane, index))
    bool keep[kCand];
    std::uint32_t dep[kCand], nout[kCand];
#pragma unroll
    for (int q = 0; q < kCand; ++q) {
        keep[q] = q < cd.n;
        dep[q] = q < cd.n ? __ldg(a.depth + cd.st[q]) : 0u;
        nout[q] = q < cd.n ? __ldg(a.out_off + cd.st[q] + 1) - __ldg(a.out_off + cd.st[q]) : 0u;
    }
    for (int src = 0; src < 32; ++src) {
        const int nsrc = __shfl_sync(0xffffffffu, cd.n, src);
        for (int r = 0; r < nsrc; ++r) {
            std::uint32_t k_r = 0, s_r = 0;
#pragma unroll
            for (int q = 0; q < kCand; ++q)
                if (q == r) {
                    k_r = cd.key[q];
                    s_r = cd.st[q];
                }
            k_r = __shfl_sync(0xffffffffu, k_r, src);
            s_r = __shfl_sync(0xffffffffu, s_r, src);
            const std::uint32_t d_r = __ldg(a.depth + s_r);
#pragma unroll
            for (int q = 0; q < kCand; ++q) {
                if (!keep[q] || k_r != cd.key[q]) continue;
                const bool me = src == lane && r == q;
                const bool earlier = src < lane || (src == lane && r < q);
                if (!me && (d_r > dep[q] || (d_r == dep[q] && earlier))) keep[q] = false;
            }
        }
    }
    // per kept candidate: rank and record prefix among kept candidates of its chunk
    std::uint32_t rank[kCand];
    unsigned long long pre[kCand];
#pragma unroll
    for (int q = 0; q < kCand; ++q) {
        rank[q] = 0;
        pre[q] = 0;
    }
    for (int src = 0; src < 32; ++src) {
        const int nsrc = __shfl_sync(0xffffffffu, cd.n, src);
        for (int r = 0; r < nsrc; ++r) {
            std::uint32_t k_r = 0, n_r = 0;
            int kp_r = 0;
#pragma unroll
            for (int q = 0; q < kCand; ++q)
                if (q == r) {
                    k_r = cd.key[q];
                    n_r = nout[q];
                    kp_r = keep[q];
                }
            k_r = __shfl_sync(0xffffffffu, k_r, src);
            n_r = __shfl_sync(0xffffffffu, n_r, src);
            kp_r = __shfl_sync(0xffffffffu, kp_r, src);
#pragma unroll
            for (int q = 0; q < kCand; ++q) {
                if (!keep[q] || !kp_r) continue;
                if ((k_r >> 24) == (cd.key[q] >> 24) && k_r < cd.key[q]) {
                    ++rank[q];
                    pre[q] += n_r;
                }
            }
        }
    }
    // export + visits
#pragma unroll
    for (int q = 0; q < kCand; ++q) {
        if (!keep[q]) continue;
        const long long c = chunk_base + (cd.key[q] >> 24);
        if (rank[q] < kExport)
            reinterpret_cast<uint4*>(a.cands)[c * kExport + rank[q]] =
                make_uint4(cd.key[q] & 0xFFFFFFu, cd.st[q], static_cast<std::uint32_t>(pre[q]),
                           static_cast<std::uint32_t>(pre[q] >> 32));
        if (a.visits) atomicAdd(a.visits + out_rank(cd.st[q], a), 1ull);
    }
    // per-chunk totals (lane per slot)
    for (int sl0 = 0; sl0 < n_slots; sl0 += 32) {
        const int sl = sl0 + lane;
        unsigned long long tot = 0;
        std::uint32_t nk = 0;
        for (int src = 0; src < 32; ++src) {
            const int nsrc = __shfl_sync(0xffffffffu, cd.n, src);
            for (int r = 0; r < nsrc; ++r) {
                std::uint32_t k_r = 0, n_r = 0;
                int kp_r = 0;
#pragma unroll
                for (int q = 0; q < kCand; ++q)
                    if (q == r) {
                        k_r = cd.key[q];
                        n_r = nout[q];
                        kp_r = keep[q];
                    }
                k_r = __shfl_sync(0xffffffffu, k_r, src);
                n_r = __shfl_sync(0xffffffffu, n_r, src);
                kp_r = __shfl_sync(0xffffffffu, kp_r, src);
                if (kp_r && static_cast<int>(k_r >> 24) == sl) {
                    tot += n_r;
                    ++nk;
                }
            }
        }
        if (sl < n_slots) {
            a.chunk_counts[chunk_base + sl] = tot;
            a.cand_n[chunk_base + sl] = nk <= static_cast<std::uint32_t>(kExport) ? nk : 0xFFFFFFFFu;
        }
    }
}

// Sparse-mode emit: one thread per chunk with matches writes the exported
// candidates' records at the chunk's slot range; a chunk whose export
// overflowed is replayed exactly (records only; its visits were counted).
__global__ void __launch_bounds__(256) sparse_emit_kernel(const ScanArgs a) {
    extern __shared__ __align__(16) std::uint8_t smem[];
    const std::uint32_t tab = smem_u32(smem);
    const long long n_work = static_cast<long long>(*a.active_count);
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    bool need_tab = false;
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n_work; t += stride)
        need_tab |= a.cand_n[a.active_list[t]] == 0xFFFFFFFFu;
    if (__syncthreads_or(need_tab)) {
        const uint4* src = reinterpret_cast<const uint4*>(a.hotH);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (std::uint32_t i = threadIdx.x; i < a.smem_table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
        __syncthreads();
    }
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n_work; t += stride) {
        const long long c = a.active_list[t];
        const std::uint32_t nk = a.cand_n[c];
        if (nk == 0xFFFFFFFFu) {
            exact_chunk_walk<kWrite>(c, tab, a);
            continue;
        }
        const long long pos0 = a.emit_from + c * a.chunk - a.halo;
        for (std::uint32_t i = 0; i < nk; ++i) {
            const uint4 cd = reinterpret_cast<const uint4*>(a.cands)[c * kExport + i];
            unsigned long long wr = a.chunk_offs[c] + (static_cast<unsigned long long>(cd.w) << 32 | cd.z), dummy = 0;
            emit<kWrite>(cd.y, pos0 + cd.x, dummy, wr, a);
        }
    }
}

// Compacts the ids of chunks with at least one match (order is irrelevant:
// every chunk writes at its own prefix offset). One atomic per block tile
// (256 threads x 8 chunks): same-address atomics serialise at L2, so
// per-warp atomics would cost ~ns each across thousands of warps.
__global__ void __launch_bounds__(256) compact_active_kernel(const unsigned long long* counts, long long n,
                                                             std::uint32_t* list, std::uint32_t* n_active) {
    __shared__ std::uint32_t warp_tot[8], base_sh;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kItems = 8;
    for (long long t0 = static_cast<long long>(blockIdx.x) * 256 * kItems; t0 < n;
         t0 += static_cast<long long>(gridDim.x) * 256 * kItems) {
        unsigned bits[kItems];
        std::uint32_t mine = 0;
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const long long i = t0 + (static_cast<long long>(warp) * kItems + k) * 32 + lane;
            bits[k] = __ballot_sync(0xFFFFFFFFu, i < n && counts[i] != 0);
            mine += __popc(bits[k]);
        }
        if (lane == 0) warp_tot[warp] = mine;
        __syncthreads();
        if (threadIdx.x == 0) {
            std::uint32_t tot = 0;
            for (int w = 0; w < 8; ++w) tot += warp_tot[w];
            base_sh = tot ? atomicAdd(n_active, tot) : 0u;
        }
        __syncthreads();
        std::uint32_t base = base_sh;
        for (int w = 0; w < warp; ++w) base += warp_tot[w];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const long long i = t0 + (static_cast<long long>(warp) * kItems + k) * 32 + lane;
            if (bits[k] & (1u << lane)) list[base + __popc(bits[k] & ((1u << lane) - 1))] = static_cast<std::uint32_t>(i);
            base += __popc(bits[k]);
        }
        __syncthreads();
    }
}

// Per-pattern counts from per-state visit counts: count(p) = sum of visits(s)
// over output states s with p in out(s). One thread per output state.
__global__ void pattern_counts_kernel(const unsigned long long* visits, const std::uint32_t* out_off,
                                      const std::uint32_t* out_ids, std::uint32_t Hn, std::uint32_t H,
                                      std::uint32_t Cn, std::uint32_t S, unsigned long long* counts) {
    (void)H;
    (void)S;
    const std::uint32_t n_out = Cn - Hn;  // output states [Hn, Cn), rank = s - Hn
    for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_out; i += gridDim.x * blockDim.x) {
        const std::uint32_t s = Hn + i;
        const unsigned long long v = visits[i];
        if (!v) continue;
        for (std::uint32_t j = out_off[s]; j < out_off[s + 1]; ++j) atomicAdd(counts + out_ids[j], v);
    }
}

// Order-independent digest of the packed records (key = end*2^20 + id) and a
// strict-order check; verification helper for the size-independent parity
// properties (tests/, bench).
__global__ void digest_kernel(const unsigned long long* rec, unsigned long long m, std::uint32_t id_bits,
                              unsigned long long* out /* [sum, xor, unsorted] */) {
    unsigned long long s = 0, x = 0, bad = 0;
    const unsigned long long mask = (1ull << id_bits) - 1;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < m;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long r = rec[i];
        const unsigned long long h = mix64(((r >> id_bits) << 20) + (r & mask));
        s += h;
        x ^= h;
        if (i + 1 < m && !(r < rec[i + 1])) bad++;
    }
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        x ^= __shfl_xor_sync(0xffffffffu, x, o);
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out + 0, s);
        atomicXor(out + 1, x);
        atomicAdd(out + 2, bad);
    }
}

// K3 of the single-pass exact mode: every chunk's slab goes to its slot range
// (one warp per chunk, coalesced); chunks whose records overflowed their slab
// are listed for the exact WRITE pass.
// With HIST, the CTA also histograms the ids it copies (shared-memory bins,
// P = n_patterns) into `counts` — the per-pattern counts without re-reading
// the records (the overflowed chunks' counts come from the WRITE pass's visits).
template <bool HIST>
__global__ void __launch_bounds__(HIST ? 1024 : 256) scratch_copy_kernel(const ScanArgs a, std::uint32_t* list,
                                                                         std::uint32_t* n_list, std::uint32_t P,
                                                                         unsigned long long* counts) {
    extern __shared__ std::uint32_t bins[];
    if (HIST) {
        for (std::uint32_t i = threadIdx.x; i < P; i += blockDim.x) bins[i] = 0;
        __syncthreads();
    }
    const unsigned long long mask = (1ull << a.id_bits) - 1;
    const int lane = threadIdx.x & 31;
    const long long wpb = blockDim.x >> 5;
    const long long warps = static_cast<long long>(gridDim.x) * wpb;
    for (long long c = static_cast<long long>(blockIdx.x) * wpb + (threadIdx.x >> 5); c < a.n_chunks; c += warps) {
        const unsigned long long k = a.chunk_counts[c];
        if (k == 0) continue;
        const unsigned long long base = a.slab_off ? a.slab_off[c] : static_cast<unsigned long long>(c) * a.scap;
        const unsigned long long cap = a.slab_off ? a.slab_off[c + 1] - base : a.scap;
        if (k > cap) {
            if (lane == 0) list[atomicAdd(n_list, 1u)] = static_cast<std::uint32_t>(c);
            continue;
        }
        const unsigned long long o = a.chunk_offs[c];
        const unsigned long long* src = a.scratch + base;
        for (unsigned long long j = lane; j < k; j += 32) {
            const unsigned long long r = src[j];
            if (o + j < a.rec_cap) a.records[o + j] = r;
            if (HIST) atomicAdd(&bins[static_cast<std::uint32_t>(r & mask)], 1u);
        }
    }
    if (HIST) {
        __syncthreads();
        for (std::uint32_t i = threadIdx.x; i < P; i += blockDim.x)
            if (bins[i]) atomicAdd(counts + i, static_cast<unsigned long long>(bins[i]));
    }
}

// Slab sizes for the next single-pass exact run from this run's chunk counts
// (+1/8 + 16 slack): out[c + 1] = size of chunk c; out[0] = 0 (prefix by CUB).
__global__ void __launch_bounds__(256) slab_sizes_kernel(const unsigned long long* counts, long long n,
                                                         unsigned long long* out) {
    for (long long c = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x; c < n;
         c += static_cast<long long>(gridDim.x) * 256) {
        const unsigned long long k = counts[c];
        out[c + 1] = k + (k >> 3) + 16;
        if (c == 0) out[0] = 0;
    }
}

// Clears up to kMax word-aligned regions in one launch (run-start counters).
struct ZeroList {
    static constexpr int kMax = 16;
    std::uint32_t* ptr[kMax];
    unsigned long long words[kMax];
    int n;
};
__global__ void __launch_bounds__(256) zero_regions_kernel(const ZeroList zl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // (may be launched programmatically)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * 256;
    for (int r = 0; r < zl.n; ++r)
        for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * 256 + threadIdx.x; i < zl.words[r];
             i += stride)
            zl.ptr[r][i] = 0u;
}

// Per-pattern counts from the final record list: per-CTA shared-memory bins
// (one u32 per pattern), flushed into the u64 counts. m = *m_ptr records,
// at most cap of them stored.
__global__ void __launch_bounds__(1024) record_hist_kernel(const unsigned long long* rec, const unsigned long long* m_ptr,
                                                           unsigned long long cap, std::uint32_t id_bits,
                                                           std::uint32_t P, unsigned long long* counts) {
    extern __shared__ std::uint32_t bins[];
    for (std::uint32_t i = threadIdx.x; i < P; i += blockDim.x) bins[i] = 0;
    __syncthreads();
    const unsigned long long m = min(*m_ptr, cap);
    const unsigned long long mask = (1ull << id_bits) - 1;
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    for (unsigned long long t = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < m; t += stride)
        atomicAdd(&bins[static_cast<std::uint32_t>(rec[t] & mask)], 1u);
    __syncthreads();
    for (std::uint32_t i = threadIdx.x; i < P; i += blockDim.x)
        if (bins[i]) atomicAdd(counts + i, static_cast<unsigned long long>(bins[i]));
}

}  // namespace kern
}  // namespace acg
