// EXACT mode, event pipeline (replaces the inline emission of
// exact_scan_kernel for list / count runs; exact_scan_kernel keeps the exact
// ScanStats walk).
//
// The reference's hot loop (acmatch::scan, proj/include/acmatch/
// aho_corasick.hpp:250-272) emits out(s) at every position whose state has
// outputs. On the GPU, doing that inside the lockstep walk made each lane load
// its state's output list from global memory and store every record itself:
// divergent, long-scoreboard bound, and a 13k-instruction kernel (ncu, cfg4:
// long_scoreboard 53 %, no_instruction 22 %). Here the walk only LOGS the
// output visits and three small passes produce the ordered list:
//
//  * KE  exact_event_kernel: the chunked lockstep DFA walk (hot rows in shared
//        memory, cold rows from L2, as exact_scan_kernel). Whenever an owned
//        step enters an output state it appends one 32-bit event
//        (offset in chunk << ob | output rank) to its chunk's event slab;
//        a full slab continues in 256-event blocks taken from a global pool
//        (linked through the slab's last slot). Per chunk: the event count.
//  * E1  event_count_kernel: per chunk, the number of records its events
//        expand to (sum of |out(s)|) -> chunk_counts (K2 prefixes them), and
//        the per-output-state visit histogram (K4 turns it into per-pattern
//        counts).
//  * E2  event_expand_kernel: one warp per chunk writes the chunk's records
//        at its slot range, coalesced: a warp scan of the events' output
//        counts, then record t of the batch is found by a binary search over
//        the scan (out ids ascending per state, positions ascending per
//        chunk: the canonical (end, id) order of aho_corasick.hpp:38-41).
#pragma once

#include <type_traits>

#include "ctab.hpp"
#include "scan_kernels.cuh"

namespace acg {
namespace kern {

constexpr std::uint32_t kEvBlock = 256;  // events per pool block (the last slot links onward)

struct EventArgs {
    std::uint32_t* ev;            // event storage: primary slabs, then the pool
    const std::uint32_t* slab_off;  // per chunk primary slab start (null: uniform c * ecap)
    std::uint32_t ecap;           // uniform primary slab size (slots incl. the link slot)
    std::uint32_t* ev_count;      // per chunk: events logged (owned steps in output states)
    std::uint32_t* pool_used;     // pool blocks taken (may exceed pool_blocks: overflow)
    std::uint32_t pool_base;      // first pool slot
    std::uint32_t pool_blocks;
    std::uint32_t ob;             // bits of the output rank in an event
    std::uint32_t n_out;          // output states (ranks)
    unsigned long long* ev_total; // E1: events of the run (sizes the next run's slabs)
};

// A run whose pool overflowed left dangling links: E1/E2 skip it (the host
// replays the run at sync with a larger pool).
__device__ __forceinline__ bool ev_pool_ok(const EventArgs& e) {
    return *static_cast<const volatile std::uint32_t*>(e.pool_used) <= e.pool_blocks;
}

__device__ __forceinline__ std::uint32_t slab_start(const EventArgs& e, long long c) {
    return e.slab_off ? e.slab_off[c] : static_cast<std::uint32_t>(c) * e.ecap;
}
__device__ __forceinline__ std::uint32_t slab_end(const EventArgs& e, long long c) {
    return e.slab_off ? e.slab_off[c + 1] : static_cast<std::uint32_t>(c + 1) * e.ecap;
}

// The slab (or block) is full: continue in a fresh pool block, linked from
// the full region's last slot `lim`. Returns the new (write slot, limit); with
// the pool exhausted it returns (1, 0) — nothing more is stored, counting goes
// on, and the host replays the run with a larger pool. (Out of line and by
// value: the walk's per-stream cursors stay in registers.)
__device__ __noinline__ uint2 ev_grow(std::uint32_t* ev, std::uint32_t* pool_used, std::uint32_t pool_base,
                                     std::uint32_t pool_blocks, std::uint32_t lim) {
    const std::uint32_t b = atomicAdd(pool_used, 1u);
    if (b >= pool_blocks) return make_uint2(1u, 0u);
    const std::uint32_t p = pool_base + b * kEvBlock;
    ev[lim] = p;
    return make_uint2(p, p + kEvBlock - 1);
}

__device__ __forceinline__ void ev_put(const EventArgs& e, std::uint32_t v, std::uint32_t& wr, std::uint32_t& lim) {
    if (wr == lim) {
        const uint2 g = ev_grow(e.ev, e.pool_used, e.pool_base, e.pool_blocks, lim);
        wr = g.x;
        lim = g.y;
    }
    if (wr < lim) e.ev[wr++] = v;
}

__device__ __forceinline__ std::uint32_t out_rank_of(std::uint32_t s, std::uint32_t H, std::uint32_t Hn,
                                                    std::uint32_t Cn) {
    (void)H;
    (void)Cn;
    return s - Hn;  // output states [Hn, Cn) are contiguous
}
__device__ __forceinline__ std::uint32_t state_of_rank(std::uint32_t r, std::uint32_t H, std::uint32_t Hn,
                                                      std::uint32_t Cn) {
    (void)H;
    (void)Cn;
    return Hn + r;
}

// ===================================================================== KE ==
// Chunk c of the stream (thread t, slot u) in CTA b: c = (t*U + u) * gridDim + b,
// so every CTA of a one-per-SM grid gets the same number of chunks whatever the
// chunk count's rounding.
//
// Per step and stream (fast path): the column from the 16-byte word (PRMT +
// a shared-memory byte map, or 2-bit codes for DNA), t = s*K + col, the hot
// row entry LDS [min(t, H*K)] (row H is all-escape), the L2 load of the cold
// row entry only under the escape predicate, then the output test on the
// contiguous output range [Hn, Cn) and a PREDICATED store of the event: no
// per-event branch. Each owned 16-step block starts with >= 16 free slots in
// the chunk's current region (else the region is closed with filler events
// and continued in a pool block), so the stores need no bounds check.
constexpr std::uint32_t kEvPad = 0xFFFFFFFFu;  // filler slot of a region closed early: expands to nothing

template <int U, int MODE>
__global__ void __launch_bounds__(U <= 2 ? 2 * kTPB : kTPB, 1) exact_event_kernel(const ScanArgs a, const EventArgs e) {
    extern __shared__ __align__(16) std::uint8_t smem[];
    std::uint8_t* smap = smem + a.smem_table_bytes;  // byte -> column (MODE 1)
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.hot16);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (std::uint32_t i = threadIdx.x; i < a.smem_table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
        if (MODE == 1)
            for (std::uint32_t i = threadIdx.x; i < 256; i += blockDim.x) smap[i] = a.symmap[i];
    }
    __syncthreads();
    const std::uint32_t hot_s = smem_u32(smem);

    const long long G = gridDim.x;
    long long cid[U];
    bool act[U], live[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        cid[u] = (static_cast<long long>(threadIdx.x) * U + u) * G + blockIdx.x;
        act[u] = cid[u] < a.n_chunks;
        live[u] = act[u];
    }
    if (!act[0]) return;  // (cid ascends with u: no stream of this thread is active)
    const std::uint32_t K = a.K, HK = a.H * a.K, Hn = a.Hn, nout = a.Cn - a.Hn, ob = e.ob;
    const long long halo = a.halo, steps = a.halo + a.chunk, n = a.n;
    const std::uint32_t* __restrict__ next = a.next;
    std::uint32_t* __restrict__ ev = e.ev;

    std::uint32_t st[U], wr[U], lim[U], cnt[U];
    long long pos0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        st[u] = 0;
        cnt[u] = 0;
        wr[u] = act[u] ? slab_start(e, cid[u]) : 0u;
        lim[u] = act[u] ? slab_end(e, cid[u]) - 1u : 0u;  // last slot = link to a pool block
        pos0[u] = a.emit_from + cid[u] * a.chunk - halo;
    }

    uint4 w[U];
    auto load = [&](long long off) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = pos0[u] + off;
            w[u] = (act[u] && p >= 0 && p < n) ? ld_stream16(a.text + p) : make_uint4(0, 0, 0, 0);
        }
    };
    // next-state lookup for the byte of column `col` (t = s*K + col)
    auto step = [&](std::uint32_t s, std::uint32_t col) -> std::uint32_t {
        const std::uint32_t t = s * K + col;
        std::uint32_t v = lds_u16z(hot_s + 2u * min(t, HK));
        if (v == kEsc16) v = __ldg(next + t);
        return v;
    };
    load(0);
    for (long long off = 0; off < steps; off += 16) {
        uint4 cur[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cur[u] = w[u];
        if (off + 16 < steps) load(off + 16);
        const bool owned_blk = off >= halo;  // halo is a multiple of 16: blocks are all-owned or all-warm-up
        std::uint32_t wr0[U];
        if (owned_blk) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (live[u] && lim[u] - wr[u] < 16u) {  // close the region, continue in a pool block
                    for (; wr[u] < lim[u]; ++wr[u], ++cnt[u]) ev[wr[u]] = kEvPad;
                    const uint2 g = ev_grow(ev, e.pool_used, e.pool_base, e.pool_blocks, lim[u]);
                    wr[u] = g.x;
                    lim[u] = g.y;
                    if (g.y == 0u) live[u] = false;  // pool exhausted: the host replays the run
                }
                wr0[u] = wr[u];
            }
        }
        bool fast = true;
        std::uint32_t pk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = pos0[u] + off;
            const bool full = p >= 0 && p + 16 <= n;
            if (MODE == 0) {
                std::uint32_t bad = 0;
                pk[u] = dna4_pack(cur[u], bad);
                fast = fast && (!act[u] || (full && bad == 0));
            } else {
                pk[u] = 0;
                fast = fast && (!act[u] || full);
            }
        }
        // event word of step k: (offset in chunk << ob) + output rank
        std::uint32_t kk = owned_blk ? static_cast<std::uint32_t>(off - halo) << ob : 0u;
        const std::uint32_t kinc = 1u << ob;
        // 16 steps of all U streams; LOG: owned block (events), else warm-up
        auto fast_block = [&](auto log_tag) {
            constexpr bool LOG = decltype(log_tag)::value;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                std::uint32_t v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    std::uint32_t col;
                    if (MODE == 0) {
                        col = (pk[u] >> (2 * k)) & 3u;
                    } else {
                        const std::uint32_t word = k < 4 ? cur[u].x : k < 8 ? cur[u].y : k < 12 ? cur[u].z : cur[u].w;
                        col = smap[__byte_perm(word, 0u, 0x4440u + (k & 3))];
                    }
                    v[u] = step(st[u], col);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    st[u] = v[u];
                    if (LOG) {
                        const std::uint32_t r = v[u] - Hn;
                        if (live[u] && r < nout) ev[wr[u]++] = kk + r;
                    }
                }
                if (LOG) kk += kinc;
            }
        };
        if (fast) {
            if (owned_blk) fast_block(std::true_type{});
            else fast_block(std::false_type{});
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!act[u]) continue;
                std::uint32_t kq = kk;
#pragma unroll 1
                for (int k = 0; k < 16; ++k, kq += kinc) {
                    const long long p = pos0[u] + off + k;
                    const bool inside = p >= 0 && p < n;
                    const std::uint32_t word = k < 4 ? cur[u].x : k < 8 ? cur[u].y : k < 12 ? cur[u].z : cur[u].w;
                    const int c = inside ? column_of<MODE>((word >> (8 * (k & 3))) & 0xFFu, smap, a) : -1;
                    const std::uint32_t nx = c >= 0 ? step(st[u], static_cast<std::uint32_t>(c)) : 0u;
                    st[u] = nx;
                    const std::uint32_t r = nx - Hn;
                    if (owned_blk && live[u] && r < nout) ev[wr[u]++] = kq + r;
                }
            }
        }
        if (owned_blk) {
#pragma unroll
            for (int u = 0; u < U; ++u) cnt[u] += wr[u] - wr0[u];
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (act[u]) e.ev_count[cid[u]] = cnt[u];
}

// =================================================================== KC ==
// The EXACT walk over the compressed hot automaton (ctab.hpp): same chunking,
// event slabs and logging as KE (chunks of at most ~2 KiB walked in rounds,
// see below), but the per-step lookup is one 32-bit
// shared-memory load of the row-displaced exception table,
//     e = tab[id + c];  next = column field of e == c ? e (tag cleared) : x
// with x = T_D[last D columns] computed from the text alone (two multiply-adds
// and one load per step, off the state's dependency chain). Cold state words
// (rare: the table holds every state that matters) step through the dense
// L2-resident table. Events carry the state word's value (hot: id, cold
// output: slots + rank); E1 maps them to output ranks.
struct CtabArgs {
    const std::uint32_t* image;   // slots exception entries, then the K^D default table
    std::uint32_t image_bytes;    // multiple of 16
    std::uint32_t slots;
    const std::uint32_t* next;    // S*K dense table, targets as state words (cold steps)
    const std::uint16_t* rank;    // id -> output rank (E1)
    const unsigned long long* info;  // event payload -> the state's packed output info (E2)
    std::uint32_t pay_mask;       // payload bits of a state word (kCtPayMask for counted words, else kCtValMask)
    bool deep;                    // deep default (ctab.hpp)
    bool cold;                    // some states are cold (else the walk carries no cold branch)
    bool counted;                 // counted words AND this run skips E1: the walk writes chunk_counts and the event total
};

// A cold state word's step: the dense L2-resident table of state words. Out of
// line so the walk's straight-line code carries one branch, not its address
// arithmetic (cold steps are rare: the table holds every state that matters).
__device__ __noinline__ std::uint32_t ctab_cold_step(const std::uint32_t* next, std::uint32_t K, std::uint32_t slots,
                                                     std::uint32_t Hn, std::uint32_t pay_mask, std::uint32_t sw,
                                                     std::uint32_t c4) {
    const std::uint32_t s = (sw & kCtOut) ? (sw & pay_mask) - slots + Hn : (sw & kCtValMask);
    return __ldg(next + static_cast<std::size_t>(s) * K + (c4 >> 2));
}

// a value the compiler must keep in a register (no rematerialisation of the
// shared-window address arithmetic inside the unrolled steps)
__device__ __forceinline__ std::uint32_t pinned_reg(std::uint32_t v) {
    std::uint32_t r;
    asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}

// Thread block: 1024 threads at one stream per thread, 512 above (the columns
// of a whole group of steps are held in registers).
template <int U, int D, bool DEEP, bool COLD>
__global__ void __launch_bounds__(U == 1 ? 2 * kTPB : kTPB, 1) ctab_event_kernel(const ScanArgs a, const EventArgs e,
                                                                                 const CtabArgs ct) {
    constexpr int GL = U <= 2 ? 16 : 8;  // steps per group: their columns are looked up together, ahead of the walk
    extern __shared__ __align__(16) std::uint8_t smem[];
    {
        std::uint8_t* smap4 = smem + ct.image_bytes;  // byte -> 4 * column
        const uint4* src = reinterpret_cast<const uint4*>(ct.image);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (std::uint32_t i = threadIdx.x; i < ct.image_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
        for (std::uint32_t i = threadIdx.x; i < 256; i += blockDim.x) smap4[i] = static_cast<std::uint8_t>(4u * a.symmap[i]);
    }
    __syncthreads();
    const std::uint32_t tab_s = pinned_reg(smem_u32(smem));
    const std::uint32_t def_s = pinned_reg(tab_s + 4u * ct.slots);
    const std::uint32_t map_s = pinned_reg(tab_s + ct.image_bytes);

    const std::uint32_t K = pinned_reg(a.K), KK = pinned_reg(a.K * a.K), esc4 = 4u * (a.K - 1u);
    const long long halo = a.halo, steps = a.halo + a.chunk, n = a.n;
    std::uint32_t* __restrict__ ev = e.ev;
    const std::uint32_t root = lds_u32(def_s + (D == 3 ? (KK + K + 1u) : (K + 1u)) * esc4);  // T_D[esc, .., esc]
    // a state word as the walk carries it: id / payload and the two flags (the
    // count byte and the entry's column field are dropped before the next address)
    const std::uint32_t amask = ct.pay_mask | kCtCold | kCtOut;
    unsigned long long evs = 0;  // events logged by this thread (sizes the next run's slabs)

    // Rounds: in round r the grid walks the chunks [r, r+1) * gridDim * blockDim * U,
    // neighbouring lanes on neighbouring chunks — the text a warp reads at any
    // time lies within 32 * U chunks (with one long chunk per stream the lanes
    // of a warp sit megabytes apart: every text load touches 32 pages).
    const long long per_round = static_cast<long long>(gridDim.x) * blockDim.x * U;
    for (long long cid0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * U; cid0 < a.n_chunks;
         cid0 += per_round) {
    long long cid[U];
    bool act[U];
    std::uint32_t live[U];  // kCtOut while the stream may log, else 0 (the log predicate is one AND)
#pragma unroll
    for (int u = 0; u < U; ++u) {
        cid[u] = cid0 + u;
        act[u] = cid[u] < a.n_chunks;
        live[u] = act[u] ? kCtOut : 0u;
    }

    std::uint32_t st[U], wr[U], lim[U], cnt[U], p1[U], p2[U];  // p1/p2: 4 * the previous two columns
    std::uint32_t xp[U];                                        // DEEP: the previous step's T_D default
    std::uint32_t recs[U];                                      // records of the chunk (counted words: byte 2)
    long long pos0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        st[u] = root & amask;
        xp[u] = root & amask;
        cnt[u] = 0;
        recs[u] = 0;
        p1[u] = p2[u] = esc4;
        wr[u] = act[u] ? slab_start(e, cid[u]) : 0u;
        lim[u] = act[u] ? slab_end(e, cid[u]) - 1u : 0u;
        pos0[u] = a.emit_from + cid[u] * a.chunk - halo;
    }
    uint4 w[U];
    auto load = [&](long long off) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = pos0[u] + off;
            w[u] = (act[u] && p >= 0 && p < n) ? ld_stream16(a.text + p) : make_uint4(0, 0, 0, 0);
        }
    };
    // the text-only default of a step: x = T_D[the step's last D columns]
    auto default_of = [&](std::uint32_t q2, std::uint32_t q1, std::uint32_t c4) -> std::uint32_t {
        const std::uint32_t r2 = q1 * K + (c4 + def_s);
        return lds_u32(D == 3 ? q2 * KK + r2 : r2);
    };
    load(0);
    for (long long off = 0; off < steps; off += 16) {
        uint4 cur[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cur[u] = w[u];
        if (off + 16 < steps) load(off + 16);
        const bool owned_blk = off >= halo;
        std::uint32_t wr0[U];
        if (owned_blk) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (live[u] && lim[u] - wr[u] < 16u) {  // close the region, continue in a pool block
                    for (; wr[u] < lim[u]; ++wr[u], ++cnt[u]) ev[wr[u]] = kEvPad;
                    const uint2 g = ev_grow(ev, e.pool_used, e.pool_base, e.pool_blocks, lim[u]);
                    wr[u] = g.x;
                    lim[u] = g.y;
                    if (g.y == 0u) live[u] = 0u;
                }
                wr0[u] = wr[u];
            }
        }
        bool fast = true;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = pos0[u] + off;
            fast = fast && (!act[u] || (p >= 0 && p + 16 <= n));
        }
        std::uint32_t kk = owned_blk ? static_cast<std::uint32_t>(off - halo) << e.ob : 0u;
        const std::uint32_t kinc = 1u << e.ob;
        // One group of GL steps of all U streams. The columns of the whole group
        // are looked up first (independent loads); each step's default is loaded
        // one step ahead of its use; the state's own chain per step is the
        // address multiply-add, the entry load, XOR, test, select.
        auto group = [&](auto log_tag, auto fast_tag, const int k0) {
            constexpr bool LOG = decltype(log_tag)::value;
            constexpr bool FAST = decltype(fast_tag)::value;
            std::uint32_t c4[U][GL];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int j = 0; j < GL; ++j) {
                    const int k = k0 + j;
                    const std::uint32_t word = k < 4 ? cur[u].x : k < 8 ? cur[u].y : k < 12 ? cur[u].z : cur[u].w;
                    std::uint32_t c = lds_u8z(map_s + __byte_perm(word, 0u, 0x4440u + (k & 3)));
                    if (!FAST) {  // a position outside the text reads as a byte outside the alphabet (root)
                        const long long p = pos0[u] + off + k;
                        if (!act[u] || p < 0 || p >= n) c = esc4;
                    }
                    c4[u][j] = c;
                }
            // xn = T_D default of the next step, en (DEEP) = the entry of the previous
            // default's row for the next step's column: both loaded one step ahead
            std::uint32_t xn[U], en[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                xn[u] = default_of(p2[u], p1[u], c4[u][0]);
                if (DEEP) en[u] = lds_u32(xp[u] * 4u + (c4[u][0] + tab_s));  // (xp is masked: no count byte)
            }
#pragma unroll
            for (int j = 0; j < GL; ++j) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const std::uint32_t c = c4[u][j];
                    std::uint32_t x = xn[u];  // (full word: its count byte is read when the step logs)
                    if (DEEP) {  // one more level: the depth-(D+1) child of the previous default, if the text spells it
                        const std::uint32_t d2 = en[u] ^ (c << (kCtColShift - 2));
                        xp[u] = x & amask;
                        if (!(d2 & kCtColMask)) x = d2;
                    }
                    if (j + 1 < GL) {
                        xn[u] = default_of(j ? c4[u][j - 1] : p1[u], c, c4[u][j + 1]);
                        if (DEEP) en[u] = lds_u32(xp[u] * 4u + (c4[u][j + 1] + tab_s));
                    }
                    const std::uint32_t sw = st[u];
                    std::uint32_t v;
                    std::uint32_t full;  // the next state's full word (count byte included)
                    if (COLD && __builtin_expect((sw & kCtCold) != 0u, 0)) {
                        full = ctab_cold_step(ct.next, K, ct.slots, a.Hn, ct.pay_mask, sw, c);
                        v = full & amask;
                    } else {
                        const std::uint32_t ent = lds_u32(sw * 4u + (c + tab_s));  // (bits 30-31 of sw fall off the multiply)
                        const std::uint32_t cx = c << (kCtColShift - 2);
                        const bool miss = ((ent ^ cx) & kCtColMask) != 0u;
                        if (DEEP) {  // (measured: the one-select form below costs the deep walk 13 %)
                            v = miss ? (x & amask) : ((ent ^ cx) & amask);
                            full = miss ? x : ent;
                        } else {
                            full = miss ? x : (ent ^ cx);  // (the XOR touches the column field only: the count byte stays)
                            v = full & amask;
                        }
                    }
                    st[u] = v;
                    if (LOG) {
                        // branch-free log (the walk is issue-bound: 97 % of the warp-steps have
                        // a logging lane, so a branch costs its overhead on top of its body):
                        // a predicated store, the slot index advanced by the hit bit. The count
                        // byte of a word without outputs is 0 (counted words), so the records
                        // are summed unconditionally.
                        if (DEEP) {
                            const std::uint32_t hit = v & live[u];  // bit 31 or nothing
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.global.u32 [%1], %2;\n\t}"
                                :
                                : "r"(hit), "l"(ev + wr[u]), "r"(kk | (v & ct.pay_mask))
                                : "memory");
                            wr[u] += hit >> 31;
                        } else {
                            asm volatile(
                                "{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.u32 p, t, 0;\n\t"
                                "@p st.global.u32 [%3], %4;\n\t@p add.u32 %0, %0, 1;\n\t}"
                                : "+r"(wr[u])
                                : "r"(v), "r"(live[u]), "l"(ev + wr[u]), "r"(kk | (v & ct.pay_mask))
                                : "memory");
                        }
                        recs[u] += __byte_perm(full, 0u, 0x4442u);
                    }
                }
                if (LOG) kk += kinc;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                p2[u] = c4[u][GL - 2];
                p1[u] = c4[u][GL - 1];
            }
        };
#pragma unroll
        for (int k0 = 0; k0 < 16; k0 += GL) {
            if (fast) {
                if (owned_blk) group(std::true_type{}, std::true_type{}, k0);
                else group(std::false_type{}, std::true_type{}, k0);
            } else {
                if (owned_blk) group(std::true_type{}, std::false_type{}, k0);
                else group(std::false_type{}, std::false_type{}, k0);
            }
        }
        if (owned_blk) {
#pragma unroll
            for (int u = 0; u < U; ++u) cnt[u] += wr[u] - wr0[u];
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (act[u]) {
            e.ev_count[cid[u]] = cnt[u];
            if (ct.counted) a.chunk_counts[cid[u]] = recs[u];  // (else E1 counts them)
            evs += cnt[u];
        }
    }  // rounds
    if (ct.counted) {  // E1 is not run: the run's event total from here
#pragma unroll
        for (int o = 16; o; o >>= 1) evs += __shfl_xor_sync(0xFFFFFFFFu, evs, o);
        if ((threadIdx.x & 31) == 0 && evs) atomicAdd(e.ev_total, evs);
    }
}

// ====================================================== SPARSE-G (generic) ==
// EXACT mode for generic alphabets without L2 lookups in the lockstep walk.
// hotG[s*K + c] (s hot) = the longest suffix of s.c in the hot set H (a BFS
// prefix, closed under "longest hot suffix") | kGCold when the TRUE target is
// cold. Walking hotG from the root gives, at every position, the longest hot
// suffix of the text, which IS the true state whenever the true state is hot.
//  * KG sparseg_walk_kernel: the walk, all in shared memory. Logs, per chunk in
//    position order: an output event for each owned step whose (hot) state has
//    outputs, and an excursion event (walk offset, source state) for each step
//    whose true target is cold (also in the halo: an excursion can run into
//    the owned part).
//  * XG sparseg_fix_kernel: one thread per chunk replays the chunk's events in
//    order: an excursion walks the true DFA (L2) from its source state until
//    the state is hot again, emitting the cold states' outputs; events inside
//    an excursion (proxy outputs, spurious excursions) are dropped; the rest
//    are exact. The result is the chunk's final event list in the format E1/E2
//    take (owned offset << ob | output rank), in slabs of chunk + 1 slots
//    (one event per owned byte at most).
constexpr std::uint32_t kGCold = 0x8000u;

template <int U>
__global__ void __launch_bounds__(U <= 2 ? 2 * kTPB : kTPB, 1) sparseg_walk_kernel(const ScanArgs a, const EventArgs e,
                                                                                   std::uint32_t n_out) {
    extern __shared__ __align__(16) std::uint8_t smem[];
    std::uint8_t* smap = smem + a.smem_table_bytes;
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.hotH);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (std::uint32_t i = threadIdx.x; i < a.smem_table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
        for (std::uint32_t i = threadIdx.x; i < 256; i += blockDim.x) smap[i] = a.symmap[i];
    }
    __syncthreads();
    const std::uint32_t hot_s = smem_u32(smem);
    const long long G = gridDim.x;
    long long cid[U];
    bool act[U], live[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        cid[u] = (static_cast<long long>(threadIdx.x) * U + u) * G + blockIdx.x;
        act[u] = cid[u] < a.n_chunks;
        live[u] = act[u];
    }
    if (!act[0]) return;
    const std::uint32_t K = a.K, Hn = a.Hn, nhot = a.H - a.Hn, ob = e.ob;
    const long long halo = a.halo, steps = a.halo + a.chunk, n = a.n;
    std::uint32_t* __restrict__ ev = e.ev;
    std::uint32_t st[U], wr[U], lim[U], cnt[U];
    long long pos0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        st[u] = 0;
        cnt[u] = 0;
        wr[u] = act[u] ? slab_start(e, cid[u]) : 0u;
        lim[u] = act[u] ? slab_end(e, cid[u]) - 1u : 0u;
        pos0[u] = a.emit_from + cid[u] * a.chunk - halo;
    }
    uint4 w[U];
    auto load = [&](long long off) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = pos0[u] + off;
            w[u] = (act[u] && p >= 0 && p < n) ? ld_stream16(a.text + p) : make_uint4(0, 0, 0, 0);
        }
    };
    const std::uint32_t kinc = 1u << ob;
    load(0);
    for (long long off = 0; off < steps; off += 16) {
        uint4 cur[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cur[u] = w[u];
        if (off + 16 < steps) load(off + 16);
        const bool owned_blk = off >= halo;
        std::uint32_t wr0[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {  // two events per step at most: 32 free slots per block
            if (live[u] && lim[u] - wr[u] < 32u) {
                for (; wr[u] < lim[u]; ++wr[u], ++cnt[u]) ev[wr[u]] = kEvPad;
                const uint2 g = ev_grow(ev, e.pool_used, e.pool_base, e.pool_blocks, lim[u]);
                wr[u] = g.x;
                lim[u] = g.y;
                if (g.y == 0u) live[u] = false;
            }
            wr0[u] = wr[u];
        }
        bool fast = true;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = pos0[u] + off;
            fast = fast && (!act[u] || (p >= 0 && p + 16 <= n));
        }
        std::uint32_t kk = static_cast<std::uint32_t>(off) << ob;
        if (fast) {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const std::uint32_t word = k < 4 ? cur[u].x : k < 8 ? cur[u].y : k < 12 ? cur[u].z : cur[u].w;
                    const std::uint32_t col = smap[__byte_perm(word, 0u, 0x4440u + (k & 3))];
                    const std::uint32_t v = lds_u16z(hot_s + 2u * (st[u] * K + col));
                    const std::uint32_t nx = v & 0x7FFFu, r = nx - Hn;
                    if (live[u] && (v & kGCold)) ev[wr[u]++] = kk + n_out + st[u];
                    if (owned_blk && live[u] && r < nhot) ev[wr[u]++] = kk + r;
                    st[u] = nx;
                }
                kk += kinc;
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!act[u]) continue;
                std::uint32_t kq = kk;
#pragma unroll 1
                for (int k = 0; k < 16; ++k, kq += kinc) {
                    const long long p = pos0[u] + off + k;
                    const std::uint32_t word = k < 4 ? cur[u].x : k < 8 ? cur[u].y : k < 12 ? cur[u].z : cur[u].w;
                    const int c = (p >= 0 && p < n) ? column_of<1>((word >> (8 * (k & 3))) & 0xFFu, smap, a) : -1;
                    std::uint32_t nx = 0;
                    if (c >= 0) {
                        const std::uint32_t v = lds_u16z(hot_s + 2u * (st[u] * K + static_cast<std::uint32_t>(c)));
                        nx = v & 0x7FFFu;
                        if (live[u] && (v & kGCold)) ev[wr[u]++] = kq + n_out + st[u];
                    }
                    const std::uint32_t r = nx - Hn;
                    if (owned_blk && live[u] && r < nhot) ev[wr[u]++] = kq + r;
                    st[u] = nx;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) cnt[u] += wr[u] - wr0[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (act[u]) e.ev_count[cid[u]] = cnt[u];
}

// XG: ew = the walk's events (walk offsets, payload < n_out: hot output rank;
// >= n_out: excursion from hot state payload - n_out); ef = the final events.
__global__ void __launch_bounds__(256) sparseg_fix_kernel(const ScanArgs a, const EventArgs ew, const EventArgs ef,
                                                          std::uint32_t n_out) {
    if (!ev_pool_ok(ew)) return;  // the walk's pool overflowed: the host replays the run
    const std::uint32_t K = a.K, H = a.H, Hn = a.Hn, wob = ew.ob, fob = ef.ob;
    const std::uint32_t wmask = (1u << wob) - 1u;
    const long long halo = a.halo, steps = a.halo + a.chunk, n = a.n;
    unsigned long long seen = 0;
    for (long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; c < a.n_chunks;
         c += static_cast<long long>(gridDim.x) * blockDim.x) {
        const std::uint32_t total = ew.ev_count[c];
        seen += total;
        const long long pos0 = a.emit_from + c * a.chunk - halo;
        std::uint32_t p = slab_start(ew, c), lim = slab_end(ew, c) - 1u;
        std::uint32_t out = static_cast<std::uint32_t>(c) * ef.ecap, o0 = out;
        long long p_end = 0;  // walk offsets below this lie inside a replayed excursion
        for (std::uint32_t i = 0; i < total; ++i) {
            if (p == lim) {
                p = ew.ev[lim];
                lim = p + kEvBlock - 1;
            }
            const std::uint32_t v = __ldcs(ew.ev + p++);
            if (v == kEvPad) continue;
            const long long off = v >> wob;
            if (off < p_end) continue;
            const std::uint32_t pay = v & wmask;
            if (pay < n_out) {  // a hot output state (exact: not inside an excursion)
                ef.ev[out++] = (static_cast<std::uint32_t>(off - halo) << fob) | pay;
                continue;
            }
            // excursion: the true DFA from the hot source state until the state is hot again
            std::uint32_t x = pay - n_out;
            long long o = off;
            for (;;) {
                const long long tp = pos0 + o;
                const int col = (tp >= 0 && tp < n) ? column_of<1>(__ldg(a.text + tp), nullptr, a) : -1;
                x = col < 0 ? 0u : __ldg(a.next + x * K + static_cast<std::uint32_t>(col));
                if (x < H) break;  // hot again at o: the walk's events from o on are exact
                if (o >= halo && x - Hn < a.Cn - Hn)
                    ef.ev[out++] = (static_cast<std::uint32_t>(o - halo) << fob) | (x - Hn);
                if (++o >= steps) break;
            }
            p_end = o;
        }
        ef.ev_count[c] = out - o0;
    }
    if (seen) atomicAdd(ew.ev_total, seen);  // the walk's events (size its next run's slabs)
}

// Per-chunk slab sizes for the next run from this run's event counts:
// sizes[c] = cnt + cnt/8 + 17 (incl. the link slot); offs[0] = 0 (CUB prefixes
// sizes into offs[1..]).
__global__ void __launch_bounds__(256) event_slab_sizes_kernel(const std::uint32_t* cnt, long long n,
                                                               std::uint32_t* sizes, std::uint32_t* offs) {
    for (long long c = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x; c < n;
         c += static_cast<long long>(gridDim.x) * 256) {
        const std::uint32_t k = cnt[c];
        sizes[c] = k + (k >> 3) + 17;
        if (c == 0) offs[0] = 0;
    }
}

// Walks chunk c's event regions (primary slab, then linked pool blocks) in
// warp-wide batches of up to 32 events: f(base_index, n_in_batch, event of
// this lane or 0, lane valid, the event's slot).
template <typename F>
__device__ __forceinline__ void for_event_batches(const EventArgs& e, long long c, std::uint32_t total, int lane, F f) {
    std::uint32_t p = slab_start(e, c), lim = slab_end(e, c) - 1u, done = 0;
    while (done < total) {
        const std::uint32_t here = min(total - done, lim - p);
        // four batches' loads in flight per warp (one load per batch left each warp
        // waiting a full memory round trip per 32 events: E1/E2 were latency-bound)
        for (std::uint32_t b = 0; b < here; b += 128) {
            std::uint32_t v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const std::uint32_t i = b + 32u * k + lane;
                v[k] = i < here ? __ldcs(e.ev + p + i) : 0u;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const std::uint32_t b0 = b + 32u * k;
                if (b0 >= here) break;
                const std::uint32_t nb = min(32u, here - b0);
                f(done + b0, nb, v[k], static_cast<std::uint32_t>(lane) < nb, p + b0 + lane);
            }
        }
        done += here;
        if (done < total) {
            p = e.ev[lim];
            lim = p + kEvBlock - 1;
        }
    }
}

// Output count of state s from its packed output info (automaton.hpp).
__device__ __forceinline__ std::uint32_t n_out_of(std::uint32_t s, unsigned long long info, const ScanArgs& a) {
    const std::uint32_t n = static_cast<std::uint32_t>(info >> 32) & 0xFFu;
    return n == 255u ? __ldg(a.out_off + s + 1) - static_cast<std::uint32_t>(info) : n;
}

// ===================================================================== E1 ==
// One warp per chunk: records per chunk (-> chunk_counts, u64 for the CUB
// prefix) and visits per output rank (shared-memory bins when they fit).
// (SMEM_NOUT: each output state's output count, as a byte (255 = look it up),
// staged after the bins: the events' record counts need no L2 lookups)
// (XL: the walk was KC — event payloads are state-word values (ctab.hpp); they
// are mapped to output ranks through the id -> rank table, staged in shared
// memory when xl_smem)
template <bool SMEM_BINS, bool SMEM_NOUT, bool XL>
__global__ void __launch_bounds__(512) event_count_kernel(const ScanArgs a, const EventArgs e, const CtabArgs ct,
                                                          const bool xl_smem) {
    extern __shared__ std::uint32_t bins[];
    std::uint8_t* nout8 = reinterpret_cast<std::uint8_t*>(bins + (SMEM_BINS ? e.n_out : 0u));
    const std::uint16_t* xrank = ct.rank;
    if (SMEM_BINS)
        for (std::uint32_t i = threadIdx.x; i < e.n_out; i += blockDim.x) bins[i] = 0;
    if (SMEM_NOUT)
        for (std::uint32_t i = threadIdx.x; i < e.n_out; i += blockDim.x)
            nout8[i] = static_cast<std::uint8_t>(__ldg(a.outinfo + a.Hn + i) >> 32);
    if (XL && xl_smem) {
        std::uint16_t* xs = reinterpret_cast<std::uint16_t*>(nout8 + (SMEM_NOUT ? ((e.n_out + 15u) & ~15u) : 0u));
        for (std::uint32_t i = threadIdx.x; i < ct.slots; i += blockDim.x) xs[i] = __ldg(ct.rank + i);
        xrank = xs;
    }
    if (SMEM_BINS || SMEM_NOUT || XL) __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long wpb = blockDim.x >> 5;
    const long long warps = static_cast<long long>(gridDim.x) * wpb;
    const std::uint32_t rmask = (1u << e.ob) - 1u, H = a.H, Hn = a.Hn, Cn = a.Cn;
    const bool visits = a.visits != nullptr;
    const bool pool_ok = ev_pool_ok(e);
    unsigned long long evs = 0;
    for (long long c = static_cast<long long>(blockIdx.x) * wpb + (threadIdx.x >> 5); c < a.n_chunks; c += warps) {
        const std::uint32_t total = pool_ok ? e.ev_count[c] : 0u;
        evs += total;
        unsigned long long recs = 0;
        if (total) {
            for_event_batches(e, c, total, lane, [&](std::uint32_t, std::uint32_t, std::uint32_t v, bool ok, std::uint32_t slot) {
                if (!ok || v == kEvPad) return;
                std::uint32_t r = v & rmask;
                if (XL) r = r < ct.slots ? (xl_smem ? xrank[r] : __ldg(ct.rank + r)) : r - ct.slots;
                (void)slot;
                const std::uint32_t s = state_of_rank(r, H, Hn, Cn);
                std::uint32_t no = SMEM_NOUT ? nout8[r] : 255u;
                if (no == 255u) no = n_out_of(s, __ldg(a.outinfo + s), a);
                recs += no;
                if (visits) {
                    if (SMEM_BINS) atomicAdd(&bins[r], 1u);
                    else atomicAdd(a.visits + r, 1ull);
                }
            });
#pragma unroll
            for (int o = 16; o; o >>= 1) recs += __shfl_xor_sync(0xFFFFFFFFu, recs, o);
        }
        if (lane == 0) a.chunk_counts[c] = recs;
    }
    if (lane == 0 && evs) atomicAdd(e.ev_total, evs);
    if (SMEM_BINS && visits) {
        __syncthreads();
        for (std::uint32_t i = threadIdx.x; i < e.n_out; i += blockDim.x)
            if (bins[i]) atomicAdd(a.visits + i, static_cast<unsigned long long>(bins[i]));
    }
}

// ===================================================================== E2 ==
// One warp per chunk with records: the events' records at the chunk's slot
// range, written by consecutive lanes (coalesced).
// (XL: KC's payloads index a payload -> output-info table directly)
// (VIS: also the per-output-state visit histogram, in shared-memory bins —
// when KC counted the records itself and E1 is not run)
template <bool XL, bool VIS>
__global__ void __launch_bounds__(256, VIS ? 5 : 4) event_expand_kernel(const ScanArgs a, const EventArgs e, const CtabArgs ct) {
    extern __shared__ std::uint32_t vbins[];
    if (VIS) {
        for (std::uint32_t i = threadIdx.x; i < e.n_out; i += blockDim.x) vbins[i] = 0;
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const long long wpb = blockDim.x >> 5;
    const long long warps = static_cast<long long>(gridDim.x) * wpb;
    const std::uint32_t rmask = (1u << e.ob) - 1u, H = a.H, Hn = a.Hn, Cn = a.Cn;
    if (!ev_pool_ok(e)) return;  // (block-uniform)
    for (long long c = static_cast<long long>(blockIdx.x) * wpb + (threadIdx.x >> 5); c < a.n_chunks; c += warps) {
        const std::uint32_t total = e.ev_count[c];
        if (!total) continue;
        unsigned long long o = a.chunk_offs[c];
        const unsigned long long cbase = a.base + static_cast<unsigned long long>(a.emit_from + c * a.chunk);
        for_event_batches(e, c, total, lane, [&](std::uint32_t, std::uint32_t nb, std::uint32_t v, bool ok, std::uint32_t) {
            std::uint32_t n = 0, lo = 0, first = 0;
            unsigned long long key = 0;
            if (ok && v != kEvPad) {
                const std::uint32_t pay = v & rmask;
#if !defined(ACG_E2_RANK)  // payload-indexed info table: one load (measured on cfg3: E2 1.48 ms against 1.63 through the rank table)
                const unsigned long long info = XL ? __ldg(ct.info + pay) : __ldg(a.outinfo + state_of_rank(pay, H, Hn, Cn));
                lo = static_cast<std::uint32_t>(info);
                n = static_cast<std::uint32_t>(info >> 32) & 0xFFu;
                if (n == 255u || VIS) {
                    const std::uint32_t r = XL ? (pay < ct.slots ? __ldg(ct.rank + pay) : pay - ct.slots) : pay;
                    if (n == 255u) n = n_out_of(state_of_rank(r, H, Hn, Cn), info, a);  // a long list: its length from the CSR offsets
                    if (VIS) atomicAdd(&vbins[r], 1u);
                }
#else
                // KC payload -> output rank (id -> rank table, L1-resident), then the rank-ordered info
                const std::uint32_t r = XL ? (pay < ct.slots ? __ldg(ct.rank + pay) : pay - ct.slots) : pay;
                const std::uint32_t s = state_of_rank(r, H, Hn, Cn);
                const unsigned long long info = __ldg(a.outinfo + s);
                lo = static_cast<std::uint32_t>(info);
                n = n_out_of(s, info, a);
                if (VIS) atomicAdd(&vbins[r], 1u);
#endif
                first = static_cast<std::uint32_t>(info >> 40);
                if (!(first || a.id_bits <= 24)) first = __ldg(a.out_ids + lo);
                key = (cbase + (v >> e.ob)) << a.id_bits;
            }
            const unsigned single = __ballot_sync(0xFFFFFFFFu, n == 1u || !ok);
            if (single == 0xFFFFFFFFu) {  // every event has one output: record = lane
                if (ok && o + lane < a.rec_cap) a.records[o + lane] = key | first;
                o += nb;
                return;
            }
            // short output lists (cfg3: one to three ids per state): the prefix of the
            // counts from four ballots (no shuffle chain); every lane writes its own event's
            // records at its prefix — neighbouring lanes, neighbouring slots — in max(n)
            // rounds; longer lists (cfg4) take the scan and the balanced assignment below
            if (__ballot_sync(0xFFFFFFFFu, n > 4u) == 0u) {
                const std::uint32_t m1 = __ballot_sync(0xFFFFFFFFu, n >= 1u), m2 = __ballot_sync(0xFFFFFFFFu, n >= 2u);
                const std::uint32_t m3 = __ballot_sync(0xFFFFFFFFu, n >= 3u), m4 = __ballot_sync(0xFFFFFFFFu, n >= 4u);
                const std::uint32_t lt = (1u << lane) - 1u;
                const std::uint32_t excl = __popc(m1 & lt) + __popc(m2 & lt) + __popc(m3 & lt) + __popc(m4 & lt);
                const std::uint32_t nmax = m4 ? 4u : m3 ? 3u : m2 ? 2u : 1u;
                const unsigned long long at = o + excl;
                for (std::uint32_t k = 0; k < nmax; ++k) {
                    if (k < n) {
                        const std::uint32_t id = k == 0 ? first : __ldg(a.out_ids + lo + k);
                        if (at + k < a.rec_cap) a.records[at + k] = key | id;
                    }
                }
                o += __popc(m1) + __popc(m2) + __popc(m3) + __popc(m4);
                return;
            }
            // inclusive scan of the output counts
            std::uint32_t incl = n;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const std::uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (lane >= d) incl += y;
            }
            const std::uint32_t T = __shfl_sync(0xFFFFFFFFu, incl, 31);
            // Events with outputs in the lanes [0, popc): the j-th of them is lane j, so the
            // owner of output t is (events whose first output lies at or before t) - 1 — one
            // warp OR of the window's start bits and a population count instead of the
            // binary search (cfg4: every event has outputs; pads and a ragged last batch
            // leave the top lanes empty, anything else takes the search below).
            const std::uint32_t nz = __ballot_sync(0xFFFFFFFFu, n != 0u);
            if ((nz & (nz + 1u)) == 0u) {
                const std::uint32_t excl = incl - n, voff = v >> e.ob;
                const std::uint32_t le = 0xFFFFFFFFu >> (31 - lane);
                std::uint32_t jbase = 0;
                // two windows of 32 outputs per iteration: two independent vote / shuffle /
                // gather chains in flight
                for (std::uint32_t t0 = 0; t0 < T; t0 += 64) {
                    const std::uint32_t rel0 = excl - t0, rel1 = rel0 - 32u;
                    const std::uint32_t s0 = __reduce_or_sync(0xFFFFFFFFu, (n != 0u && rel0 < 32u) ? 1u << rel0 : 0u);
                    const std::uint32_t s1 = __reduce_or_sync(0xFFFFFFFFu, (n != 0u && rel1 < 32u) ? 1u << rel1 : 0u);
                    const int j0 = static_cast<int>(jbase + __popc(s0 & le)) - 1;
                    jbase += __popc(s0);
                    const int j1 = static_cast<int>(jbase + __popc(s1 & le)) - 1;
                    jbase += __popc(s1);
                    const std::uint32_t e0 = __shfl_sync(0xFFFFFFFFu, excl, j0), e1 = __shfl_sync(0xFFFFFFFFu, excl, j1);
                    const std::uint32_t l0 = __shfl_sync(0xFFFFFFFFu, lo, j0), l1 = __shfl_sync(0xFFFFFFFFu, lo, j1);
                    const std::uint32_t v0 = __shfl_sync(0xFFFFFFFFu, voff, j0), v1 = __shfl_sync(0xFFFFFFFFu, voff, j1);
                    const std::uint32_t ta = t0 + lane, tb = ta + 32u;
                    const bool wa = ta < T && o + ta < a.rec_cap, wb = tb < T && o + tb < a.rec_cap;
                    const std::uint32_t ia = wa ? __ldg(a.out_ids + l0 + (ta - e0)) : 0u;
                    const std::uint32_t ib = wb ? __ldg(a.out_ids + l1 + (tb - e1)) : 0u;
                    if (wa) a.records[o + ta] = ((cbase + v0) << a.id_bits) | ia;
                    if (wb) a.records[o + tb] = ((cbase + v1) << a.id_bits) | ib;
                }
                o += T;
                return;
            }
            for (std::uint32_t t0 = 0; t0 < T; t0 += 32) {
                const std::uint32_t t = t0 + lane;
                // owner j = the first lane with incl_j > t (binary search over the scan)
                int j = 0;
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const std::uint32_t iv = __shfl_sync(0xFFFFFFFFu, incl, j + step - 1);
                    if (iv <= t) j += step;
                }
                const std::uint32_t ij = __shfl_sync(0xFFFFFFFFu, incl, j);
                const std::uint32_t nj = __shfl_sync(0xFFFFFFFFu, n, j);
                const std::uint32_t loj = __shfl_sync(0xFFFFFFFFu, lo, j);
                const std::uint32_t fj = __shfl_sync(0xFFFFFFFFu, first, j);
                const unsigned long long kj = __shfl_sync(0xFFFFFFFFu, key, j);
                if (t < T) {
                    const std::uint32_t k = t - (ij - nj);
                    const std::uint32_t id = k == 0 ? fj : __ldg(a.out_ids + loj + k);
                    if (o + t < a.rec_cap) a.records[o + t] = kj | id;
                }
            }
            o += T;
        });
    }
    if (VIS) {
        __syncthreads();
        for (std::uint32_t i = threadIdx.x; i < e.n_out; i += blockDim.x)
            if (vbins[i]) atomicAdd(a.visits + i, static_cast<unsigned long long>(vbins[i]));
    }
}

}  // namespace kern
}  // namespace acg
