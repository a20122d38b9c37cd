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
// non-output, [Cn,S) cold output; rows [0,H) are "hot" (shared memory).
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

namespace acg {
namespace kern {

enum Pass : int { kCount = 0, kWrite = 1 };
constexpr int kTPB = 512;  // threads per block of the scan kernels
constexpr std::uint32_t kEsc16 = 0xFFFFu;

struct ScanArgs {
    const std::uint8_t* text;  // 16-byte aligned; byte i of this buffer = global byte base+i
    long long n;               // bytes in the buffer
    long long emit_from;       // first owned byte (multiple of 16)
    unsigned long long base;   // global offset of text[0] (added to record ends)
    long long chunk;           // owned bytes per chunk (multiple of 16)
    int halo;                  // warm-up bytes (multiple of 16)
    long long n_chunks;
    // DFA
    const std::uint32_t* next;     // S*K exact transitions (device ids)
    const std::uint16_t* hot16;    // (H+1)*K exact hot rows; 0xFFFF = consult `next`; row H = all 0xFFFF
    const std::uint16_t* hotH;     // H*K truncated-automaton rows: id | 0x8000 attention
    const std::uint32_t* out_off;  // S+1
    const std::uint32_t* out_ids;
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
    // sparse-mode event log: per chunk `ev_cap` 16-byte events (see K1s)
    std::uint32_t* events;
    std::uint32_t* ev_count;                // per chunk (may exceed ev_cap: overflow)
    std::uint32_t ev_cap;
    unsigned long long* ev_total;           // sum of events (mode heuristic)
};

__device__ __forceinline__ uint4 ld_stream16(const std::uint8_t* p) {
    uint4 v;
    asm volatile("ld.global.nc.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ std::uint32_t lds_u16(std::uint32_t saddr) {
    std::uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(saddr));
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
    return s < a.H ? s - a.Hn : (a.H - a.Hn) + (s - a.Cn);
}

__device__ __forceinline__ bool has_out(std::uint32_t s, const ScanArgs& a) {
    return (s >= a.Hn && s < a.H) || s >= a.Cn;
}

// Column of byte b (-1 = escape: every state goes to the root).
template <int MODE>
__device__ __forceinline__ int column_of(std::uint32_t b, const std::uint8_t* smap, const ScanArgs& a) {
    if (MODE == 0) return (b == 'A' || b == 'C' || b == 'G' || b == 'T') ? static_cast<int>((b >> 1) & 3u) : -1;
    const std::uint32_t c = smap ? smap[b] : a.symmap[b];
    return c == a.K - 1 ? -1 : static_cast<int>(c);
}

// Output handling at owned buffer position `pos` for state s (has outputs).
template <int PASS>
__device__ __forceinline__ void emit(std::uint32_t s, long long pos, unsigned long long& cnt, unsigned long long& wr,
                                     const ScanArgs& a) {
    const std::uint32_t lo = __ldg(a.out_off + s), hi = __ldg(a.out_off + s + 1);
    // per-state visits are recorded by whichever pass the host enables them for
    if (a.visits) atomicAdd(a.visits + out_rank(s, a), 1ull);
    if (PASS == kCount) {
        cnt += hi - lo;
    } else {
        const unsigned long long endk = (a.base + static_cast<unsigned long long>(pos)) << a.id_bits;
        for (std::uint32_t j = lo; j < hi; ++j) {
            if (wr < a.rec_cap) a.records[wr] = endk | __ldg(a.out_ids + j);
            ++wr;
        }
    }
}

// ===================================================================== K1x ==
// Exact lockstep walk. One step of U streams: U shared loads issued together
// (cold source rows clamp to the all-escape row H), then U L2 loads for the
// escapes, so a warp waits for at most one L2 latency per step.
template <int U, int MODE, int PASS, bool STATS>
__global__ void __launch_bounds__(kTPB, 1) exact_scan_kernel(const ScanArgs a) {
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
    unsigned long long cnt[U], wr[U], fol[U];
    long long pos0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        st[u] = 0;
        cnt[u] = 0;
        fol[u] = 0;
        wr[u] = (PASS == kWrite && act[u]) ? a.chunk_offs[chunk_id[u]] : 0ull;
        pos0[u] = a.emit_from + chunk_id[u] * a.chunk - a.halo;
    }
    const std::uint32_t K = a.K, H = a.H, Hn = a.Hn;
    const long long steps = a.halo + a.chunk;

    uint4 w[U];
    auto load = [&](long long off) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = pos0[u] + off;
            w[u] = (act[u] && p >= 0 && p + 16 <= a.n) ? ld_stream16(a.text + p) : make_uint4(0, 0, 0, 0);
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
#pragma unroll
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
                        emit<PASS>(st[u], pos0[u] + off + k, cnt[u], wr[u], a);
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
                    const int c = inside ? column_of<MODE>(a.text[p], smap, a) : -1;
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
                    if (owned_blk && nx >= Hn && has_out(nx, a)) emit<PASS>(nx, p, cnt[u], wr[u], a);
                }
            }
        }
    }
    if (PASS == kCount) {
        unsigned long long f = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!act[u]) continue;
            a.chunk_counts[chunk_id[u]] = cnt[u];
            f += fol[u];
        }
        if (STATS && a.follows_total && f) atomicAdd(a.follows_total, f);
    }
}

// ===================================================================== K1s ==
// Truncated-automaton fast pass (dna4 alphabet). Per step and stream: one
// shared u16 load and an OR into the sub-block flag accumulator. Text is read
// in 16*RB-byte refills per stream (RB 16-byte vector loads of one span,
// prefetched one refill ahead), so every DRAM sector is consumed whole.
// Every flagged 4-step sub-block logs one 8-byte event:
//   w0 = walk offset of the sub-block << 15 | A_H state at its start
//   w1 = the block's 16 packed 2-bit symbols (0xFFFFFFFF: escapes/edges)
template <int U, int RB, int TPB>  // RB = 16-byte blocks per refill (64-byte refills at RB=4)
__global__ void __launch_bounds__(TPB, 1) sparse_scan_kernel(const ScanArgs a) {
    extern __shared__ __align__(16) std::uint8_t smem[];
    const std::uint32_t tab = smem_u32(smem);
    const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (static_cast<long long>(blockIdx.x) * blockDim.x * U >= a.n_chunks) return;
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.hotH);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (std::uint32_t i = threadIdx.x; i < a.smem_table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const long long c0 = tid * U;  // streams walk chunks c0 .. c0+U-1
    if (c0 >= a.n_chunks) return;
    const int n_act = static_cast<int>(min(static_cast<long long>(U), a.n_chunks - c0));
    const long long p0 = a.emit_from + c0 * a.chunk - a.halo;  // stream u starts at p0 + u*chunk
    const std::uint32_t cap = a.ev_cap;
    uint2* evbase = reinterpret_cast<uint2*>(a.events) + static_cast<unsigned long long>(c0) * cap;

    std::uint32_t st[U], nev[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        st[u] = 0;
        nev[u] = 0;
    }
    const long long steps = a.halo + a.chunk;

    uint4 w[U][RB];
    auto load = [&](long long off) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int b = 0; b < RB; ++b) {
                const long long p = p0 + u * a.chunk + off + 16 * b;
                if (u < n_act && p >= 0 && p + 16 <= a.n && off + 16 * b < steps) {
                    asm volatile("ld.global.nc.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(w[u][b].x), "=r"(w[u][b].y), "=r"(w[u][b].z), "=r"(w[u][b].w)
                                 : "l"(a.text + p));
                } else {
                    w[u][b] = make_uint4(0, 0, 0, 0);
                }
            }
        }
    };
    load(0);
    for (long long off64 = 0; off64 < steps; off64 += 16 * RB) {
        std::uint32_t pk[U][RB];
        std::uint32_t fastm = (1u << RB) - 1;  // per block: every active stream in range and valid
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int b = 0; b < RB; ++b) {
                const long long p = p0 + u * a.chunk + off64 + 16 * b;
                std::uint32_t bad = 0;
                pk[u][b] = dna4_pack(w[u][b], bad);
                if (u < n_act && !(p >= 0 && p + 16 <= a.n && bad == 0)) fastm &= ~(1u << b);
            }
        }
        if (off64 + 16 * RB < steps) load(off64 + 16 * RB);
        const int nblk = static_cast<int>(min(static_cast<long long>(RB), (steps - off64) >> 4));
#pragma unroll
        for (int b = 0; b < RB; ++b) {
            if (b >= nblk) break;
            const long long off = off64 + 16 * b;
            std::uint32_t pkb[U];
            const std::uint32_t offw = static_cast<std::uint32_t>(off);
            if ((fastm >> b) & 1u) {
#pragma unroll
                for (int u = 0; u < U; ++u) pkb[u] = pk[u][b];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    std::uint32_t acc[U], ss[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        ss[u] = st[u];
                        acc[u] = 0;
                    }
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const int k = 4 * j + kk;
                        std::uint32_t v[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const std::uint32_t c2 = k ? (pkb[u] >> (2 * k - 1)) & 6u : (pkb[u] << 1) & 6u;
                            v[u] = lds_u16(tab + (st[u] << 3) + c2);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            acc[u] |= v[u];
                            st[u] = v[u] & 0x7FFFu;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (acc[u] & 0x8000u) {
                            if (nev[u] < cap)
                                evbase[static_cast<unsigned long long>(u) * cap + nev[u]] =
                                    make_uint2(((offw + 4u * j) << 15) | ss[u], pkb[u]);
                            ++nev[u];
                        }
                    }
                }
            } else {
                // block with escapes or text edges: per byte; escapes reset to the
                // root (exact in both automata: the root is hot and has no outputs)
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (u >= n_act) continue;
                    const long long pb = p0 + u * a.chunk + off;
                    std::uint32_t ss = st[u], acc = 0;
#pragma unroll 1
                    for (int k = 0; k < 16; ++k) {
                        if ((k & 3) == 0) {
                            ss = st[u];
                            acc = 0;
                        }
                        const long long p = pb + k;
                        const std::uint32_t bb = (p >= 0 && p < a.n) ? a.text[p] : 0u;
                        if (bb == 'A' || bb == 'C' || bb == 'G' || bb == 'T') {
                            const std::uint32_t v = lds_u16(tab + (st[u] << 3) + (((bb >> 1) & 3u) << 1));
                            acc |= v;
                            st[u] = v & 0x7FFFu;
                        } else {
                            st[u] = 0;
                        }
                        if ((k & 3) == 3 && (acc & 0x8000u)) {
                            if (nev[u] < cap)
                                evbase[static_cast<unsigned long long>(u) * cap + nev[u]] =
                                    make_uint2(((offw + static_cast<std::uint32_t>(k - 3)) << 15) | ss, 0xFFFFFFFFu);
                            ++nev[u];
                        }
                    }
                }
            }
        }
    }
    unsigned long long tot = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (u >= n_act) continue;
        a.ev_count[c0 + u] = nev[u];
        tot += nev[u];
    }
    if (a.ev_total && tot) atomicAdd(a.ev_total, tot);
}

// ===================================================================== K1f ==
// Event replay, one warp per chunk, lanes over the chunk's flagged
// sub-blocks. Every flagged step is walked INDEPENDENTLY: re-walk A_H over
// the 4-step sub-block from its recorded start state (reproducing the fast
// pass's states exactly), and from every flagged transition (s, c) walk the
// full DFA until the state is hot again, collecting candidate outputs
// (offset, state).
//
// Exactness without ordering: a flagged transition taken from a PROXY state
// (inside a true cold excursion) starts a walk whose state is, at every
// offset, a node-suffix of the text - a suffix of the true state - so its
// outputs are a subset of the true outputs there, and it only reaches offsets
// the true excursion covers (while its state is cold, the true state is at
// least as deep). Every true excursion starts with an exact flagged
// transition. Hence out(deepest candidate at each offset) is exactly the true
// output set: per chunk, keep for each offset the deepest candidate.
// Candidates are rare in sparse mode; a lane holding more than kCand falls
// back to an exact walk of the chunk.
constexpr int kCand = 4;

struct Cands {
    std::uint32_t off[kCand];
    std::uint32_t st[kCand];
    int n;  // may exceed kCand (overflow)
};

__device__ __forceinline__ void walk_event(const uint2 e, long long pos0, long long steps, std::uint32_t tab,
                                           Cands& cd, const ScanArgs& a) {
    const long long sb = e.x >> 15;
    const std::uint32_t pk = e.y;
    const bool pk_ok = pk != 0xFFFFFFFFu;
    const std::uint32_t H = a.H;
    auto col_at = [&](long long o) -> int {
        if (pk_ok && (o >> 4) == (sb >> 4)) return static_cast<int>((pk >> (2 * (o & 15))) & 3u);
        const long long p = pos0 + o;
        const std::uint32_t b = (p >= 0 && p < a.n) ? a.text[p] : 0u;
        return column_of<0>(b, nullptr, a);
    };
    std::uint32_t s = e.x & 0x7FFFu;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        const long long i = sb + kk;
        const int col = col_at(i);
        if (col < 0) {
            s = 0;
            continue;
        }
        const std::uint32_t v = lds_u16(tab + (s << 3) + (static_cast<std::uint32_t>(col) << 1));
        if (v & 0x8000u) {
            // independent walk of the full DFA from (s, col) at offset i
            std::uint32_t x = __ldg(a.next + s * 4u + static_cast<std::uint32_t>(col));
            long long k = i;
            for (;;) {
                if (k >= a.halo && has_out(x, a)) {
                    if (cd.n < kCand) {
                        cd.off[cd.n] = static_cast<std::uint32_t>(k);
                        cd.st[cd.n] = x;
                    }
                    ++cd.n;
                }
                if (x < H || k + 1 >= steps) break;
                ++k;
                const int cc = col_at(k);
                x = cc < 0 ? 0u : __ldg(a.next + x * 4u + static_cast<std::uint32_t>(cc));
            }
        }
        s = v & 0x7FFFu;
    }
}

// Exact walk of a whole chunk window by one lane (event-log or candidate overflow).
template <int PASS>
__device__ __noinline__ void exact_chunk_walk(long long c, const ScanArgs& a) {
    const long long pos0 = a.emit_from + c * a.chunk - a.halo;
    const long long steps = a.halo + a.chunk;
    unsigned long long cnt = 0, wr = PASS == kWrite ? a.chunk_offs[c] : 0ull;
    std::uint32_t s = 0;
    for (long long o = 0; o < steps; ++o) {
        const long long p = pos0 + o;
        const int col = column_of<0>((p >= 0 && p < a.n) ? a.text[p] : 0u, nullptr, a);
        s = col < 0 ? 0u : __ldg(a.next + s * 4u + static_cast<std::uint32_t>(col));
        if (o >= a.halo && has_out(s, a)) emit<PASS>(s, p, cnt, wr, a);
    }
    if (PASS == kCount) a.chunk_counts[c] = cnt;
}

// Per-offset deepest-candidate selection and output (count or ordered write).
template <int PASS>
__device__ __noinline__ void resolve_candidates(long long c, Cands cd, int lane, const ScanArgs& a) {
    const long long pos0 = a.emit_from + c * a.chunk - a.halo;
    bool keep[kCand];
    std::uint32_t dep[kCand];
#pragma unroll
    for (int q = 0; q < kCand; ++q) {
        keep[q] = q < cd.n;
        dep[q] = q < cd.n ? __ldg(a.depth + cd.st[q]) : 0u;
    }
    for (int src = 0; src < 32; ++src) {
        const int nsrc = __shfl_sync(0xffffffffu, cd.n, src);
        for (int r = 0; r < nsrc; ++r) {
            std::uint32_t o_r = 0, s_r = 0;
#pragma unroll
            for (int q = 0; q < kCand; ++q)
                if (q == r) {
                    o_r = cd.off[q];
                    s_r = cd.st[q];
                }
            o_r = __shfl_sync(0xffffffffu, o_r, src);
            s_r = __shfl_sync(0xffffffffu, s_r, src);
            const std::uint32_t d_r = __ldg(a.depth + s_r);
#pragma unroll
            for (int q = 0; q < kCand; ++q) {
                if (!keep[q] || o_r != cd.off[q]) continue;
                const bool me = src == lane && r == q;
                const bool earlier = src < lane || (src == lane && r < q);
                if (!me && (d_r > dep[q] || (d_r == dep[q] && earlier))) keep[q] = false;
            }
        }
    }
    unsigned long long mine = 0;
#pragma unroll
    for (int q = 0; q < kCand; ++q)
        if (keep[q]) mine += __ldg(a.out_off + cd.st[q] + 1) - __ldg(a.out_off + cd.st[q]);
    if (PASS == kCount) {
        unsigned long long sum = mine;
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) a.chunk_counts[c] = sum;
        return;
    }
    const unsigned long long wr0 = a.chunk_offs[c];
#pragma unroll
    for (int q = 0; q < kCand; ++q) {
        // slot = outputs of kept candidates at smaller offsets (kept offsets are distinct)
        unsigned long long before = 0;
        for (int src = 0; src < 32; ++src) {
            const int nsrc = __shfl_sync(0xffffffffu, cd.n, src);
            for (int r = 0; r < nsrc; ++r) {
                std::uint32_t o_r = 0, s_r = 0;
                int k_r = 0;
#pragma unroll
                for (int z = 0; z < kCand; ++z)
                    if (z == r) {
                        o_r = cd.off[z];
                        s_r = cd.st[z];
                        k_r = keep[z];
                    }
                o_r = __shfl_sync(0xffffffffu, o_r, src);
                s_r = __shfl_sync(0xffffffffu, s_r, src);
                k_r = __shfl_sync(0xffffffffu, k_r, src);
                if (k_r && keep[q] && o_r < cd.off[q])
                    before += __ldg(a.out_off + s_r + 1) - __ldg(a.out_off + s_r);
            }
        }
        if (keep[q]) {
            unsigned long long w2 = wr0 + before, dummy = 0;
            emit<PASS>(cd.st[q], pos0 + cd.off[q], dummy, w2, a);
        }
    }
}

template <int PASS>
__device__ __forceinline__ void fixup_chunk(long long c, std::uint32_t tab, int lane, const ScanArgs& a) {
    const long long pos0 = a.emit_from + c * a.chunk - a.halo;
    const long long steps = a.halo + a.chunk;
    const std::uint32_t ne = a.ev_count[c];
    const uint2* ev = reinterpret_cast<const uint2*>(a.events) + static_cast<unsigned long long>(c) * a.ev_cap;
    Cands cd;
    cd.n = 0;
    if (ne <= a.ev_cap)
        for (std::uint32_t j = lane; j < ne; j += 32) walk_event(ev[j], pos0, steps, tab, cd, a);
    const bool overflow = __any_sync(0xffffffffu, cd.n > kCand) || ne > a.ev_cap;
    if (overflow) {
        if (lane == 0) exact_chunk_walk<PASS>(c, a);
        return;
    }
    if (!__any_sync(0xffffffffu, cd.n > 0)) {
        if (PASS == kCount && lane == 0) a.chunk_counts[c] = 0;
        return;
    }
    resolve_candidates<PASS>(c, cd, lane, a);
}

// Persistent: one CTA per SM stages the truncated table once; warps stride
// over the chunks (COUNT: all; WRITE: the compacted chunks with matches).
template <int PASS>
__global__ void __launch_bounds__(1024, 1) fixup_kernel(const ScanArgs a) {
    extern __shared__ __align__(16) std::uint8_t smem[];
    const std::uint32_t tab = smem_u32(smem);
    const int lane = threadIdx.x & 31;
    const long long n_work = PASS == kWrite ? static_cast<long long>(*a.active_count) : a.n_chunks;
    const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    const long long w0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if ((static_cast<long long>(blockIdx.x) * blockDim.x >> 5) >= n_work) return;
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.hotH);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (std::uint32_t i = threadIdx.x; i < a.smem_table_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    for (long long w = w0; w < n_work; w += warps)
        fixup_chunk<PASS>(PASS == kWrite ? static_cast<long long>(a.active_list[w]) : w, tab, lane, a);
}

// Compacts the ids of chunks with at least one match (order is irrelevant:
// every chunk writes at its own prefix offset).
__global__ void compact_active_kernel(const unsigned long long* counts, long long n, std::uint32_t* list,
                                      std::uint32_t* n_active) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const bool on = counts[i] != 0;
        const unsigned m = __ballot_sync(__activemask(), on);
        if (!m) continue;
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(m) - 1;
        std::uint32_t base = 0;
        if (lane == leader) base = atomicAdd(n_active, static_cast<std::uint32_t>(__popc(m)));
        base = __shfl_sync(m | (1u << lane), base, leader);
        if (on) list[base + __popc(m & ((1u << lane) - 1))] = static_cast<std::uint32_t>(i);
    }
}

// Per-pattern counts from per-state visit counts: count(p) = sum of visits(s)
// over output states s with p in out(s). One thread per output state.
__global__ void pattern_counts_kernel(const unsigned long long* visits, const std::uint32_t* out_off,
                                      const std::uint32_t* out_ids, std::uint32_t Hn, std::uint32_t H,
                                      std::uint32_t Cn, std::uint32_t S, unsigned long long* counts) {
    const std::uint32_t n_hot_out = H - Hn;
    const std::uint32_t n_out = n_hot_out + (S - Cn);
    for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_out; i += gridDim.x * blockDim.x) {
        const std::uint32_t s = i < n_hot_out ? Hn + i : Cn + (i - n_hot_out);
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

}  // namespace kern
}  // namespace acg
