// Compressed hot automaton (CTAB) for the EXACT walk on small generic
// alphabets (at most kCtMaxK columns incl. the escape column: proteins),
// shared by the host build (automaton.cpp) and the walk (exact_kernels.cuh).
//
// Why. The dense u16 hot rows of KE (K entries per state) hold ~5,500 of
// cfg3's 26,198 states in shared memory; 3 % of the steps leave them and every
// warp-step with one such lane waits an L2 round trip. Most entries of a dense
// row carry no information: delta(s, c) is a SHALLOW state for most c, and a
// shallow target is a function of the last few text bytes alone.
//
// Scheme. Let D be the default depth (3 for K <= 21). For every position the
// walk computes, from the text only (off the state's dependency chain),
//     x = T_D[last D columns] = the longest suffix of those D symbols that is
//         a trie prefix (the true DFA walked from the root over them).
// The true next state t = delta(s, c) equals x whenever depth(t) <= D. The
// pairs (s, c) with depth(t) > D are the EXCEPTIONS of row s (cfg3: 4.3 per
// state instead of 21 dense entries). Exceptions of the hot states live in one
// row-displaced table (Tarjan & Yao's sparse-table compression): state s has
// an id b(s) — its row's displacement, unique per state — and its exception
// for column c sits in slot b(s) + c, tagged with c. A lookup is ONE
// shared-memory load on the state's dependency chain:
//     e = tab[id + c];  next = (col field of e == c) ? e's state word : x
// (slot id + c belongs to at most one row; a row with base b' != id that owns
// it stores column id + c - b' != c, so a foreign entry never matches; empty
// slots hold column 31). Hot rows are complete, so the walk is exact; a state
// outside the hot set is a COLD state word and steps through the dense
// L2-resident table (`next`, device ids) until it is hot again.
//
// Deep default. When every state of depth <= D is hot, the default takes one
// more level from the same table, still from the text alone: the depth-(D+1)
// children of the depth-D states are entries of their rows, so
//     x' = (entry of row x_{i-1} for column c_i matches) ? that child : x_i
// is the longest suffix of the last D+1 symbols that is a trie prefix, and the
// other rows keep only the pairs whose target is deeper than D + 1 (cfg3:
// 37,771 entries for ALL 26,198 states — the whole automaton is hot, against
// 112,338 entries with the plain default).
//
// State word (u32): bits 0-24 value, 25-29 zero (the entry's column field),
// bit 30 cold, bit 31 has outputs.
//   hot:  value = id (slot index < slots)
//   cold: value = slots + output rank (output states), else the device id
// An output visit logs the event payload (hot: id, cold output: slots + rank);
// E1 / E2 map payloads back to output ranks (id -> rank table).
// Counted words (Dfa::ct_cnt: every payload < 2^16 and every output list
// shorter than 255): byte 2 of an output state's word holds its output count,
// the payload is bits 0-15 — the walk then sums each chunk's record count
// itself (one PRMT and one add per logged step) and the separate counting pass
// (E1) is not run for list scans; E2 takes the visit histogram.
#pragma once

#include <cstdint>

namespace acg {

constexpr std::uint32_t kCtMaxK = 31;            // columns (5-bit column field; 31 = empty slot)
constexpr std::uint32_t kCtValMask = 0x01FFFFFFu;
constexpr std::uint32_t kCtColShift = 25;
constexpr std::uint32_t kCtColMask = 0x3E000000u;
constexpr std::uint32_t kCtCold = 0x40000000u;
constexpr std::uint32_t kCtOut = 0x80000000u;
constexpr std::uint32_t kCtEmpty = kCtColMask;   // column 31, value 0: matches no column
constexpr std::uint32_t kCtDefaultMaxBytes = 40 * 1024;  // T_D table bound (K^D u32 entries)
constexpr std::uint32_t kCtNoRank = 0xFFFFu;
constexpr std::uint32_t kCtPayBits = 16;         // counted words: payload bits; the output count is byte 2
constexpr std::uint32_t kCtPayMask = (1u << kCtPayBits) - 1u;

}  // namespace acg
