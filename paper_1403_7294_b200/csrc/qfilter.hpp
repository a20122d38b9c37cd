// Sampled q-gram prefilter shared by the host build (automaton.cpp) and the
// device scan (filter_kernels.cuh).
//
// Idea. Every occurrence [i, e] of a pattern of length L >= q + kQSample - 1
// contains, at the first sample position j >= i (samples = buffer offsets
// that are multiples of kQSample), the q-gram text[j, j+q) = P[j-i, j-i+q)
// with offset o = j - i in [0, kQSample). So:
//
//   1. KQ streams the text and tests the q-gram at every sample against a
//      blocked Bloom filter of all (pattern, o) q-grams (shared memory, one
//      32-bit word per probe, four bits per key; no false negatives);
//   2. V0 confirms each survivor j exactly: the q-gram's (pattern, o) list
//      from an exact hash table, then a byte compare of the pattern against
//      the text at i = j - o. A confirmed occurrence marks the 64-byte block
//      holding its end e = i + L - 1 as dirty;
//   3. only dirty blocks are walked with the real automaton (V1 counts, V2
//      writes in order), which emits every match ending in them.
//
// Every match's block is dirty (steps 1-2 have no false negatives for its
// owned sample), and every match is emitted once, by the block holding its
// end. The automaton stays the single source of truth for what is emitted.
//
// Codes. Base b -> 2-bit code (b >> 1) & 3 (A0 C1 T2 G3, the dna4 column);
// a q-gram's code has base k at bits 2k (q <= 16: one 32-bit word).
#pragma once

#include <cstdint>

namespace acg {

constexpr std::uint32_t kQSample = 4;   // sample stride (bytes)
constexpr std::uint32_t kQMaxQ = 16;    // q-gram length cap (32-bit codes)
constexpr std::uint32_t kQMinQ = 10;    // below this the filter is not selective
constexpr std::uint32_t kQBlock = 64;   // dirty-block size (bytes)
constexpr std::uint32_t kQChunkBlocks = 128;  // blocks per output chunk (8 KiB)
constexpr std::uint32_t kQWords = 57344;      // Bloom words (224 KiB: all of the opt-in shared memory but 3 KiB)
// Bitmap level 1 (dictionaries of at most kQBitmapMaxKeys keys): a 2^20-bit
// bitmap of the keys' 10-gram prefixes (128 KiB, direct index: no hash),
// then a blocked Bloom filter of the full q-grams in the rest of shared memory.
constexpr std::uint32_t kQBitmapWords = 1u << 15;
constexpr std::uint32_t kQWordsBM = 24576;      // level-2 Bloom words beside the bitmap (96 KiB)
constexpr std::uint32_t kQBitmapMaxKeys = 60000;  // bitmap density <= 5.7 %
constexpr std::uint32_t kQMul0 = 0x9E3779B1u, kQMul1 = 0x85EBCA77u, kQMul2 = 0xC2B2AE3Du;
constexpr std::uint32_t kQEmpty = 0xFFFFFFFFu;  // exact-table slot marker
constexpr std::uint32_t kQSingle = 0x80000000u;  // slot payload = kQSingle | the bucket's only entry

#if defined(__CUDACC__)
#define ACG_HD __host__ __device__ __forceinline__
#else
#define ACG_HD inline
#endif

ACG_HD std::uint32_t qmulhi(std::uint32_t a, std::uint32_t b) {
#if defined(__CUDA_ARCH__)
    return __umulhi(a, b);
#else
    return static_cast<std::uint32_t>((static_cast<std::uint64_t>(a) * b) >> 32);
#endif
}

ACG_HD std::uint32_t qperm(std::uint32_t x, std::uint32_t y, std::uint32_t sel) {  // PRMT, selectors < 8
#if defined(__CUDA_ARCH__)
    return __byte_perm(x, y, sel);
#else
    const std::uint64_t v = (static_cast<std::uint64_t>(y) << 32) | x;
    std::uint32_t r = 0;
    for (int i = 0; i < 4; ++i) r |= static_cast<std::uint32_t>((v >> (8 * ((sel >> (4 * i)) & 7u))) & 0xFFu) << (8 * i);
    return r;
#endif
}

// Bloom probe of a q-gram given as y = code << (32 - 2q) (the code in the
// top bits). Both parts come from one multiplicative hash h = y * kQMul0 —
// on the device h = window * (2^(32-2q) * kQMul0), one multiply from the
// unmasked 32-bit window, since the bases past the q-gram fall off the top.
// qword: the word index (h's high bits scaled to the table); qmask: four
// bits, one in each byte of the word (bit (sel_i & 7) of byte i, sel from
// the high half of h * kQMul1, independent of the word index) — one PRMT.
ACG_HD std::uint32_t qhash(std::uint32_t y) { return y * kQMul0; }
ACG_HD std::uint32_t qword(std::uint32_t h, std::uint32_t words) { return qmulhi(h, words); }
ACG_HD std::uint32_t qmask(std::uint32_t h) {
    return qperm(0x08040201u, 0x80402010u, qmulhi(h, kQMul1) & 0x7777u);
}
// Level-2 filter: its own word from h2 = h * kQMul3; the mask tested is level 1's
// (given the mask, the two words' contents are independent, so the pass rates multiply).
constexpr std::uint32_t kQMul3 = 0x27D4EB2Fu;
constexpr double kQLevel1Max = 0.30;  // a level-1 pass rate above this is not worth streaming
ACG_HD std::uint32_t qhash2(std::uint32_t h) { return h * kQMul3; }
ACG_HD std::uint32_t qtop(std::uint32_t code, std::uint32_t q) { return q >= 16 ? code : code << (32 - 2 * q); }
// Exact table slot of code c in a table of 2^bits slots.
ACG_HD std::uint32_t qslot(std::uint32_t c, std::uint32_t bits) { return (c * kQMul2) >> (32 - bits); }

#undef ACG_HD

}  // namespace acg
