// Sampled q-gram prefilter shared by the host build (automaton.cpp) and the
// device scan (filter_kernels.cuh).
//
// Idea. Every occurrence [i, e] of a pattern of length L >= q + kQSample - 1
// contains, at the first sample position j >= i (samples = buffer offsets
// that are multiples of kQSample), the q-gram text[j, j+q) = P[j-i, j-i+q)
// with j - i in [0, kQSample). The filter stores the q-grams of every pattern
// at offsets 0..kQSample-1 in a three-stage Bloom filter (no false
// negatives). A sample whose q-gram passes marks the 64-byte blocks holding
// every end it could own ([j+q-1, j+maxlen-1]) as dirty, and only dirty
// blocks are walked with the exact automaton. Every match is therefore found,
// and reported exactly once (by the block holding its end).
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
// Bloom stages: 2^20, 2^19 and 2^18 bits = 224 KiB of shared memory in total.
constexpr std::uint32_t kQLog0 = 20, kQLog1 = 19, kQLog2 = 18;
constexpr std::uint32_t kQOff1 = (1u << kQLog0) / 32;               // word offset of stage 1
constexpr std::uint32_t kQOff2 = kQOff1 + (1u << kQLog1) / 32;      // word offset of stage 2
constexpr std::uint32_t kQWords = kQOff2 + (1u << kQLog2) / 32;     // 57344 words
constexpr std::uint32_t kQMul0 = 0x9E3779B1u, kQMul1 = 0x85EBCA77u, kQMul2 = 0xC2B2AE3Du;

#if defined(__CUDACC__)
#define ACG_HD __host__ __device__ __forceinline__
#else
#define ACG_HD inline
#endif

// Bit index of code c in stage k (multiplicative hashing, top bits).
ACG_HD std::uint32_t qhash0(std::uint32_t c) { return (c * kQMul0) >> (32 - kQLog0); }
ACG_HD std::uint32_t qhash1(std::uint32_t c) { return (c * kQMul1) >> (32 - kQLog1); }
ACG_HD std::uint32_t qhash2(std::uint32_t c) { return (c * kQMul2) >> (32 - kQLog2); }

#undef ACG_HD

}  // namespace acg
