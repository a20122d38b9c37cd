// Output step on the GPU: the match list as the
// reference's `acmatch match` output (proj/include/acmatch/cli.hpp:58-76):
//   TSV:  "<end>\t<pattern_id>\t<pattern bytes>\n" per record (:71-74)
//   JSON: [{"end":E,"pattern":"<escaped>","pattern_id":I},...]\n (:63-69;
//         nlohmann dump(-1): compact, keys in std::map order, strings escaped
//         by the host into a per-pattern table, so both formats are one kernel)
// Records are packed u64 (end << id_bits | id) in canonical order. Two passes
// over a window of records: F1 sums the line lengths per 256-record tile (CUB
// scans the tile sums into tile offsets); F2 recomputes each line's length,
// block-scans the tile, assembles the tile's lines in shared memory and
// writes the tile's bytes contiguously (coalesced byte stores). A tile whose
// text exceeds the staging buffer (very long patterns) is written per thread.
#pragma once

#include <cstdint>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

namespace acg {
namespace kern {

constexpr int kFmtTile = 256;
constexpr int kFmtStage = 40 * 1024;  // staging bytes per tile

struct FmtArgs {
    const unsigned long long* rec;  // records of the window
    unsigned long long m;           // records in the window
    std::uint32_t id_bits;
    const std::uint8_t* str;        // per pattern: raw bytes (TSV) or JSON-escaped bytes
    const unsigned long long* str_off;  // P + 1
    int json;
    int open;   // JSON: the window holds the list's first record ("[")
    int close;  // JSON: the window holds the list's last record ("]\n"; no "," after it)
    unsigned long long* tile_sum;   // F1 out: bytes per tile
    const unsigned long long* tile_off;  // F2 in: exclusive prefix (tile 0 -> 0)
    std::uint8_t* out;
};

__device__ __forceinline__ std::uint32_t ndigits(unsigned long long x) {
    std::uint32_t d = 1;
    while (x >= 10ull) {
        x /= 10ull;
        ++d;
    }
    return d;
}

// JSON literal pieces: {"end":  ,"pattern":"  ","pattern_id":  }
__device__ __constant__ char kJ0[] = "{\"end\":";
__device__ __constant__ char kJ1[] = ",\"pattern\":\"";
__device__ __constant__ char kJ2[] = "\",\"pattern_id\":";
constexpr std::uint32_t kJ0n = 7, kJ1n = 12, kJ2n = 15;

__device__ __forceinline__ std::uint32_t line_len(const FmtArgs& a, unsigned long long i) {
    const unsigned long long r = a.rec[i];
    const unsigned long long end = r >> a.id_bits;
    const std::uint32_t id = static_cast<std::uint32_t>(r & ((1ull << a.id_bits) - 1));
    const std::uint32_t s = static_cast<std::uint32_t>(a.str_off[id + 1] - a.str_off[id]);
    if (!a.json) return ndigits(end) + 1 + ndigits(id) + 1 + s + 1;
    std::uint32_t L = kJ0n + ndigits(end) + kJ1n + s + kJ2n + ndigits(id) + 1;
    if (a.open && i == 0) L += 1;                                  // "["
    L += (a.close && i + 1 == a.m) ? 2u : 1u;                      // "]\n" or ","
    return L;
}

template <typename Put>
__device__ __forceinline__ void put_digits(unsigned long long x, std::uint32_t n, std::uint32_t at, Put put) {
    for (std::uint32_t k = n; k-- > 0;) {
        put(at + k, static_cast<std::uint8_t>('0' + x % 10ull));
        x /= 10ull;
    }
}

template <typename Put>
__device__ __forceinline__ void put_line(const FmtArgs& a, unsigned long long i, std::uint32_t at, Put put) {
    const unsigned long long r = a.rec[i];
    const unsigned long long end = r >> a.id_bits;
    const std::uint32_t id = static_cast<std::uint32_t>(r & ((1ull << a.id_bits) - 1));
    const unsigned long long s0 = a.str_off[id], s1 = a.str_off[id + 1];
    const std::uint32_t de = ndigits(end), di = ndigits(id);
    auto str = [&](std::uint32_t p) {
        for (unsigned long long k = s0; k < s1; ++k) put(p++, __ldg(a.str + k));
        return p;
    };
    if (!a.json) {
        put_digits(end, de, at, put);
        at += de;
        put(at++, '\t');
        put_digits(id, di, at, put);
        at += di;
        put(at++, '\t');
        at = str(at);
        put(at, '\n');
        return;
    }
    if (a.open && i == 0) put(at++, '[');
    for (std::uint32_t k = 0; k < kJ0n; ++k) put(at++, kJ0[k]);
    put_digits(end, de, at, put);
    at += de;
    for (std::uint32_t k = 0; k < kJ1n; ++k) put(at++, kJ1[k]);
    at = str(at);
    for (std::uint32_t k = 0; k < kJ2n; ++k) put(at++, kJ2[k]);
    put_digits(id, di, at, put);
    at += di;
    put(at++, '}');
    if (a.close && i + 1 == a.m) {
        put(at++, ']');
        put(at, '\n');
    } else {
        put(at, ',');
    }
}

__global__ void __launch_bounds__(kFmtTile) format_len_kernel(const FmtArgs a) {
    using Scan = cub::BlockReduce<unsigned long long, kFmtTile>;
    __shared__ typename Scan::TempStorage tmp;
    const unsigned long long tiles = (a.m + kFmtTile - 1) / kFmtTile;
    for (unsigned long long t = blockIdx.x; t < tiles; t += gridDim.x) {
        const unsigned long long i = t * kFmtTile + threadIdx.x;
        const unsigned long long L = i < a.m ? line_len(a, i) : 0ull;
        const unsigned long long sum = Scan(tmp).Sum(L);
        if (threadIdx.x == 0) a.tile_sum[t] = sum;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kFmtTile) format_write_kernel(const FmtArgs a) {
    using Scan = cub::BlockScan<std::uint32_t, kFmtTile>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ __align__(16) std::uint8_t stage[kFmtStage];
    __shared__ std::uint32_t total_sh;
    const unsigned long long tiles = (a.m + kFmtTile - 1) / kFmtTile;
    for (unsigned long long t = blockIdx.x; t < tiles; t += gridDim.x) {
        const unsigned long long i = t * kFmtTile + threadIdx.x;
        const std::uint32_t L = i < a.m ? line_len(a, i) : 0u;
        std::uint32_t off = 0, total = 0;
        Scan(tmp).ExclusiveSum(L, off, total);
        if (threadIdx.x == 0) total_sh = total;
        __syncthreads();
        total = total_sh;
        std::uint8_t* dst = a.out + a.tile_off[t];
        if (total <= static_cast<std::uint32_t>(kFmtStage)) {
            if (i < a.m) put_line(a, i, off, [&](std::uint32_t p, std::uint8_t c) { stage[p] = c; });
            __syncthreads();
            for (std::uint32_t k = threadIdx.x; k < total; k += kFmtTile) dst[k] = stage[k];
        } else if (i < a.m) {
            put_line(a, i, off, [&](std::uint32_t p, std::uint8_t c) { dst[p] = c; });
        }
        __syncthreads();
    }
}

}  // namespace kern
}  // namespace acg
