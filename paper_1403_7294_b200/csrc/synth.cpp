// Deterministic synthetic corpora for the five BASELINE.json workloads.
//
// Workload synthesis only: this library is neither the scan nor the oracle.
// Every byte is a pure function of (kind, seed, N, offset), so the host
// (threaded) and any window of the text can be regenerated independently, and
// the bench, the tests and the golden script all see identical bytes. Draws use
// splitmix64 with `x % n` reductions, never std::*_distribution (which is
// implementation-defined; the reference makes the same portability choice at
// proj/include/acmatch/corpus.hpp:37-42).
//
// kinds:
//   0 DNA          iid uniform ACGT text; pattern k even = text substring at a
//                  uniform offset, k odd = iid ACGT (configs[0..2]).
//   1 PROTEIN      iid over ACDEFGHIKLMNPQRSTVWY with P(rank r) ~ 1/(r+1) over
//                  a seed-shuffled letter order; patterns iid from the same law
//                  (configs[3]).
//   2 ADVERSARIAL  fair-coin segments: iid ACGT or a tandem repeat (period
//                  U[1,6], random ACGT unit), segment length U[256,65536], last
//                  segment truncated; patterns: k%5<2 are tandem repeats
//                  (period U[1,6]), the rest iid ACGT (configs[4]).
// Patterns are redrawn until distinct, so P is exact.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr std::uint64_t kTextSalt = 0x7465787400000001ull;
constexpr std::uint64_t kPatSalt = 0x7061747400000002ull;
constexpr std::uint64_t kSegSalt = 0x7365677300000003ull;
constexpr std::uint64_t kPermSalt = 0x7065726d00000004ull;

inline std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Counter-based draw: the i-th 64-bit value of stream (seed, salt).
inline std::uint64_t draw_at(std::uint64_t seed, std::uint64_t salt, std::uint64_t i) {
    return mix64(mix64(seed ^ salt) + (i + 1) * kGolden);
}

// Sequential generator (splitmix64).
struct Seq {
    std::uint64_t x;
    Seq(std::uint64_t seed, std::uint64_t salt) : x(mix64(seed ^ salt)) {}
    std::uint64_t next() {
        x += kGolden;
        return mix64(x);
    }
    std::uint64_t below(std::uint64_t n) { return next() % n; }
};

const char kDna[4] = {'A', 'C', 'G', 'T'};
const char kAmino[21] = "ACDEFGHIKLMNPQRSTVWY";

struct ProteinLaw {
    char order[20];
    std::uint64_t thr[20];  // cumulative thresholds on a 32-bit uniform
};

ProteinLaw protein_law(std::uint64_t seed) {
    ProteinLaw law;
    std::memcpy(law.order, kAmino, 20);
    Seq rng(seed, kPermSalt);
    for (int i = 19; i > 0; --i) {  // Fisher-Yates
        const int j = static_cast<int>(rng.below(static_cast<std::uint64_t>(i + 1)));
        std::swap(law.order[i], law.order[j]);
    }
    double h = 0.0;
    for (int r = 0; r < 20; ++r) h += 1.0 / (r + 1);
    double acc = 0.0;
    for (int r = 0; r < 20; ++r) {
        acc += 1.0 / (r + 1) / h;
        law.thr[r] = static_cast<std::uint64_t>(acc * 4294967296.0);
    }
    law.thr[19] = 4294967296ull;
    return law;
}

inline char protein_letter(const ProteinLaw& law, std::uint32_t u) {
    int r = 0;
    while (r < 19 && u >= law.thr[r]) ++r;
    return law.order[r];
}

struct Segment {
    std::uint64_t start;
    std::uint32_t period;  // 0 = iid segment
    char unit[6];
};

std::vector<Segment> adversarial_segments(std::uint64_t seed, std::uint64_t n) {
    std::vector<Segment> segs;
    Seq rng(seed, kSegSalt);
    std::uint64_t pos = 0;
    while (pos < n) {
        Segment s{};
        s.start = pos;
        const bool repeat = rng.next() & 1;
        const std::uint64_t len = 256 + rng.below(65536 - 256 + 1);
        if (repeat) {
            s.period = 1 + static_cast<std::uint32_t>(rng.below(6));
            for (std::uint32_t k = 0; k < s.period; ++k) s.unit[k] = kDna[rng.below(4)];
        }
        segs.push_back(s);
        pos += len;
    }
    return segs;
}

inline char dna_at(std::uint64_t seed, std::uint64_t i) {
    const std::uint64_t h = draw_at(seed, kTextSalt, i >> 5);
    return kDna[(h >> ((i & 31) * 2)) & 3];
}

struct TextGen {
    int kind;
    std::uint64_t seed, n;
    ProteinLaw law{};
    std::vector<Segment> segs;

    TextGen(int k, std::uint64_t s, std::uint64_t total) : kind(k), seed(s), n(total) {
        if (kind == 1) law = protein_law(seed);
        if (kind == 2) segs = adversarial_segments(seed, n);
    }

    void fill(std::uint64_t lo, std::uint64_t hi, std::uint8_t* out) const {
        if (kind == 0) {
            std::uint64_t i = lo;
            while (i < hi) {
                const std::uint64_t h = draw_at(seed, kTextSalt, i >> 5);
                const std::uint64_t end = std::min(hi, (i | 31) + 1);
                for (; i < end; ++i) out[i - lo] = static_cast<std::uint8_t>(kDna[(h >> ((i & 31) * 2)) & 3]);
            }
        } else if (kind == 1) {
            for (std::uint64_t i = lo; i < hi; ++i) {
                const std::uint64_t h = draw_at(seed, kTextSalt, i >> 1);
                const auto u = static_cast<std::uint32_t>(h >> ((i & 1) * 32));
                out[i - lo] = static_cast<std::uint8_t>(protein_letter(law, u));
            }
        } else {
            // segment containing lo
            std::size_t k = std::upper_bound(segs.begin(), segs.end(), lo,
                                             [](std::uint64_t v, const Segment& s) { return v < s.start; }) -
                            segs.begin() - 1;
            std::uint64_t i = lo;
            while (i < hi) {
                const Segment& s = segs[k];
                const std::uint64_t seg_end = (k + 1 < segs.size()) ? segs[k + 1].start : n;
                const std::uint64_t end = std::min(hi, seg_end);
                if (s.period == 0) {
                    for (; i < end; ++i) out[i - lo] = static_cast<std::uint8_t>(dna_at(seed, i));
                } else {
                    for (; i < end; ++i) out[i - lo] = static_cast<std::uint8_t>(s.unit[(i - s.start) % s.period]);
                }
                ++k;
            }
        }
    }
};

}  // namespace

extern "C" {

// Bytes [lo, hi) of the kind's text of total length n, written to out[0, hi-lo).
// Returns 0, or -1 on bad arguments.
int acg_synth_text(int kind, std::uint64_t seed, std::uint64_t n, std::uint64_t lo, std::uint64_t hi,
                   std::uint8_t* out, int threads) {
    if (kind < 0 || kind > 2 || lo > hi || hi > n || (hi > lo && !out)) return -1;
    const TextGen gen(kind, seed, n);
    const std::uint64_t len = hi - lo;
    if (threads < 1) threads = 1;
    if (len < (1u << 22)) threads = 1;
    if (threads == 1) {
        gen.fill(lo, hi, out);
        return 0;
    }
    std::vector<std::thread> pool;
    const std::uint64_t step = ((len + threads - 1) / threads + 63) & ~std::uint64_t(63);
    for (int t = 0; t < threads; ++t) {
        const std::uint64_t a = lo + std::min(len, step * t);
        const std::uint64_t b = lo + std::min(len, step * (t + 1));
        if (a >= b) break;
        pool.emplace_back([&gen, a, b, out, lo] { gen.fill(a, b, out + (a - lo)); });
    }
    for (auto& th : pool) th.join();
    return 0;
}

// P distinct patterns, concatenated into buf (capacity cap bytes) with
// offsets offs[0..P]. Returns total bytes, or -1 on bad arguments / overflow,
// -2 when the pattern space is too small to draw P distinct patterns.
long long acg_synth_patterns(int kind, std::uint64_t seed, std::uint64_t n, std::uint32_t count,
                             std::uint32_t len_lo, std::uint32_t len_hi, std::uint8_t* buf,
                             std::uint64_t cap, std::uint64_t* offs) {
    if (kind < 0 || kind > 2 || len_lo < 1 || len_hi < len_lo || !offs) return -1;
    if (kind == 0 && n < len_hi) return -1;
    const TextGen gen(kind, seed, n);
    Seq rng(seed, kPatSalt);
    std::unordered_set<std::string> seen;
    seen.reserve(count * 2ull);
    std::uint64_t total = 0;
    std::string word;
    std::uint64_t attempts = 0;
    offs[0] = 0;
    for (std::uint32_t k = 0; k < count;) {
        if (++attempts > 64ull * count + 1000) return -2;
        const std::uint32_t len = len_lo + static_cast<std::uint32_t>(rng.below(len_hi - len_lo + 1));
        word.assign(len, '\0');
        if (kind == 0) {
            if ((k & 1) == 0) {
                const std::uint64_t off = rng.below(n - len + 1);
                gen.fill(off, off + len, reinterpret_cast<std::uint8_t*>(word.data()));
            } else {
                for (auto& c : word) c = kDna[rng.below(4)];
            }
        } else if (kind == 1) {
            for (auto& c : word) c = protein_letter(gen.law, static_cast<std::uint32_t>(rng.next() >> 32));
        } else {
            if (k % 5 < 2) {
                const std::uint32_t period = 1 + static_cast<std::uint32_t>(rng.below(6));
                char unit[6];
                for (std::uint32_t j = 0; j < period; ++j) unit[j] = kDna[rng.below(4)];
                for (std::uint32_t j = 0; j < len; ++j) word[j] = unit[j % period];
            } else {
                for (auto& c : word) c = kDna[rng.below(4)];
            }
        }
        if (!seen.insert(word).second) continue;  // redraw duplicates
        if (buf) {
            if (total + len > cap) return -1;
            std::memcpy(buf + total, word.data(), len);
        }
        total += len;
        ++k;
        offs[k] = total;
    }
    return static_cast<long long>(total);
}

}  // extern "C"
