// Drop-in for the reference's file I/O (/root/reference/proj/include/acmatch/
// io.hpp:15-98): same types, functions, line rules and errors, over the C ABI
// loaders of include/acg.h (acg_load_input: parallel reads into page-locked
// memory; acg_load_patterns). New here: PinnedInput keeps the page-locked
// buffer (no copy into a std::string) and scan(Automaton, PinnedInput) runs
// the pipelined host scan (acg_scan_pipelined: H2D copies overlapped with the
// scan and the record read-back).
#pragma once

#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "acg.h"
#include "acmatch/aho_corasick.hpp"
#include "acmatch/errors.hpp"

namespace acmatch {

// Dictionary read from a one-pattern-per-line file, plus load diagnostics (:17-22).
struct PatternFile {
    std::vector<Pattern> patterns;
    std::size_t duplicates = 0;     // repeated lines dropped (first occurrence kept)
    std::size_t skipped_empty = 0;  // empty lines
};

// A whole file in page-locked host memory (acg_load_input). Move-only.
class PinnedInput {
public:
    explicit PinnedInput(const std::filesystem::path& path) {
        detail::check(acg_load_input(path.string().c_str(), &data_, &n_));
    }
    PinnedInput(PinnedInput&& o) noexcept : data_(std::exchange(o.data_, nullptr)), n_(std::exchange(o.n_, 0)) {}
    PinnedInput& operator=(PinnedInput&& o) noexcept {
        if (this != &o) {
            acg_host_free(data_);
            data_ = std::exchange(o.data_, nullptr);
            n_ = std::exchange(o.n_, 0);
        }
        return *this;
    }
    PinnedInput(const PinnedInput&) = delete;
    PinnedInput& operator=(const PinnedInput&) = delete;
    ~PinnedInput() { acg_host_free(data_); }

    std::string_view view() const noexcept { return {reinterpret_cast<const char*>(data_), n_}; }
    const std::uint8_t* data() const noexcept { return data_; }
    std::size_t size() const noexcept { return n_; }

private:
    std::uint8_t* data_ = nullptr;
    std::uint64_t n_ = 0;
};

// Whole file as raw bytes; no decoding, no newline treatment (:25-31).
inline std::string load_input(const std::filesystem::path& path) {
    const PinnedInput in(path);
    return std::string(in.view());
}

// Splits on LF, strips one trailing CR per line, skips empty lines,
// deduplicates keeping the first occurrence, dense ids in load order (:37-65).
inline PatternFile load_patterns(const std::filesystem::path& path) {
    std::uint8_t* concat = nullptr;
    std::uint64_t* offs = nullptr;
    std::uint32_t count = 0;
    std::uint64_t dups = 0, empty = 0;
    detail::check(acg_load_patterns(path.string().c_str(), &concat, &offs, &count, &dups, &empty));
    PatternFile result;
    result.patterns.reserve(count);
    for (std::uint32_t i = 0; i < count; ++i)
        result.patterns.push_back(
            Pattern{i, std::string(reinterpret_cast<const char*>(concat) + offs[i], offs[i + 1] - offs[i])});
    result.duplicates = dups;
    result.skipped_empty = empty;
    acg_host_free(concat);
    acg_host_free(offs);
    return result;
}

// Raw byte write (:68-76).
inline void write_bytes(const std::filesystem::path& path, std::string_view bytes) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open " + path.string());
    out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
    out.flush();
    if (!out) throw IoError("write failed: " + path.string());
}

// Writes patterns one per line, LF-terminated (:79-90).
inline void write_pattern_file(const std::filesystem::path& path, const std::vector<Pattern>& patterns) {
    std::string buffer;
    for (const Pattern& p : patterns) {
        if (p.bytes.find('\n') != std::string::npos)
            throw Error("patterns containing newline bytes cannot be written one per line");
        buffer += p.bytes;
        buffer += '\n';
    }
    write_bytes(path, buffer);
}

// acmatch::scan over a page-locked file image: the pipelined host scan
// (copies overlapped with the scan and the record read-back), widened to
// MatchRecord in canonical (end, pattern_id) order.
inline std::vector<MatchRecord> scan(const Automaton& automaton, const PinnedInput& input, int device = 0) {
    std::uint64_t m = 0;
    std::uint32_t id_bits = 1;
    // first pass sizes the output: counts only (cheap), then the list
    detail::check(acg_scan_pipelined(automaton.handle(), device, input.data(), input.size(), 0, 0, 0, 0, nullptr, 0, nullptr,
                                     &m, &id_bits, nullptr));
    std::vector<std::uint64_t> packed(m);
    detail::check(acg_scan_pipelined(automaton.handle(), device, input.data(), input.size(), 0, 0, 0, 0, packed.data(), m,
                                     nullptr, &m, &id_bits, nullptr));
    std::vector<MatchRecord> out(m);
    const std::uint64_t mask = (1ull << id_bits) - 1;
    for (std::uint64_t i = 0; i < m; ++i)
        out[i] = MatchRecord{static_cast<std::uint32_t>(packed[i] & mask), static_cast<std::size_t>(packed[i] >> id_bits)};
    return out;
}

}  // namespace acmatch
