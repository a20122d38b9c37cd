// Drop-in for the reference's core automaton API
// (/root/reference/proj/include/acmatch/aho_corasick.hpp): same names, types,
// numbering and error behaviour, implemented over the C ABI of libacg.so
// (include/acg.h). build() constructs the machine on the host exactly as the
// reference does (DFS-preorder numbering, BFS failure links, suffix-closed
// sorted outputs); scan() runs on the GPU. Link with -lacg.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "acg.h"
#include "acmatch/errors.hpp"

namespace acmatch {

using StateId = std::uint32_t;  // aho_corasick.hpp:18

inline constexpr StateId kRoot = 0;  // :20

// One dictionary keyword; ids are dense, 0-based, in load order (:23-26).
struct Pattern {
    std::uint32_t id = 0;
    std::string bytes;
};

// One occurrence: end = 0-based offset of its last byte (:30-35).
struct MatchRecord {
    std::uint32_t pattern_id = 0;
    std::size_t end = 0;

    friend bool operator==(const MatchRecord&, const MatchRecord&) = default;
};

// Canonical order (end, pattern_id) ascending (:38-41).
inline bool match_before(const MatchRecord& a, const MatchRecord& b) noexcept {
    if (a.end != b.end) return a.end < b.end;
    return a.pattern_id < b.pattern_id;
}

// Failure links followed by the reference scan's NFA walk (:46-48).
struct ScanStats {
    std::uint64_t failure_follows = 0;
};

namespace detail {

[[noreturn]] inline void throw_acg(int rc) {
    const std::string msg = acg_last_error();
    switch (rc) {
        case ACG_ERR_EMPTY_DICTIONARY: throw EmptyDictionaryError(msg);
        case ACG_ERR_EMPTY_PATTERN: throw EmptyPatternError(msg);
        case ACG_ERR_INVALID_WORKER_COUNT: throw InvalidWorkerCountError(msg);
        case ACG_ERR_CUDA:
        case ACG_ERR_OUT_OF_MEMORY:
        case ACG_ERR_NO_DEVICE: throw DeviceError(msg);
        case ACG_ERR_IO: throw IoError(msg);
        default: throw Error(msg);
    }
}

inline void check(int rc) {
    if (rc != ACG_OK) throw_acg(rc);
}

}  // namespace detail

// The pattern-matching machine (:58-121). Immutable and copyable; copies
// share the host automaton and its device tables. Any number of threads may
// scan with it concurrently.
class Automaton {
public:
    std::size_t state_count() const noexcept { return h_ ? acg_state_count(h_.get()) : 0; }

    const std::vector<Pattern>& patterns() const noexcept {
        static const std::vector<Pattern> none;  // (a default-constructed machine has no patterns)
        return patterns_ ? *patterns_ : none;
    }

    // Goto edge out of s on byte b, if any (:67-74).
    std::optional<StateId> goto_transition(StateId s, unsigned char b) const {
        StateId to = 0;
        if (h_ && acg_goto_transition(h_.get(), s, b, &to)) return to;
        return std::nullopt;
    }

    // Goto edges out of s, sorted by byte (:77-80).
    std::span<const std::pair<unsigned char, StateId>> transitions(StateId s) const {
        if (!edge_off_) return {};
        const std::uint32_t lo = (*edge_off_)[s], hi = (*edge_off_)[s + 1];
        return {edges_->data() + lo, hi - lo};
    }

    StateId failure(StateId s) const { return h_ ? acg_failure(h_.get(), s) : kRoot; }  // :84-87

    // Pattern ids ending at s, ascending, suffix-closed (:92-95).
    std::span<const std::uint32_t> outputs(StateId s) const {
        if (!h_) return {};
        const std::uint32_t* ids = nullptr;
        const std::uint32_t n = acg_outputs(h_.get(), s, &ids);
        return {ids, n};
    }

    std::uint32_t depth(StateId s) const { return h_ ? acg_depth(h_.get(), s) : 0; }  // :98-101

    // The C ABI handle (device-resident scanning: acg_scanner_*).
    const acg_automaton* handle() const noexcept { return h_.get(); }

private:
    std::shared_ptr<acg_automaton> h_;
    std::shared_ptr<const std::vector<Pattern>> patterns_;
    std::shared_ptr<const std::vector<std::pair<unsigned char, StateId>>> edges_;
    std::shared_ptr<const std::vector<std::uint32_t>> edge_off_;

    friend Automaton build(std::vector<Pattern> patterns);
};

// Builds the machine (:130-233). Throws EmptyDictionaryError /
// EmptyPatternError, and Error when ids are not dense in load order.
inline Automaton build(std::vector<Pattern> patterns) {
    if (patterns.empty()) throw EmptyDictionaryError("dictionary is empty");
    for (std::size_t i = 0; i < patterns.size(); ++i) {
        if (patterns[i].bytes.empty()) throw EmptyPatternError("pattern " + std::to_string(i) + " is empty");
        if (patterns[i].id != i) throw Error("pattern ids must be dense and follow load order");
    }
    std::vector<std::uint64_t> offs(patterns.size() + 1, 0);
    std::string concat;
    for (std::size_t i = 0; i < patterns.size(); ++i) {
        concat += patterns[i].bytes;
        offs[i + 1] = concat.size();
    }
    acg_automaton* raw = nullptr;
    detail::check(acg_build(reinterpret_cast<const std::uint8_t*>(concat.data()), offs.data(),
                            static_cast<std::uint32_t>(patterns.size()), &raw));
    Automaton a;
    a.h_ = std::shared_ptr<acg_automaton>(raw, acg_automaton_destroy);
    const std::uint32_t n = acg_state_count(raw);
    auto edges = std::make_shared<std::vector<std::pair<unsigned char, StateId>>>();
    auto eoff = std::make_shared<std::vector<std::uint32_t>>(n + 1, 0);
    edges->reserve(n ? n - 1 : 0);
    for (std::uint32_t s = 0; s < n; ++s) {
        const std::uint8_t* bytes = nullptr;
        const std::uint32_t* to = nullptr;
        const std::uint32_t k = acg_transitions(raw, s, &bytes, &to);
        for (std::uint32_t j = 0; j < k; ++j) edges->emplace_back(bytes[j], to[j]);
        (*eoff)[s + 1] = static_cast<std::uint32_t>(edges->size());
    }
    a.edges_ = std::move(edges);
    a.edge_off_ = std::move(eoff);
    a.patterns_ = std::make_shared<const std::vector<Pattern>>(std::move(patterns));
    return a;
}

// Total transition function (:238-245).
inline StateId next_state(const Automaton& a, StateId s, unsigned char b) {
    return acg_next_state(a.handle(), s, b);
}

namespace detail {

inline std::vector<MatchRecord> scan_impl(const Automaton& a, std::string_view input, ScanStats* stats) {
    acg_result* r = nullptr;
    const std::uint32_t flags = ACG_SCAN_LIST | (stats ? ACG_SCAN_STATS : 0u);
    check(acg_scan(a.handle(), reinterpret_cast<const std::uint8_t*>(input.data()), input.size(), flags, &r));
    std::unique_ptr<acg_result, void (*)(acg_result*)> guard(r, acg_result_destroy);
    const std::uint64_t m = acg_result_match_count(r);
    const std::uint32_t* ids = acg_result_ids(r);
    const std::uint64_t* ends = acg_result_ends(r);
    std::vector<MatchRecord> out(m);
    for (std::uint64_t i = 0; i < m; ++i) out[i] = MatchRecord{ids[i], static_cast<std::size_t>(ends[i])};
    if (stats) stats->failure_follows += acg_result_failure_follows(r);
    return out;
}

}  // namespace detail

// Every occurrence, overlapping and nested, in (end, pattern_id) order
// (:250-272); the instrumented overload also counts failure follows exactly as
// the reference's NFA walk does.
inline std::vector<MatchRecord> scan(const Automaton& a, std::string_view input, ScanStats& stats) {
    return detail::scan_impl(a, input, &stats);
}

inline std::vector<MatchRecord> scan(const Automaton& a, std::string_view input) {  // :274-277
    return detail::scan_impl(a, input, nullptr);
}

// Occurrence count (:280-282).
inline std::size_t match_count(std::span<const MatchRecord> records) noexcept { return records.size(); }

}  // namespace acmatch
