// ORACLE — test infrastructure, NOT the product.
//
// A C-ABI shim over the UNMODIFIED reference headers, compiled by
// oracle/Makefile from the sources where they lie under
// /root/reference/proj/{include,tests} into oracle/_ref/libacref.so.
// Used by the tests (to pin oracle/ac_oracle.c), by oracle/make_goldens.py
// (golden fixtures) and by bench.py --impl reference / cpu_baseline (the
// reference's own CPU scan timed on the host cores). No reference source is
// copied into this repository; this file only #includes it.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <sstream>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "acmatch/aho_corasick.hpp"
#include "acmatch/io.hpp"
#include "acmatch/partition.hpp"
#include "support/oracle.hpp"

using acmatch::Automaton;
using acmatch::MatchRecord;
using acmatch::Pattern;

namespace {

std::vector<Pattern> to_patterns(const std::uint8_t* concat, const std::uint64_t* offs, std::uint32_t count) {
    std::vector<Pattern> p;
    p.reserve(count);
    for (std::uint32_t i = 0; i < count; ++i)
        p.push_back(Pattern{i, std::string(reinterpret_cast<const char*>(concat) + offs[i], offs[i + 1] - offs[i])});
    return p;
}

int error_code(const std::exception& e) {
    if (dynamic_cast<const acmatch::EmptyDictionaryError*>(&e)) return 1;
    if (dynamic_cast<const acmatch::EmptyPatternError*>(&e)) return 2;
    if (dynamic_cast<const acmatch::InvalidWorkerCountError*>(&e)) return 4;
    return 3;
}

inline std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct Prepared {
    std::vector<std::vector<std::uint32_t>> chunks;
    std::vector<Automaton> machines;
};

}  // namespace

extern "C" {

int ref_build(const std::uint8_t* concat, const std::uint64_t* offs, std::uint32_t count, void** out) {
    *out = nullptr;
    try {
        *out = new Automaton(acmatch::build(to_patterns(concat, offs, count)));
        return 0;
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

void ref_free(void* h) { delete static_cast<Automaton*>(h); }

std::uint32_t ref_state_count(void* h) { return static_cast<std::uint32_t>(static_cast<Automaton*>(h)->state_count()); }
std::uint32_t ref_failure(void* h, std::uint32_t s) { return static_cast<Automaton*>(h)->failure(s); }
std::uint32_t ref_depth(void* h, std::uint32_t s) { return static_cast<Automaton*>(h)->depth(s); }
std::uint32_t ref_next_state(void* h, std::uint32_t s, std::uint8_t b) {
    return acmatch::next_state(*static_cast<Automaton*>(h), s, b);
}
int ref_goto(void* h, std::uint32_t s, std::uint8_t b, std::uint32_t* to) {
    const auto t = static_cast<Automaton*>(h)->goto_transition(s, b);
    if (t) *to = *t;
    return t.has_value();
}
std::uint32_t ref_outputs(void* h, std::uint32_t s, std::uint32_t* ids, std::uint32_t cap) {
    const auto o = static_cast<Automaton*>(h)->outputs(s);
    for (std::size_t i = 0; i < o.size() && i < cap; ++i) ids[i] = o[i];
    return static_cast<std::uint32_t>(o.size());
}
std::uint32_t ref_transitions(void* h, std::uint32_t s, std::uint8_t* bytes, std::uint32_t* to, std::uint32_t cap) {
    const auto e = static_cast<Automaton*>(h)->transitions(s);
    for (std::size_t i = 0; i < e.size() && i < cap; ++i) {
        bytes[i] = e[i].first;
        to[i] = e[i].second;
    }
    return static_cast<std::uint32_t>(e.size());
}

// The whole machine through the public accessors (aho_corasick.hpp:77-101),
// as CSR arrays: sizes first (any output pointer null), then the copy.
void ref_export(void* h, std::uint64_t* sizes, std::uint32_t* fail, std::uint32_t* depth, std::uint32_t* edge_off,
                std::uint8_t* edge_byte, std::uint32_t* edge_to, std::uint32_t* out_off, std::uint32_t* out_ids) {
    const Automaton& a = *static_cast<Automaton*>(h);
    const auto S = static_cast<std::uint32_t>(a.state_count());
    std::uint64_t ne = 0, no = 0;
    for (std::uint32_t s = 0; s < S; ++s) {
        ne += a.transitions(s).size();
        no += a.outputs(s).size();
    }
    sizes[0] = S;
    sizes[1] = ne;
    sizes[2] = no;
    if (!fail) return;
    std::uint32_t e = 0, o = 0;
    for (std::uint32_t s = 0; s < S; ++s) {
        fail[s] = a.failure(s);
        depth[s] = a.depth(s);
        edge_off[s] = e;
        for (const auto& [b, t] : a.transitions(s)) {
            edge_byte[e] = b;
            edge_to[e++] = t;
        }
        out_off[s] = o;
        for (const auto id : a.outputs(s)) out_ids[o++] = id;
    }
    edge_off[S] = e;
    out_off[S] = o;
}

// acmatch::load_patterns (include/acmatch/io.hpp:37-65): 0 ok (sizes first with
// null outputs), 9 IoError, 1 EmptyDictionaryError.
int ref_load_patterns(const char* path, std::uint64_t* sizes, std::uint8_t* concat, std::uint64_t* offs) {
    try {
        const acmatch::PatternFile f = acmatch::load_patterns(path);
        std::uint64_t total = 0;
        for (const auto& p : f.patterns) total += p.bytes.size();
        sizes[0] = f.patterns.size();
        sizes[1] = total;
        sizes[2] = f.duplicates;
        sizes[3] = f.skipped_empty;
        if (concat) {
            std::uint64_t o = 0;
            offs[0] = 0;
            for (std::size_t i = 0; i < f.patterns.size(); ++i) {
                std::memcpy(concat + o, f.patterns[i].bytes.data(), f.patterns[i].bytes.size());
                o += f.patterns[i].bytes.size();
                offs[i + 1] = o;
            }
        }
        return 0;
    } catch (const acmatch::IoError&) {
        return 9;
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

// acmatch::load_input (include/acmatch/io.hpp:25-31): bytes copied when out is non-null.
int ref_load_input(const char* path, std::uint64_t* n, std::uint8_t* out) {
    try {
        const std::string s = acmatch::load_input(path);
        *n = s.size();
        if (out) std::memcpy(out, s.data(), s.size());
        return 0;
    } catch (const acmatch::IoError&) {
        return 9;
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

// `acmatch match --output tsv` bytes for text[0, n): the reference scan, then
// cmd_match's TSV loop restated (proj/include/acmatch/cli.hpp:71-74; cli.hpp
// itself needs CLI11/nlohmann, absent here). Returns the size; copies when it fits.
std::uint64_t ref_match_tsv(void* h, const std::uint8_t* text, std::uint64_t n, std::uint8_t* out, std::uint64_t cap) {
    const Automaton& a = *static_cast<Automaton*>(h);
    const auto recs = acmatch::scan(a, std::string_view(reinterpret_cast<const char*>(text), n));
    std::ostringstream os;
    for (const MatchRecord& r : recs) os << r.end << '\t' << r.pattern_id << '\t' << a.patterns()[r.pattern_id].bytes << '\n';
    const std::string s = os.str();
    if (out && s.size() <= cap) std::memcpy(out, s.data(), s.size());
    return s.size();
}

// acmatch::scan (include/acmatch/aho_corasick.hpp:250-272) over text[0, n).
std::uint64_t ref_scan(void* h, const std::uint8_t* text, std::uint64_t n, std::uint64_t* follows,
                       std::uint32_t* ids, std::uint64_t* ends, std::uint64_t cap) {
    acmatch::ScanStats st;
    const auto recs = acmatch::scan(*static_cast<Automaton*>(h),
                                    std::string_view(reinterpret_cast<const char*>(text), n), st);
    if (follows) *follows = st.failure_follows;
    for (std::size_t i = 0; i < recs.size() && i < cap; ++i) {
        ids[i] = recs[i].pattern_id;
        ends[i] = recs[i].end;
    }
    return recs.size();
}

// Windowed reference scan for golden statistics: the reference scan of
// text[0, n) (from the root), keeping records with end >= emit_from. The
// window starts at absolute offset abs_base of the whole text; digest keys use
// absolute ends (key = (abs_base + end)*2^20 + id). Accumulates per-pattern
// counts, the record count, the order-independent digest and the failure
// follows of the steps at positions >= emit_from. Also verifies (end, id)
// strict order. Returns 0, or 5 if the output was not strictly increasing.
int ref_window_digest(void* h, const std::uint8_t* text, std::uint64_t n, std::uint64_t emit_from,
                      std::uint64_t abs_base, std::uint64_t* counts, std::uint64_t* m, std::uint64_t* dsum,
                      std::uint64_t* dxor, std::uint64_t* follows) {
    const Automaton& a = *static_cast<Automaton*>(h);
    const char* base = reinterpret_cast<const char*>(text);
    acmatch::ScanStats all, pre;
    const auto recs = acmatch::scan(a, std::string_view(base, n), all);
    if (emit_from > 0) (void)acmatch::scan(a, std::string_view(base, emit_from), pre);
    *follows += all.failure_follows - pre.failure_follows;
    int rc = 0;
    bool first = true;
    MatchRecord prev{};
    for (const MatchRecord& r : recs) {
        if (r.end < emit_from) continue;
        if (!first && !acmatch::match_before(prev, r)) rc = 5;
        prev = r;
        first = false;
        counts[r.pattern_id]++;
        const std::uint64_t k = mix64(((abs_base + r.end) << 20) + r.pattern_id);
        *dsum += k;
        *dxor ^= k;
        ++*m;
    }
    return rc;
}

// ref_window_digest over text[start, n) of a whole-text buffer.
int ref_scan_window_stats(void* h, const std::uint8_t* text, std::uint64_t n, std::uint64_t start,
                          std::uint64_t emit_from, std::uint64_t* counts, std::uint64_t* m,
                          std::uint64_t* dsum, std::uint64_t* dxor, std::uint64_t* follows) {
    return ref_window_digest(h, text + start, n - start, emit_from > start ? emit_from - start : 0, start, counts, m,
                             dsum, dxor, follows);
}

// acmatch::run_partitioned (include/acmatch/partition.hpp:108-170), as is.
int ref_run_partitioned(const std::uint8_t* concat, const std::uint64_t* offs, std::uint32_t count,
                        const std::uint8_t* text, std::uint64_t n, std::uint32_t workers, std::uint32_t* ids,
                        std::uint64_t* ends, std::uint64_t cap, std::uint64_t* m, double* wall_s,
                        std::uint32_t* launched) {
    try {
        const auto run = acmatch::run_partitioned(to_patterns(concat, offs, count),
                                                  std::string_view(reinterpret_cast<const char*>(text), n), workers);
        *m = run.matches.size();
        for (std::size_t i = 0; i < run.matches.size() && i < cap; ++i) {
            ids[i] = run.matches[i].pattern_id;
            ends[i] = run.matches[i].end;
        }
        if (wall_s) *wall_s = run.total_wall_s;
        if (launched) *launched = run.workers_launched;
        return 0;
    } catch (const std::exception& e) {
        return error_code(e);
    }
}

// run_partitioned with the per-worker builds hoisted out of the timed region:
// prepare = split_patterns + one reference build per non-empty chunk
// (partition.hpp:113, :132-136); scan = one std::thread per machine running
// the reference scan over the whole input, the id remap (:142) and the
// reference k-way merge_matches (:167). This is the reference's only parallel
// mode with the automata already built, i.e. the same boundary the GPU path
// is timed at.
void* ref_partitioned_prepare(const std::uint8_t* concat, const std::uint64_t* offs, std::uint32_t count,
                              std::uint32_t workers) {
    try {
        const auto patterns = to_patterns(concat, offs, count);
        const auto plan = acmatch::split_patterns(patterns, workers);
        auto* p = new Prepared;
        for (const auto& chunk : plan.chunks) {
            if (chunk.empty()) continue;
            std::vector<Pattern> local;
            for (std::size_t j = 0; j < chunk.size(); ++j)
                local.push_back(Pattern{static_cast<std::uint32_t>(j), patterns[chunk[j]].bytes});
            p->chunks.push_back(chunk);
            p->machines.push_back(acmatch::build(std::move(local)));
        }
        return p;
    } catch (...) {
        return nullptr;
    }
}

double ref_partitioned_scan(void* h, const std::uint8_t* text, std::uint64_t n, std::uint64_t* m) {
    auto* p = static_cast<Prepared*>(h);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::vector<MatchRecord>> lists(p->machines.size());
    std::vector<std::thread> threads;
    const std::string_view input(reinterpret_cast<const char*>(text), n);
    for (std::size_t k = 0; k < p->machines.size(); ++k)
        threads.emplace_back([&, k] {
            lists[k] = acmatch::scan(p->machines[k], input);
            for (MatchRecord& r : lists[k]) r.pattern_id = p->chunks[k][r.pattern_id];
        });
    for (auto& t : threads) t.join();
    const auto merged = acmatch::merge_matches(lists);
    *m = merged.size();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

std::uint32_t ref_partitioned_workers(void* h) {
    return static_cast<std::uint32_t>(static_cast<Prepared*>(h)->machines.size());
}

void ref_partitioned_free(void* h) { delete static_cast<Prepared*>(h); }

// testsupport's randomised trial (tests/acceptance/acceptance_main.cpp:120-126):
// random_dictionary(rng, max_count, min_len, max_len) then random_input(rng,
// max_input). Used to pin the oracle's mt19937_64 replay.
std::uint32_t ref_random_trial(std::uint64_t seed, std::uint32_t max_count, std::uint32_t min_len,
                               std::uint32_t max_len, std::uint64_t max_input, std::uint8_t* concat,
                               std::uint64_t* offs, std::uint8_t* text, std::uint64_t* text_len) {
    std::mt19937_64 rng(seed);
    const auto patterns = testsupport::random_dictionary(rng, max_count, min_len, max_len);
    const std::string input = testsupport::random_input(rng, max_input);
    offs[0] = 0;
    for (std::size_t i = 0; i < patterns.size(); ++i) {
        std::memcpy(concat + offs[i], patterns[i].bytes.data(), patterns[i].bytes.size());
        offs[i + 1] = offs[i] + patterns[i].bytes.size();
    }
    std::memcpy(text, input.data(), input.size());
    *text_len = input.size();
    return static_cast<std::uint32_t>(patterns.size());
}

// testsupport::naive_find_all (tests/support/oracle.hpp:31-43).
std::uint64_t ref_naive_find_all(const std::uint8_t* concat, const std::uint64_t* offs, std::uint32_t count,
                                 const std::uint8_t* text, std::uint64_t n, std::uint32_t* ids, std::uint64_t* ends,
                                 std::uint64_t cap) {
    const auto recs = testsupport::naive_find_all(to_patterns(concat, offs, count),
                                                  std::string_view(reinterpret_cast<const char*>(text), n));
    for (std::size_t i = 0; i < recs.size() && i < cap; ++i) {
        ids[i] = recs[i].pattern_id;
        ends[i] = recs[i].end;
    }
    return recs.size();
}

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

}  // extern "C"
