// Host automaton build (reference algorithm) and dense-DFA compilation.
#include "automaton.hpp"
#include "parallel.hpp"
#include "ctab.hpp"
#include "qfilter.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

namespace acg {

bool Nfa::goto_transition(StateId s, std::uint8_t b, StateId* out) const {
    // sorted-edge binary search: aho_corasick.hpp:67-74
    const std::uint8_t* lo = edge_byte.data() + edge_off[s];
    const std::uint8_t* hi = edge_byte.data() + edge_off[s + 1];
    const std::uint8_t* it = std::lower_bound(lo, hi, b);
    if (it != hi && *it == b) {
        *out = edge_to[static_cast<std::size_t>(it - edge_byte.data())];
        return true;
    }
    return false;
}

StateId Nfa::next_state(StateId s, std::uint8_t b) const {
    // total transition: aho_corasick.hpp:238-245
    for (;;) {
        StateId t;
        if (goto_transition(s, b, &t)) return t;
        if (s == 0) return 0;
        s = fail[s];
    }
}

namespace {

using Clock = std::chrono::steady_clock;
const bool g_build_prof = [] {  // ACG_BUILD_PROFILE=1: phase times of the build on stderr
    const char* e = std::getenv("ACG_BUILD_PROFILE");
    return e && e[0] == '1';
}();
struct Phase {
    const char* what;
    Clock::time_point t0 = Clock::now();
    explicit Phase(const char* w) : what(w) {}
    void next(const char* w) {  // close this phase, open the next
        report();
        what = w;
        t0 = Clock::now();
    }
    void report() const {
        if (g_build_prof)
            std::fprintf(stderr, "[acg build] %-22s %8.2f ms\n", what,
                         std::chrono::duration<double, std::milli>(Clock::now() - t0).count());
    }
    ~Phase() { report(); }
};

}  // namespace

// The reference's build (aho_corasick.hpp:130-233) inserts the patterns one by
// one into a trie whose children keep insertion order, numbers the states in
// DFS preorder, then walks BFS to set failure links (a chain walk per edge)
// and suffix-closed output sets. The same machine is built here in bulk:
//  1. patterns sorted by (bytes, id) on the pool; one sweep over the sorted
//     list creates every distinct prefix (a trie node) in lexicographic order,
//     with the smallest pattern id through it (= its creation time under the
//     reference's id-order insertion: siblings are ordered by it);
//  2. subtree sizes, then DFS-preorder ids with children in creation order;
//     edges sorted by byte come for free from the lexicographic order;
//  3. BFS levels: within a level every state is independent, so the failure
//     link (delta(fail(parent), byte)), the dense transition row (the fail
//     state's row with the state's own edges), the follow counts and the
//     output-set sizes are computed in parallel; output sets are filled level
//     by level (a merge of the state's own ids with its fail state's set).
int build_nfa(const std::uint8_t* concat, const std::uint64_t* offs, std::uint32_t count, Nfa& nfa) {
    if (count == 0) return kErrEmptyDictionary;  // aho_corasick.hpp:131
    std::uint64_t total = 0;
    std::uint32_t max_len = 0, min_len = ~0u;
    for (std::uint32_t i = 0; i < count; ++i) {
        const std::uint64_t len = offs[i + 1] - offs[i];
        if (len == 0) return kErrEmptyPattern;  // :133-134
        total += len;
        max_len = std::max<std::uint32_t>(max_len, static_cast<std::uint32_t>(len));
        min_len = std::min<std::uint32_t>(min_len, static_cast<std::uint32_t>(len));
    }
    // states are u32 (StateId, aho_corasick.hpp:18): up to total + 1 of them
    if (total >= 0xFFFFFFF0ull) return kErrTooLarge;
    const std::uint8_t* const base = concat;
    auto pat = [&](std::uint32_t id) { return base + offs[id]; };
    auto plen = [&](std::uint32_t id) { return static_cast<std::uint32_t>(offs[id + 1] - offs[id]); };

    // ---- 1. sorted sweep: trie nodes in lexicographic preorder ------------
    std::vector<std::uint32_t> ord(count);
    {
        Phase ph("sort patterns");
        std::iota(ord.begin(), ord.end(), 0u);
        parallel_sort(ord, [&](std::uint32_t x, std::uint32_t y) {
            const std::uint32_t lx = plen(x), ly = plen(y);
            const int c = std::memcmp(pat(x), pat(y), std::min(lx, ly));
            if (c) return c < 0;
            if (lx != ly) return lx < ly;
            return x < y;
        });
    }
    std::vector<std::uint32_t> lpar, lmin, own_first, own_cnt;
    std::vector<std::uint8_t> lbyte;
    std::vector<std::uint32_t> ldepth;
    {
        Phase ph("trie sweep");
        const std::size_t guess = static_cast<std::size_t>(std::min<std::uint64_t>(total + 1, 1ull << 28));
        lpar.reserve(guess);
        lmin.reserve(guess);
        lbyte.reserve(guess);
        ldepth.reserve(guess);
        lpar.push_back(0);
        lmin.push_back(0);
        lbyte.push_back(0);
        ldepth.push_back(0);
        own_first.assign(1, ~0u);
        own_cnt.assign(1, 0);
        std::vector<std::uint32_t> path(static_cast<std::size_t>(max_len) + 1, 0);
        const std::uint8_t* prev = nullptr;
        std::uint32_t prev_len = 0;
        for (std::uint32_t k = 0; k < count; ++k) {
            const std::uint32_t id = ord[k], L = plen(id);
            const std::uint8_t* s = pat(id);
            std::uint32_t l = 0;
            const std::uint32_t lim = std::min(L, prev_len);
            if (prev)
                while (l < lim && s[l] == prev[l]) ++l;
            for (std::uint32_t d = 1; d <= l; ++d) lmin[path[d]] = std::min(lmin[path[d]], id);
            for (std::uint32_t d = l + 1; d <= L; ++d) {
                const auto t = static_cast<std::uint32_t>(lpar.size());
                lpar.push_back(path[d - 1]);
                lmin.push_back(id);
                lbyte.push_back(s[d - 1]);
                ldepth.push_back(d);
                path[d] = t;
            }
            const std::uint32_t term = path[L];
            if (term >= own_first.size()) {
                own_first.resize(lpar.size(), ~0u);
                own_cnt.resize(lpar.size(), 0);
            }
            if (own_cnt[term]++ == 0) own_first[term] = k;  // ids ascending (:165, :192)
            prev = s;
            prev_len = L;
        }
        own_first.resize(lpar.size(), ~0u);
        own_cnt.resize(lpar.size(), 0);
    }
    const auto n = static_cast<std::uint32_t>(lpar.size());

    // ---- 2. DFS preorder with children in creation order (:170-183) -------
    std::vector<std::uint32_t> kid_off(n + 1, 0), kids, id_of(n);
    {
        Phase ph("preorder numbering");
        for (std::uint32_t v = 1; v < n; ++v) ++kid_off[lpar[v] + 1];
        for (std::uint32_t v = 0; v < n; ++v) kid_off[v + 1] += kid_off[v];
        kids.resize(n ? n - 1 : 0);
        {
            std::vector<std::uint32_t> fill(kid_off.begin(), kid_off.end() - 1);
            for (std::uint32_t v = 1; v < n; ++v) kids[fill[lpar[v]]++] = v;  // byte order (lexicographic)
        }
        std::vector<std::uint32_t> size(n, 1);
        for (std::uint32_t v = n - 1; v >= 1; --v) size[lpar[v]] += size[v];
        id_of[0] = 0;
        std::vector<std::uint32_t> tmp;
        for (std::uint32_t v = 0; v < n; ++v) {
            const std::uint32_t k0 = kid_off[v], k1 = kid_off[v + 1];
            std::uint32_t next = id_of[v] + 1;
            if (k1 - k0 == 1) {
                id_of[kids[k0]] = next;
                continue;
            }
            tmp.assign(kids.begin() + k0, kids.begin() + k1);
            std::sort(tmp.begin(), tmp.end(), [&](std::uint32_t x, std::uint32_t y) { return lmin[x] < lmin[y]; });
            for (const std::uint32_t c : tmp) {
                id_of[c] = next;
                next += size[c];
            }
        }
    }

    // ---- freeze: per-state edges sorted by byte (:185-196) ----------------
    std::vector<std::uint32_t> par(n), own_lo(n), own_n(n);
    std::vector<std::uint8_t> in_byte(n);
    {
        Phase ph("edges");
        nfa.edge_off.assign(static_cast<std::size_t>(n) + 1, 0);
        nfa.depth.assign(n, 0);
        for (std::uint32_t v = 0; v < n; ++v) nfa.edge_off[id_of[v] + 1] = kid_off[v + 1] - kid_off[v];
        for (std::uint32_t s = 0; s < n; ++s) nfa.edge_off[s + 1] += nfa.edge_off[s];
        nfa.edge_byte.resize(n - 1);
        nfa.edge_to.resize(n - 1);
        parallel_for(n, 1 << 14, [&](std::size_t lo, std::size_t hi) {
            for (std::size_t v = lo; v < hi; ++v) {
                const std::uint32_t s = id_of[v];
                nfa.depth[s] = ldepth[v];
                par[s] = id_of[lpar[v]];
                in_byte[s] = lbyte[v];
                own_lo[s] = own_first[v];
                own_n[s] = own_cnt[v];
                std::uint32_t e = nfa.edge_off[s];
                for (std::uint32_t k = kid_off[v]; k < kid_off[v + 1]; ++k, ++e) {
                    nfa.edge_byte[e] = lbyte[kids[k]];
                    nfa.edge_to[e] = id_of[kids[k]];
                }
            }
        });
    }
    // (lexicographic scratch no longer needed)
    std::vector<std::uint32_t>().swap(lpar);
    std::vector<std::uint32_t>().swap(lmin);
    std::vector<std::uint32_t>().swap(kids);

    // ---- alphabet: the symbol classes of the dense image -------------------
    {
        bool used[256] = {};
        for (std::uint32_t s = 1; s < n; ++s) used[in_byte[s]] = true;
        std::uint32_t n_sym = 0;
        bool dna = true;
        for (int b = 0; b < 256; ++b) {
            n_sym += used[b];
            if (used[b] && b != 'A' && b != 'C' && b != 'G' && b != 'T') dna = false;
        }
        nfa.n_sym = n_sym;
        std::memset(nfa.symmap, 0, sizeof nfa.symmap);
        if (dna) {
            nfa.mode = kAlphaDna4;
            nfa.K = 4;
            nfa.col_byte = {'A', 'C', 'T', 'G'};  // column = (byte >> 1) & 3
            for (int c = 0; c < 4; ++c) nfa.symmap[nfa.col_byte[c]] = static_cast<std::uint8_t>(c);
        } else {
            nfa.mode = kAlphaGeneric;
            nfa.K = n_sym + 1;
            nfa.col_byte.clear();
            std::uint32_t c = 0;
            for (int b = 0; b < 256; ++b)
                if (used[b]) {
                    nfa.symmap[b] = static_cast<std::uint8_t>(c++);
                    nfa.col_byte.push_back(b);
                }
            for (int b = 0; b < 256; ++b)
                if (!used[b]) nfa.symmap[b] = static_cast<std::uint8_t>(n_sym);  // escape column
            nfa.col_byte.push_back(-1);
        }
    }
    const std::uint32_t K = nfa.K;
    int col_of[256];
    std::fill(std::begin(col_of), std::end(col_of), -1);
    for (std::uint32_t c = 0; c < K; ++c)
        if (nfa.col_byte[c] >= 0) col_of[nfa.col_byte[c]] = static_cast<int>(c);

    // ---- 3. BFS levels: failure links, dense rows, follows, output sizes ---
    nfa.bfs.assign(1, 0);
    nfa.bfs.reserve(n);
    std::vector<std::uint32_t> level_at{0, 1};
    {
        Phase ph("bfs order");
        for (std::size_t head = 0; head < nfa.bfs.size(); ++head) {
            const std::uint32_t u = nfa.bfs[head];
            for (std::uint32_t j = nfa.edge_off[u]; j < nfa.edge_off[u + 1]; ++j) nfa.bfs.push_back(nfa.edge_to[j]);
            if (head + 1 == level_at.back() && nfa.bfs.size() > level_at.back())
                level_at.push_back(static_cast<std::uint32_t>(nfa.bfs.size()));
        }
    }
    nfa.fail.assign(n, 0);
    nfa.delta.assign(static_cast<std::size_t>(n) * K, 0u);
    nfa.fol.assign(static_cast<std::size_t>(n) * K, 0);
    nfa.fesc.assign(n, 0);
    std::vector<std::uint32_t> olen(n, 0);
    auto own_edges = [&](std::uint32_t s) {
        const std::size_t row = static_cast<std::size_t>(s) * K;
        for (std::uint32_t j = nfa.edge_off[s]; j < nfa.edge_off[s + 1]; ++j) {
            const int c = col_of[nfa.edge_byte[j]];
            nfa.delta[row + c] = nfa.edge_to[j];
            nfa.fol[row + c] = 0;
        }
    };
    {
        Phase ph("levels: fail + rows");
        own_edges(0);  // root: its own edges, every other column stays at the root, no follows
        for (std::size_t L = 1; L + 1 < level_at.size(); ++L) {
            const std::uint32_t l0 = level_at[L], l1 = level_at[L + 1];
            parallel_for(l1 - l0, 4096, [&](std::size_t lo, std::size_t hi) {
                for (std::size_t i = l0 + lo; i < l0 + hi; ++i) {
                    const std::uint32_t s = nfa.bfs[i], p = par[s];
                    // fail(child of p by b) = next_state(fail(p), b) (:205-215)
                    const std::uint32_t f =
                        p == 0 ? 0u : nfa.delta[static_cast<std::size_t>(nfa.fail[p]) * K + col_of[in_byte[s]]];
                    nfa.fail[s] = f;
                    const std::size_t row = static_cast<std::size_t>(s) * K, frow = static_cast<std::size_t>(f) * K;
                    for (std::uint32_t c = 0; c < K; ++c) {
                        nfa.delta[row + c] = nfa.delta[frow + c];
                        const std::uint32_t v = 1u + nfa.fol[frow + c];  // one failure link, then retry
                        nfa.fol[row + c] = static_cast<std::uint16_t>(std::min<std::uint32_t>(v, 0xFFFF));
                    }
                    own_edges(s);
                    nfa.fesc[s] = static_cast<std::uint16_t>(std::min<std::uint32_t>(1u + nfa.fesc[f], 0xFFFF));
                    olen[s] = own_n[s] + olen[f];  // own ids and out(fail(s)) are disjoint (:219-225)
                }
            });
        }
    }
    {
        Phase ph("levels: outputs");
        nfa.out_off.assign(static_cast<std::size_t>(n) + 1, 0);
        for (std::uint32_t s = 0; s < n; ++s) nfa.out_off[s + 1] = nfa.out_off[s] + olen[s];
        nfa.out_ids.resize(nfa.out_off[n]);
        for (std::size_t L = 1; L + 1 < level_at.size(); ++L) {
            const std::uint32_t l0 = level_at[L], l1 = level_at[L + 1];
            parallel_for(l1 - l0, 4096, [&](std::size_t lo, std::size_t hi) {
                for (std::size_t i = l0 + lo; i < l0 + hi; ++i) {
                    const std::uint32_t s = nfa.bfs[i];
                    if (!olen[s]) continue;
                    const std::uint32_t f = nfa.fail[s];
                    const std::uint32_t* own = ord.data() + (own_n[s] ? own_lo[s] : 0);
                    std::merge(own, own + own_n[s], nfa.out_ids.begin() + nfa.out_off[f],
                               nfa.out_ids.begin() + nfa.out_off[f] + olen[f], nfa.out_ids.begin() + nfa.out_off[s]);
                }
            });
        }
    }

    // dense root row (:230-231)
    std::fill(std::begin(nfa.root_row), std::end(nfa.root_row), 0u);
    for (std::uint32_t j = nfa.edge_off[0]; j < nfa.edge_off[1]; ++j) nfa.root_row[nfa.edge_byte[j]] = nfa.edge_to[j];
    nfa.n_patterns = count;
    nfa.max_len = max_len;
    nfa.min_len = min_len;
    nfa.pat_bytes.assign(concat, concat + offs[count]);
    nfa.pat_off.assign(offs, offs + count + 1);
    for (auto& o : nfa.pat_off) o -= offs[0];
    (void)base;
    return kOk;
}

namespace {

// The q-gram prefilter (qfilter.hpp): every pattern's q-grams at offsets
// 0..kQSample-1 into the blocked Bloom filter and the exact (code -> (pattern,
// offset) list) hash table.
void compile_qfilter(const Nfa& nfa, Dfa& d) {
    Phase ph_all("compile_qfilter");
    d.filter_ok = false;
    d.qbm = false;
    d.qbloom.clear();
    d.qbloom2.clear();
    d.qtab.clear();
    d.qb_off.clear();
    d.qb_ent.clear();
    if (d.mode != kAlphaDna4 || nfa.min_len < kQMinQ + kQSample - 1) return;
    if (nfa.pat_bytes.size() >= (1ull << 32) || nfa.n_patterns >= (1u << 30)) return;
    const std::uint32_t q = std::min(kQMaxQ, nfa.min_len - (kQSample - 1));
    const std::uint32_t qm = q >= 16 ? 0xFFFFFFFFu : (1u << (2 * q)) - 1u;
    d.q = q;
    // (code, pattern << 2 | offset), grouped by code
    std::vector<std::pair<std::uint32_t, std::uint32_t>> grams;
    grams.reserve(static_cast<std::size_t>(nfa.n_patterns) * kQSample);
    for (std::uint32_t p = 0; p < nfa.n_patterns; ++p) {
        const std::uint8_t* b = nfa.pat_bytes.data() + nfa.pat_off[p];
        for (std::uint32_t o = 0; o < kQSample; ++o) {
            std::uint32_t c = 0;
            for (std::uint32_t k = 0; k < q; ++k) c |= ((static_cast<std::uint32_t>(b[o + k]) >> 1) & 3u) << (2 * k);
            grams.emplace_back(c, (p << 2) | o);
        }
    }
    Phase ph_g("  grams sort+tables");
    parallel_sort(grams, [](const std::pair<std::uint32_t, std::uint32_t>& x, const std::pair<std::uint32_t, std::uint32_t>& y) { return x < y; });
    ph_g.next("  bloom level 1");
    std::uint32_t keys = 0;
    for (std::size_t i = 0; i < grams.size(); ++i) keys += !i || grams[i].first != grams[i - 1].first;
    // level 1: a bitmap of the keys' 10-gram prefixes for dictionaries it keeps
    // selective (qfilter.hpp), with the Bloom filter of the full q-grams after it;
    // else the Bloom filter alone in all of shared memory
    // Off by default (ACG_QBITMAP=1 turns it on): on cfg1 it halves the
    // survivors (V1 24.6 -> 18.5 us) but KQ runs 0.242 ms against 0.226 with the
    // Bloom filter alone — the lanes' level-1 hits (3.8 % of samples) make the
    // level-2 probes a divergent loop of dependent hash/LDS chains.
    static const bool bm_on = [] {
        const char* e = std::getenv("ACG_QBITMAP");
        return e && e[0] == '1';
    }();
    d.qbm = bm_on && q >= 10 && keys <= kQBitmapMaxKeys;
    std::uint32_t words = d.qbm ? kQWordsBM : kQWords;
    if (const char* e = std::getenv("ACG_QWORDS")) {  // experiments only (Bloom size sweeps)
        const long v = std::strtol(e, nullptr, 10);
        if (!d.qbm && v >= 1024 && v <= 57344) words = static_cast<std::uint32_t>(v) & ~3u;
    }
    std::vector<std::uint32_t> bloom(words, 0u), bitmap(d.qbm ? kQBitmapWords : 0u, 0u);
    for (std::size_t i = 0; i < grams.size(); ++i) {
        if (i && grams[i].first == grams[i - 1].first) continue;
        const std::uint32_t h = qhash(qtop(grams[i].first, q));
        bloom[qword(h, words)] |= qmask(h);
        if (d.qbm) {
            const std::uint32_t idx = grams[i].first & 0xFFFFFu;  // bases 0..9 (2 bits each)
            bitmap[idx >> 5] |= 1u << (idx & 31);
        }
    }
    // the shared-memory image the KQ kernel stages: [bitmap | Bloom] or [Bloom]
    d.qbloom = bitmap;
    d.qbloom.insert(d.qbloom.end(), bloom.begin(), bloom.end());
    ph_g.next("  q-gram table");
    // load factor <= 1/4: a random (non-key) code ends its probe in ~1.4 slots
    d.qtab_bits = 10;
    while (d.qtab_bits < 28 && (1ull << d.qtab_bits) < 4ull * keys) ++d.qtab_bits;
    d.qtab.assign(2ull << d.qtab_bits, kQEmpty);
    d.qb_off.reserve(keys + 1);
    d.qb_ent.reserve(grams.size());
    for (std::size_t i = 0; i < grams.size();) {
        const std::uint32_t c = grams[i].first;
        std::uint32_t slot = qslot(c, d.qtab_bits);
        while (d.qtab[2 * slot + 1] != kQEmpty) slot = (slot + 1) & ((1u << d.qtab_bits) - 1);
        d.qtab[2 * slot] = c;
        d.qtab[2 * slot + 1] = static_cast<std::uint32_t>(d.qb_off.size());
        d.qb_off.push_back(static_cast<std::uint32_t>(d.qb_ent.size()));
        const std::size_t first = i;
        for (; i < grams.size() && grams[i].first == c; ++i) d.qb_ent.push_back(grams[i].second);
        // a one-entry bucket is stored in the slot itself (one dependent load less)
        if (i - first == 1 && grams[first].second < 0x7FFFFFFFu) d.qtab[2 * slot + 1] = kQSingle | grams[first].second;
    }
    d.qb_off.push_back(static_cast<std::uint32_t>(d.qb_ent.size()));
    ph_g.next("  pattern codes");
    d.pat_off32.assign(nfa.pat_off.begin(), nfa.pat_off.end());
    d.pat_code.assign(2ull * nfa.n_patterns, 0ull);
    parallel_for(nfa.n_patterns, 8192, [&](std::size_t p0, std::size_t p1) {
        for (std::size_t p = p0; p < p1; ++p) {
            const std::uint64_t lo = nfa.pat_off[p];
            const std::uint32_t len = static_cast<std::uint32_t>(std::min<std::uint64_t>(nfa.pat_off[p + 1] - lo, 64));
            for (std::uint32_t k = 0; k < len; ++k)
                d.pat_code[2 * p + k / 32] |= static_cast<std::uint64_t>((nfa.pat_bytes[lo + k] >> 1) & 3u) << (2 * (k % 32));
        }
    });
    // pass rates of random q-grams (splitmix64 sample), level 1 and overall
    auto pass_rates = [&](double& fp1, double& fp) {
        const std::uint32_t trials = 1u << 20, pieces = 64;
        const std::uint32_t words2 = static_cast<std::uint32_t>(d.qbloom2.size());
        std::vector<std::uint64_t> c1(pieces, 0), c2(pieces, 0);
        parallel_for(pieces, 1, [&](std::size_t k0, std::size_t k1) {
          for (std::size_t piece = k0; piece < k1; ++piece) {
            std::uint64_t& p1 = c1[piece];
            std::uint64_t& p2 = c2[piece];
            for (std::uint32_t t = static_cast<std::uint32_t>(piece) * (trials / pieces);
                 t < static_cast<std::uint32_t>(piece + 1) * (trials / pieces); ++t) {
            std::uint64_t r = 0x14037294ull + (static_cast<std::uint64_t>(t) + 1) * 0x9E3779B97F4A7C15ull;
            r = (r ^ (r >> 30)) * 0xBF58476D1CE4E5B9ull;
            r = (r ^ (r >> 27)) * 0x94D049BB133111EBull;
            const std::uint32_t c = static_cast<std::uint32_t>(r ^ (r >> 31)) & qm;
            const std::uint32_t h = qhash(qtop(c, q));
            const std::uint32_t m = qmask(h);
            if (d.qbm) {
                const std::uint32_t idx = c & 0xFFFFFu;
                if (!(bitmap[idx >> 5] >> (idx & 31) & 1u)) continue;
                ++p1;
                p2 += (bloom[qword(h, words)] & m) == m;
                continue;
            }
            if ((bloom[qword(h, words)] & m) != m) continue;
            ++p1;
            if (!words2) {
                ++p2;
                continue;
            }
            p2 += (d.qbloom2[qword(qhash2(h), words2)] & m) == m;  // level 2: its own word, level 1's mask
            }
          }
        });
        std::uint64_t p1 = 0, p2 = 0;
        for (std::uint32_t k = 0; k < pieces; ++k) p1 += c1[k], p2 += c2[k];
        fp1 = static_cast<double>(p1) / trials;
        fp = static_cast<double>(p2) / trials;
    };
    {
        Phase ph("  filter pass rates");
        pass_rates(d.filter_fp1, d.filter_fp);
    }
    ph_g.next("  level 2");
    if (!d.qbm && d.filter_fp > 5e-3 && d.filter_fp1 <= kQLevel1Max) {
        // level 2: ~1.5 % of its bits set (4 bits per key)
        std::uint64_t w2 = (static_cast<std::uint64_t>(keys) * 4 * 100 / 3 / 32 + 3) & ~3ull;
        w2 = std::min<std::uint64_t>(std::max<std::uint64_t>(w2, 1024), 16ull << 20);
        d.qbloom2.assign(w2, 0u);
        for (std::size_t i = 0; i < grams.size(); ++i) {
            if (i && grams[i].first == grams[i - 1].first) continue;
            const std::uint32_t h = qhash(qtop(grams[i].first, q));
            d.qbloom2[qword(qhash2(h), static_cast<std::uint32_t>(w2))] |= qmask(h);
        }
        pass_rates(d.filter_fp1, d.filter_fp);
    }
    // worth it when few samples survive (each survivor costs an exact probe)
    d.filter_ok = d.filter_fp <= 5e-3;
    if (!d.filter_ok) {
        d.qbm = false;
        d.pat_code.clear();
        d.qbloom2.clear();
        d.qbloom.clear();
        d.qtab.clear();
        d.qb_off.clear();
        d.qb_ent.clear();
    }
}

}  // namespace


// Compressed hot automaton (ctab.hpp): T_D default table + row-displaced
// exception entries of the hottest states, sized for `budget` bytes of shared
// memory. Leaves d.ctab empty when the scheme does not apply.
static void compile_ctab(const Nfa& nfa, const std::vector<std::uint32_t>& hot_order, std::size_t budget, Dfa& d,
                         std::uint32_t hot_limit, const std::vector<std::uint64_t>* visits) {
    d.ctab.clear();
    d.ct_rank.clear();
    d.ct_sw.clear();
    d.ct_next.clear();
    d.ct_slots = d.ct_D = d.ct_hot = 0;
    d.ct_deep = false;
    d.ct_cnt = false;
    const std::uint32_t S = d.S, K = d.K;
    const std::uint32_t n_out = d.Cn - d.Hn;
    if (d.mode != kAlphaGeneric || K > kCtMaxK || K < 2 || S <= d.H) return;  // (all states in the dense hot rows: KE has no cold steps)
    if (S >= kCtValMask || n_out >= kCtNoRank) return;
    const std::uint32_t D = (static_cast<std::uint64_t>(K) * K * K * 4 <= kCtDefaultMaxBytes) ? 3u : 2u;
    std::uint32_t nd = 1;
    for (std::uint32_t i = 0; i < D; ++i) nd *= K;
    if (budget < static_cast<std::size_t>(nd) * 4 + 64 * K * 4) return;
    const std::uint32_t slots =
        static_cast<std::uint32_t>(std::min<std::size_t>((budget - static_cast<std::size_t>(nd) * 4) / 4 & ~std::size_t(3), 0xFFF0u));
    if (slots + n_out >= kCtValMask) return;
    const std::vector<std::uint32_t>& delta = nfa.delta;
    auto has_out = [&](std::uint32_t s) { return nfa.out_off[s + 1] > nfa.out_off[s]; };
    const std::uint32_t max_ids = slots - K + 1;
    std::vector<std::uint32_t> masks, id_of, order_nfa;
    bool deep = false;
    // exception columns of state s as a bit mask. Plain: targets deeper than D.
    // Deep (the default itself takes one more level from the table, ctab.hpp):
    // targets deeper than D + 1, plus the depth-(D+1) children of depth-D states.
    auto exc_mask = [&](std::uint32_t s) {
        std::uint32_t m = 0;
        const std::size_t row = static_cast<std::size_t>(s) * K;
        const std::uint32_t ds = nfa.depth[s];
        for (std::uint32_t c = 0; c < K; ++c) {
            const std::uint32_t dt = nfa.depth[delta[row + c]];
            if (deep ? (dt > D + 1 || (dt == D + 1 && ds == D)) : dt > D) m |= 1u << c;
        }
        return m;
    };
    auto try_place = [&](std::size_t n_hot) -> bool {
        // first-fit row displacement, largest rows first (occupancy and id bitsets)
        std::vector<std::uint64_t> occ((slots + 64 + 63) / 64 + 1, 0), idu((slots + 63) / 64 + 1, 0);
        std::vector<std::uint32_t> order(n_hot);
        for (std::size_t i = 0; i < n_hot; ++i) order[i] = static_cast<std::uint32_t>(i);
        std::stable_sort(order.begin(), order.end(), [&](std::uint32_t x, std::uint32_t y) {
            return __builtin_popcount(masks[x]) > __builtin_popcount(masks[y]);
        });
        id_of.assign(n_hot, 0xFFFFFFFFu);
        std::uint32_t lo = 0;  // every slot below lo is occupied
        for (std::uint32_t i : order) {
            const std::uint32_t m = masks[i];
            if (!m) break;  // (sorted: the rest have no exceptions)
            const std::uint32_t c0 = static_cast<std::uint32_t>(__builtin_ctz(m));
            std::uint32_t b = lo > c0 ? lo - c0 : 0;
            bool placed = false;
            for (; b < max_ids; ++b) {
                const std::uint32_t w = b >> 6, sh = b & 63;
                const std::uint64_t win = sh ? (occ[w] >> sh) | (occ[w + 1] << (64 - sh)) : occ[w];
                if ((win & m) == 0 && !((idu[w] >> sh) & 1)) {
                    placed = true;
                    break;
                }
            }
            if (!placed) return false;
            id_of[i] = b;
            idu[b >> 6] |= 1ull << (b & 63);
            for (std::uint32_t mm = m; mm; mm &= mm - 1) {
                const std::uint32_t t = b + static_cast<std::uint32_t>(__builtin_ctz(mm));
                occ[t >> 6] |= 1ull << (t & 63);
            }
            while (lo < slots && ((occ[lo >> 6] >> (lo & 63)) & 1)) ++lo;
        }
        // states without exceptions: any id no row uses
        std::uint32_t b = 0;
        for (std::uint32_t i : order) {
            if (masks[i]) continue;
            while (b < max_ids && ((idu[b >> 6] >> (b & 63)) & 1)) ++b;
            if (b >= max_ids) return false;
            id_of[i] = b;
            idu[b >> 6] |= 1ull << (b & 63);
        }
        return true;
    };
    // the longest prefix of `order_nfa` whose exceptions fill at most `fill` of the slots and that places
    auto choose = [&](std::size_t must) -> std::size_t {
        for (double fill = 0.94; fill > 0.3; fill -= 0.06) {
            const std::uint64_t cap = static_cast<std::uint64_t>(fill * slots);
            std::uint64_t used = 0;
            std::size_t n_hot = 0;
            masks.clear();
            while (n_hot < S && n_hot < max_ids && (!hot_limit || n_hot < hot_limit)) {  // (hot_limit: diagnostics, cold paths)
                const std::uint32_t m = exc_mask(order_nfa[n_hot]);
                const std::uint32_t k = static_cast<std::uint32_t>(__builtin_popcount(m));
                if (used + k > cap) break;
                used += k;
                masks.push_back(m);
                ++n_hot;
            }
            if (n_hot < must) return 0;
            if (n_hot && try_place(n_hot)) return n_hot;
        }
        return 0;
    };
    // Plain default when a visit profile says its hot set takes >= 99.5 % of the
    // steps (3 loads per step; measured on cfg3: 4.27 ms per 2 GiB against 4.53
    // for the deep default's 4 loads); else the deep default, which holds far
    // more states (all of cfg3's): every state of depth <= D must then be hot
    // (their rows carry the default's extra level).
    std::size_t n_hot = 0;
    if (visits && visits->size() == S) {
        order_nfa = hot_order;
        n_hot = choose(1);
        unsigned long long in = 0, all = 0;
        for (std::size_t i = 0; i < S; ++i) {
            all += (*visits)[order_nfa[i]];
            if (i < n_hot) in += (*visits)[order_nfa[i]];
        }
        if (!n_hot || (n_hot < S && static_cast<double>(in) < 0.995 * static_cast<double>(all))) n_hot = 0;
    }
    if (!n_hot) {
        std::size_t shallow = 0;
        order_nfa.clear();
        order_nfa.reserve(S);
        for (std::uint32_t s : nfa.bfs) {
            if (nfa.depth[s] > D) break;
            order_nfa.push_back(s);
        }
        shallow = order_nfa.size();
        for (std::uint32_t s : hot_order)
            if (nfa.depth[s] > D) order_nfa.push_back(s);
        deep = true;
        n_hot = choose(shallow);
        if (!n_hot) {
            deep = false;
            order_nfa = hot_order;
            n_hot = choose(1);
        }
    }
    if (!n_hot) return;
    // counted words: the output count above a 17-bit payload (cold non-output words keep a plain device id)
    std::uint32_t max_out = 0;
    for (std::uint32_t s = 0; s < S; ++s) max_out = std::max(max_out, nfa.out_off[s + 1] - nfa.out_off[s]);
    // (S <= 2^16: a cold word without outputs carries its device id, whose byte 2 must stay 0 —
    // the walk sums the count byte of every owned step's word)
    const bool cnt = slots + n_out <= kCtPayMask && max_out < 255 && S <= (1u << kCtPayBits);
    auto out_bits = [&](std::uint32_t s) {
        return has_out(s) ? kCtOut | (cnt ? (nfa.out_off[s + 1] - nfa.out_off[s]) << kCtPayBits : 0u) : 0u;
    };
    // state words (device order) and the id -> rank table
    d.ct_sw.assign(S, 0);
    d.ct_rank.assign(slots, static_cast<std::uint16_t>(kCtNoRank));
    std::vector<std::uint32_t> sw_nfa(S);
    std::vector<std::uint8_t> is_hot(S, 0);
    for (std::size_t i = 0; i < n_hot; ++i) {
        const std::uint32_t s = order_nfa[i];
        is_hot[s] = 1;
        sw_nfa[s] = id_of[i] | out_bits(s);
        if (has_out(s)) d.ct_rank[id_of[i]] = static_cast<std::uint16_t>(d.dev_of[s] - d.Hn);
    }
    for (std::uint32_t s = 0; s < S; ++s) {
        if (!is_hot[s]) sw_nfa[s] = kCtCold | (has_out(s) ? out_bits(s) | (slots + d.dev_of[s] - d.Hn) : d.dev_of[s]);
        d.ct_sw[d.dev_of[s]] = sw_nfa[s];
    }
    d.ctab.assign(static_cast<std::size_t>(slots) + nd, kCtEmpty);
    for (std::size_t i = 0; i < n_hot; ++i) {
        const std::uint32_t s = order_nfa[i];
        const std::size_t row = static_cast<std::size_t>(s) * K;
        for (std::uint32_t mm = masks[i]; mm; mm &= mm - 1) {
            const std::uint32_t c = static_cast<std::uint32_t>(__builtin_ctz(mm));
            d.ctab[id_of[i] + c] = sw_nfa[delta[row + c]] | (c << kCtColShift);
        }
    }
    // T_D: index = sum_j col_{i-j} * K^j (the latest column is the lowest digit)
    for (std::uint32_t idx = 0; idx < nd; ++idx) {
        std::uint32_t cols[3], t = idx;
        for (std::uint32_t j = 0; j < D; ++j) {
            cols[j] = t % K;
            t /= K;
        }
        std::uint32_t st = 0;
        for (std::uint32_t j = D; j-- > 0;) st = delta[static_cast<std::size_t>(st) * K + cols[j]];
        d.ctab[slots + idx] = sw_nfa[st];
    }
    d.ct_next.resize(static_cast<std::size_t>(S) * K);
    parallel_for(S, 1 << 13, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo * K; i < hi * K; ++i) d.ct_next[i] = d.ct_sw[d.next[i]];
    });
    d.ct_slots = slots;
    d.ct_D = D;
    d.ct_hot = static_cast<std::uint32_t>(n_hot);
    d.ct_deep = deep;
    d.ct_cnt = cnt;
}

void compile_dfa(const Nfa& nfa, std::size_t hot_budget_bytes, const std::vector<std::uint64_t>* visits, Dfa& d,
                 std::uint32_t hot_limit, std::size_t ctab_budget_bytes) {
    Phase ph_all("compile_dfa (total)");
    Phase ph_ord("  hot order");
    const std::uint32_t S = nfa.state_count();
    // alphabet and dense rows come from the build (build_nfa: delta, fol, fesc)
    d.mode = nfa.mode;
    d.K = nfa.K;
    d.n_sym = nfa.n_sym;
    std::memcpy(d.symmap, nfa.symmap, sizeof d.symmap);
    const std::uint32_t K = d.K;
    d.S = S;
    const std::vector<std::uint32_t>& delta = nfa.delta;

    // Hotness order: BFS (shallow first), or visit counts on a text sample.
    std::vector<std::uint32_t> hot_order(nfa.bfs.begin(), nfa.bfs.end());
    if (visits && visits->size() == S) {
        std::vector<std::uint32_t> bfs_rank(S);
        for (std::uint32_t i = 0; i < S; ++i) bfs_rank[nfa.bfs[i]] = i;
        std::stable_sort(hot_order.begin(), hot_order.end(), [&](std::uint32_t a, std::uint32_t b) {
            if ((*visits)[a] != (*visits)[b]) return (*visits)[a] > (*visits)[b];
            return bfs_rank[a] < bfs_rank[b];
        });
        // keep the root first so it is always device id 0
        auto it = std::find(hot_order.begin(), hot_order.end(), 0u);
        std::rotate(hot_order.begin(), it, it + 1);
    }
    // (H+1) rows of K u16 entries (row H is the all-escape sink row)
    std::size_t H = hot_budget_bytes / (static_cast<std::size_t>(K) * 2);
    H = H > 1 ? H - 1 : 1;
    H = std::min<std::size_t>({H, S, 0x7FFEu});
    if (hot_limit) H = std::min<std::size_t>(H, hot_limit);
    if (H < 1) H = 1;
    auto has_out = [&](std::uint32_t s) { return nfa.out_off[s + 1] > nfa.out_off[s]; };
    d.nfa_of.clear();
    d.nfa_of.reserve(S);
    for (std::size_t i = 0; i < H; ++i)
        if (!has_out(hot_order[i])) d.nfa_of.push_back(hot_order[i]);
    d.Hn = static_cast<std::uint32_t>(d.nfa_of.size());
    for (std::size_t i = 0; i < H; ++i)
        if (has_out(hot_order[i])) d.nfa_of.push_back(hot_order[i]);
    d.H = static_cast<std::uint32_t>(H);
    for (std::size_t i = H; i < S; ++i)
        if (has_out(hot_order[i])) d.nfa_of.push_back(hot_order[i]);
    d.Cn = static_cast<std::uint32_t>(d.nfa_of.size());
    for (std::size_t i = H; i < S; ++i)
        if (!has_out(hot_order[i])) d.nfa_of.push_back(hot_order[i]);
    d.dev_of.assign(S, 0);
    for (std::uint32_t i = 0; i < S; ++i) d.dev_of[d.nfa_of[i]] = i;

    ph_ord.next("  (sub-phase end)");
    Phase ph_ren("  renumber rows");
    d.next.resize(static_cast<std::size_t>(S) * K);
    d.follows.resize(static_cast<std::size_t>(S) * K);
    d.follows_esc.resize(S);
    d.out_off.assign(S + 1, 0);
    d.depth.resize(S);
    for (std::uint32_t i = 0; i < S; ++i) {
        const std::uint32_t s = d.nfa_of[i];
        d.out_off[i + 1] = d.out_off[i] + (nfa.out_off[s + 1] - nfa.out_off[s]);
    }
    d.out_ids.resize(d.out_off[S]);
    d.outinfo.assign(S, 0ull);
    parallel_for(S, 1 << 14, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            const std::uint32_t s = d.nfa_of[i];
            d.depth[i] = nfa.depth[s];
            const std::size_t row = i * K, srow = static_cast<std::size_t>(s) * K;
            for (std::uint32_t c = 0; c < K; ++c) {
                d.next[row + c] = d.dev_of[delta[srow + c]];
                d.follows[row + c] = nfa.fol[srow + c];
            }
            d.follows_esc[i] = nfa.fesc[s];
            std::copy(nfa.out_ids.begin() + nfa.out_off[s], nfa.out_ids.begin() + nfa.out_off[s + 1],
                      d.out_ids.begin() + d.out_off[i]);
            const std::uint32_t lo2 = d.out_off[i], cnt = d.out_off[i + 1] - lo2;
            if (!cnt) continue;
            const std::uint64_t first = d.out_ids[lo2];
            d.outinfo[i] = lo2 | (static_cast<std::uint64_t>(std::min<std::uint32_t>(cnt, 255)) << 32) |
                           ((first < (1u << 24) ? first : 0ull) << 40);
        }
    });
    ph_ren.next("  hot tables");
    d.hot16.assign(static_cast<std::size_t>(H + 1) * K, 0xFFFF);
    for (std::size_t i = 0; i < static_cast<std::size_t>(H) * K; ++i)
        if (d.next[i] < H) d.hot16[i] = static_cast<std::uint16_t>(d.next[i]);

    // Truncated automaton A_H: valid when the hot set is a BFS prefix (closed
    // under longest-hot-suffix) and the alphabet is dna4 (4 columns, 8-byte rows).
    d.sparse_ok = !(visits && visits->size() == S) && d.mode == kAlphaDna4 && H <= 0x7FFF;
    if (d.sparse_ok) {
        d.hotH.assign(static_cast<std::size_t>(H) * K, 0);
        parallel_for(H, 4096, [&](std::size_t lo, std::size_t hi) {
            for (std::size_t i = lo; i < hi; ++i) {
                for (std::uint32_t c = 0; c < K; ++c) {
                    const std::uint32_t t = d.next[i * K + c];  // true target (device id)
                    std::uint32_t h = d.nfa_of[t];
                    while (d.dev_of[h] >= H) h = nfa.fail[h];  // first hot state on t's fail chain
                    const bool attn = t >= H || has_out(d.nfa_of[t]);
                    d.hotH[i * K + c] = static_cast<std::uint16_t>(d.dev_of[h] | (attn ? 0x8000u : 0u));
                }
            }
        });
    }
    // Truncated automaton for generic alphabets (SPARSE-G, exact_kernels.cuh):
    // hotG = longest hot suffix of the target | 0x8000 when the true target is
    // cold (BFS-ordered hot set only: closed under longest hot suffix).
    d.hotG.clear();
    if (d.mode == kAlphaGeneric && !(visits && visits->size() == S) && H <= 0x7FFF && H < S) {
        d.hotG.assign(static_cast<std::size_t>(H) * K, 0);
        parallel_for(H, 4096, [&](std::size_t lo, std::size_t hi) {
            for (std::size_t i = lo; i < hi; ++i) {
                for (std::uint32_t c = 0; c < K; ++c) {
                    const std::uint32_t t = d.next[i * K + c];
                    std::uint32_t h = d.nfa_of[t];
                    while (d.dev_of[h] >= H) h = nfa.fail[h];
                    d.hotG[i * K + c] = static_cast<std::uint16_t>(d.dev_of[h] | (t >= H ? 0x8000u : 0u));
                }
            }
        });
    }
    compile_ctab(nfa, hot_order, ctab_budget_bytes ? ctab_budget_bytes : hot_budget_bytes, d, hot_limit, visits);
    d.id_bits = 1;
    while ((1ull << d.id_bits) < nfa.n_patterns) ++d.id_bits;
    d.halo = (nfa.max_len + 15u) & ~15u;
    d.max_len = nfa.max_len;
    compile_qfilter(nfa, d);
}

}  // namespace acg
