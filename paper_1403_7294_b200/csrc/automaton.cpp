// Host automaton build (reference algorithm) and dense-DFA compilation.
#include "automaton.hpp"
#include "qfilter.hpp"

#include <algorithm>
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

// Open-addressing map (node, byte) -> child for trie insertion. Lookup only;
// the insertion order of children is kept separately in sibling lists, which
// is what the reference's preorder depends on (aho_corasick.hpp:139-166).
struct EdgeMap {
    std::vector<std::uint64_t> keys;
    std::vector<std::uint32_t> vals;
    std::uint64_t mask = 0;
    std::size_t used = 0;

    explicit EdgeMap(std::size_t expect) {
        std::size_t cap = 1024;
        while (cap < expect * 2) cap <<= 1;
        keys.assign(cap, ~0ull);
        vals.assign(cap, 0);
        mask = cap - 1;
    }
    static std::uint64_t hash(std::uint64_t k) {
        k ^= k >> 33;
        k *= 0xff51afd7ed558ccdull;
        k ^= k >> 33;
        return k;
    }
    std::uint32_t* find_or_slot(std::uint64_t key, bool* found) {
        std::uint64_t i = hash(key) & mask;
        for (;;) {
            if (keys[i] == key) {
                *found = true;
                return &vals[i];
            }
            if (keys[i] == ~0ull) {
                *found = false;
                keys[i] = key;
                ++used;
                return &vals[i];
            }
            i = (i + 1) & mask;
        }
    }
};

}  // namespace

int build_nfa(const std::uint8_t* concat, const std::uint64_t* offs, std::uint32_t count, Nfa& nfa) {
    if (count == 0) return kErrEmptyDictionary;  // aho_corasick.hpp:131
    std::uint64_t total = 0;
    std::uint32_t max_len = 0;
    for (std::uint32_t i = 0; i < count; ++i) {
        const std::uint64_t len = offs[i + 1] - offs[i];
        if (len == 0) return kErrEmptyPattern;  // :133-134
        total += len;
        max_len = std::max<std::uint32_t>(max_len, static_cast<std::uint32_t>(len));
    }
    // states are u32 (StateId, aho_corasick.hpp:18): up to total + 1 of them
    if (total >= 0xFFFFFFF0ull) return kErrTooLarge;

    // Phase 1: keyword trie, children in insertion order.
    std::vector<std::uint32_t> first_kid(1, 0), next_sib(1, 0), last_kid(1, 0), tdepth(1, 0);
    std::vector<std::uint8_t> tbyte(1, 0);
    std::vector<std::uint32_t> own_head(1, ~0u);  // first pattern id ending here
    std::vector<std::uint32_t> own_next(count, ~0u), own_tail(1, ~0u);
    EdgeMap map(static_cast<std::size_t>(std::min<std::uint64_t>(total, 1ull << 30)) + 16);
    for (std::uint32_t p = 0; p < count; ++p) {
        std::uint32_t node = 0;
        for (std::uint64_t k = offs[p]; k < offs[p + 1]; ++k) {
            const std::uint8_t b = concat[k];
            bool found;
            std::uint32_t* slot = map.find_or_slot((static_cast<std::uint64_t>(node) << 8) | b, &found);
            if (found) {
                node = *slot;
                continue;
            }
            const auto child = static_cast<std::uint32_t>(first_kid.size());
            *slot = child;
            first_kid.push_back(0);
            next_sib.push_back(0);
            last_kid.push_back(0);
            tdepth.push_back(tdepth[node] + 1);
            tbyte.push_back(b);
            own_head.push_back(~0u);
            own_tail.push_back(~0u);
            if (last_kid[node]) next_sib[last_kid[node]] = child;
            else first_kid[node] = child;
            last_kid[node] = child;
            node = child;
        }
        // own ids in id order: ascending (:165, :192)
        if (own_head[node] == ~0u) own_head[node] = p;
        else own_next[own_tail[node]] = p;
        own_tail[node] = p;
    }
    const auto n = static_cast<std::uint32_t>(first_kid.size());

    // Phase 2: DFS preorder, children in insertion order (:170-183).
    std::vector<std::uint32_t> order;
    order.reserve(n);
    {
        std::vector<std::uint32_t> stack{0}, kids;
        while (!stack.empty()) {
            const std::uint32_t v = stack.back();
            stack.pop_back();
            order.push_back(v);
            kids.clear();
            for (std::uint32_t k = first_kid[v]; k; k = next_sib[k]) kids.push_back(k);
            for (auto it = kids.rbegin(); it != kids.rend(); ++it) stack.push_back(*it);
        }
    }
    std::vector<std::uint32_t> renum(n);
    for (std::uint32_t s = 0; s < n; ++s) renum[order[s]] = s;

    // Freeze: per-state edges sorted by byte (:185-196).
    nfa.edge_off.assign(n + 1, 0);
    nfa.edge_byte.resize(n - 1);
    nfa.edge_to.resize(n - 1);
    nfa.depth.assign(n, 0);
    nfa.fail.assign(n, 0);
    {
        std::uint32_t e = 0;
        std::vector<std::pair<std::uint8_t, std::uint32_t>> tmp;
        for (std::uint32_t s = 0; s < n; ++s) {
            const std::uint32_t t = order[s];
            nfa.depth[s] = tdepth[t];
            nfa.edge_off[s] = e;
            tmp.clear();
            for (std::uint32_t k = first_kid[t]; k; k = next_sib[k]) tmp.emplace_back(tbyte[k], renum[k]);
            std::sort(tmp.begin(), tmp.end());
            for (const auto& [b, c] : tmp) {
                nfa.edge_byte[e] = b;
                nfa.edge_to[e] = c;
                ++e;
            }
        }
        nfa.edge_off[n] = e;
    }

    // Phase 3: BFS failure links + suffix-closed outputs (:201-226).
    // fail(child of u by b) = next_state(fail(u), b); the reference finds it
    // with the same chain walk (:205-215).
    nfa.bfs.clear();
    nfa.bfs.reserve(n);
    nfa.bfs.push_back(0);
    std::vector<std::uint32_t> out_start(n, 0), out_len(n, 0);
    std::vector<std::uint32_t> pool;
    pool.reserve(count * 2ull);
    auto own_list = [&](std::uint32_t s, std::vector<std::uint32_t>& dst) {
        dst.clear();
        for (std::uint32_t p = own_head[order[s]]; p != ~0u; p = own_next[p]) dst.push_back(p);
    };
    std::vector<std::uint32_t> own, merged;
    for (std::uint32_t j = nfa.edge_off[0]; j < nfa.edge_off[1]; ++j) {
        const std::uint32_t c = nfa.edge_to[j];
        nfa.fail[c] = 0;
        nfa.bfs.push_back(c);
    }
    for (std::size_t head = 1; head < nfa.bfs.size(); ++head) {
        const std::uint32_t u = nfa.bfs[head];
        // outputs of u: own merged with out(fail(u)) (fail(u) precedes u in BFS)
        own_list(u, own);
        const std::uint32_t f = nfa.fail[u];
        merged.clear();
        std::merge(own.begin(), own.end(), pool.begin() + out_start[f], pool.begin() + out_start[f] + out_len[f],
                   std::back_inserter(merged));
        out_start[u] = static_cast<std::uint32_t>(pool.size());
        out_len[u] = static_cast<std::uint32_t>(merged.size());
        pool.insert(pool.end(), merged.begin(), merged.end());
        for (std::uint32_t j = nfa.edge_off[u]; j < nfa.edge_off[u + 1]; ++j) {
            const std::uint8_t b = nfa.edge_byte[j];
            const std::uint32_t child = nfa.edge_to[j];
            if (u != 0) nfa.fail[child] = nfa.next_state(nfa.fail[u], b);
            nfa.bfs.push_back(child);
        }
    }
    nfa.out_off.assign(n + 1, 0);
    for (std::uint32_t s = 0; s < n; ++s) nfa.out_off[s + 1] = nfa.out_off[s] + out_len[s];
    nfa.out_ids.resize(nfa.out_off[n]);
    for (std::uint32_t s = 0; s < n; ++s)
        std::copy_n(pool.begin() + out_start[s], out_len[s], nfa.out_ids.begin() + nfa.out_off[s]);

    // dense root row (:230-231)
    std::fill(std::begin(nfa.root_row), std::end(nfa.root_row), 0u);
    for (std::uint32_t j = nfa.edge_off[0]; j < nfa.edge_off[1]; ++j) nfa.root_row[nfa.edge_byte[j]] = nfa.edge_to[j];
    nfa.n_patterns = count;
    nfa.max_len = max_len;
    nfa.min_len = ~0u;
    for (std::uint32_t i = 0; i < count; ++i)
        nfa.min_len = std::min<std::uint32_t>(nfa.min_len, static_cast<std::uint32_t>(offs[i + 1] - offs[i]));
    nfa.pat_bytes.assign(concat, concat + offs[count]);
    nfa.pat_off.assign(offs, offs + count + 1);
    for (auto& o : nfa.pat_off) o -= offs[0];
    return kOk;
}

namespace {

// The q-gram prefilter (qfilter.hpp): every pattern's q-grams at offsets
// 0..kQSample-1 into the blocked Bloom filter and the exact (code -> (pattern,
// offset) list) hash table.
void compile_qfilter(const Nfa& nfa, Dfa& d) {
    d.filter_ok = false;
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
    std::sort(grams.begin(), grams.end());
    std::uint32_t words = kQWords;
    if (const char* e = std::getenv("ACG_QWORDS")) {  // experiments only (Bloom size sweeps)
        const long v = std::strtol(e, nullptr, 10);
        if (v >= 1024 && v <= 57344) words = static_cast<std::uint32_t>(v) & ~3u;
    }
    d.qbloom.assign(words, 0u);
    std::uint32_t keys = 0;
    for (std::size_t i = 0; i < grams.size(); ++i) {
        if (i && grams[i].first == grams[i - 1].first) continue;
        ++keys;
        const std::uint32_t h = qhash(qtop(grams[i].first, q));
        d.qbloom[qword(h, words)] |= qmask(h);
    }
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
    d.pat_off32.assign(nfa.pat_off.begin(), nfa.pat_off.end());
    d.pat_code.assign(2ull * nfa.n_patterns, 0ull);
    for (std::uint32_t p = 0; p < nfa.n_patterns; ++p) {
        const std::uint32_t lo = nfa.pat_off[p], len = std::min<std::uint32_t>(nfa.pat_off[p + 1] - lo, 64);
        for (std::uint32_t k = 0; k < len; ++k)
            d.pat_code[2ull * p + k / 32] |= static_cast<std::uint64_t>((nfa.pat_bytes[lo + k] >> 1) & 3u) << (2 * (k % 32));
    }
    // pass rates of random q-grams (splitmix64 sample), level 1 and overall
    auto pass_rates = [&](double& fp1, double& fp) {
        std::uint64_t z = 0x14037294ull, p1 = 0, p2 = 0;
        const std::uint32_t trials = 1u << 20;
        const std::uint32_t words2 = static_cast<std::uint32_t>(d.qbloom2.size());
        for (std::uint32_t t = 0; t < trials; ++t) {
            z += 0x9E3779B97F4A7C15ull;
            std::uint64_t r = z;
            r = (r ^ (r >> 30)) * 0xBF58476D1CE4E5B9ull;
            r = (r ^ (r >> 27)) * 0x94D049BB133111EBull;
            const std::uint32_t c = static_cast<std::uint32_t>(r ^ (r >> 31)) & qm;
            const std::uint32_t h = qhash(qtop(c, q));
            const std::uint32_t m = qmask(h);
            if ((d.qbloom[qword(h, words)] & m) != m) continue;
            ++p1;
            if (!words2) {
                ++p2;
                continue;
            }
            const std::uint32_t h2 = qhash2(h), m2 = qmask(h2);
            p2 += (d.qbloom2[qword(h2, words2)] & m2) == m2;
        }
        fp1 = static_cast<double>(p1) / trials;
        fp = static_cast<double>(p2) / trials;
    };
    pass_rates(d.filter_fp1, d.filter_fp);
    if (d.filter_fp > 5e-3 && d.filter_fp1 <= kQLevel1Max) {
        // level 2: ~1.5 % of its bits set (4 bits per key)
        std::uint64_t w2 = (static_cast<std::uint64_t>(keys) * 4 * 100 / 3 / 32 + 3) & ~3ull;
        w2 = std::min<std::uint64_t>(std::max<std::uint64_t>(w2, 1024), 16ull << 20);
        d.qbloom2.assign(w2, 0u);
        for (std::size_t i = 0; i < grams.size(); ++i) {
            if (i && grams[i].first == grams[i - 1].first) continue;
            const std::uint32_t h2 = qhash2(qhash(qtop(grams[i].first, q)));
            d.qbloom2[qword(h2, static_cast<std::uint32_t>(w2))] |= qmask(h2);
        }
        pass_rates(d.filter_fp1, d.filter_fp);
    }
    // worth it when few samples survive (each survivor costs an exact probe)
    d.filter_ok = d.filter_fp <= 5e-3;
    if (!d.filter_ok) {
        d.pat_code.clear();
        d.qbloom2.clear();
        d.qbloom.clear();
        d.qtab.clear();
        d.qb_off.clear();
        d.qb_ent.clear();
    }
}

}  // namespace


void compile_dfa(const Nfa& nfa, std::size_t hot_budget_bytes, const std::vector<std::uint64_t>* visits, Dfa& d,
                 std::uint32_t hot_limit) {
    const std::uint32_t S = nfa.state_count();
    // Alphabet: which bytes occur in patterns (as goto labels).
    bool used[256] = {};
    for (std::uint8_t b : nfa.edge_byte) used[b] = true;
    std::uint32_t n_sym = 0;
    for (bool u : used) n_sym += u;
    const bool dna = [&] {
        for (int b = 0; b < 256; ++b)
            if (used[b] && b != 'A' && b != 'C' && b != 'G' && b != 'T') return false;
        return true;
    }();
    // column -> byte (or -1 for the escape column)
    std::vector<int> col_byte;
    if (dna) {
        d.mode = kAlphaDna4;
        d.K = 4;
        col_byte = {'A', 'C', 'T', 'G'};  // column = (byte >> 1) & 3
        std::memset(d.symmap, 0, sizeof d.symmap);
        for (int c = 0; c < 4; ++c) d.symmap[col_byte[c]] = static_cast<std::uint8_t>(c);
    } else {
        d.mode = kAlphaGeneric;
        d.K = n_sym + 1;
        std::uint32_t c = 0;
        for (int b = 0; b < 256; ++b)
            if (used[b]) {
                d.symmap[b] = static_cast<std::uint8_t>(c++);
                col_byte.push_back(b);
            }
        for (int b = 0; b < 256; ++b)
            if (!used[b]) d.symmap[b] = static_cast<std::uint8_t>(n_sym);  // escape column
        col_byte.push_back(-1);
    }
    d.n_sym = n_sym;
    const std::uint32_t K = d.K;
    d.S = S;

    // Dense delta in NFA numbering, computed in BFS order:
    // delta(s,c) = goto(s,c) if present else delta(fail(s),c); root misses stay at root.
    std::vector<std::uint32_t> delta(static_cast<std::size_t>(S) * K);
    std::vector<std::uint32_t> fol(static_cast<std::size_t>(S) * K);
    std::vector<std::uint32_t> fesc(S, 0);
    // (row = the fail state's row, one more follow per column, then the state's
    // own goto edges; the fail state precedes s in BFS order)
    int col_of[256];
    std::fill(std::begin(col_of), std::end(col_of), -1);
    for (std::uint32_t c = 0; c < K; ++c)
        if (col_byte[c] >= 0) col_of[col_byte[c]] = static_cast<int>(c);
    for (std::uint32_t s : nfa.bfs) {
        const std::size_t row = static_cast<std::size_t>(s) * K;
        if (s == 0) {
            std::fill_n(delta.begin() + row, K, 0u);
            std::fill_n(fol.begin() + row, K, 0u);
        } else {
            const std::size_t frow = static_cast<std::size_t>(nfa.fail[s]) * K;
            for (std::uint32_t c = 0; c < K; ++c) {
                delta[row + c] = delta[frow + c];
                fol[row + c] = 1 + fol[frow + c];  // reference follows one failure link, then retries
            }
        }
        for (std::uint32_t j = nfa.edge_off[s]; j < nfa.edge_off[s + 1]; ++j) {
            const int c = col_of[nfa.edge_byte[j]];
            if (c < 0) continue;  // (every pattern byte has a column)
            delta[row + c] = nfa.edge_to[j];
            fol[row + c] = 0;
        }
        fesc[s] = s == 0 ? 0 : 1 + fesc[nfa.fail[s]];
    }

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
        if (!has_out(hot_order[i])) d.nfa_of.push_back(hot_order[i]);
    d.Cn = static_cast<std::uint32_t>(d.nfa_of.size());
    for (std::size_t i = H; i < S; ++i)
        if (has_out(hot_order[i])) d.nfa_of.push_back(hot_order[i]);
    d.dev_of.assign(S, 0);
    for (std::uint32_t i = 0; i < S; ++i) d.dev_of[d.nfa_of[i]] = i;

    d.next.resize(static_cast<std::size_t>(S) * K);
    d.follows.resize(static_cast<std::size_t>(S) * K);
    d.follows_esc.resize(S);
    d.out_off.assign(S + 1, 0);
    d.depth.resize(S);
    for (std::uint32_t i = 0; i < S; ++i) {
        const std::uint32_t s = d.nfa_of[i];
        d.depth[i] = nfa.depth[s];
        for (std::uint32_t c = 0; c < K; ++c) {
            d.next[static_cast<std::size_t>(i) * K + c] = d.dev_of[delta[static_cast<std::size_t>(s) * K + c]];
            const std::uint32_t f = fol[static_cast<std::size_t>(s) * K + c];
            d.follows[static_cast<std::size_t>(i) * K + c] = static_cast<std::uint16_t>(std::min<std::uint32_t>(f, 0xFFFF));
        }
        d.follows_esc[i] = static_cast<std::uint16_t>(std::min<std::uint32_t>(fesc[s], 0xFFFF));
        d.out_off[i + 1] = d.out_off[i] + (nfa.out_off[s + 1] - nfa.out_off[s]);
    }
    d.out_ids.resize(d.out_off[S]);
    for (std::uint32_t i = 0; i < S; ++i) {
        const std::uint32_t s = d.nfa_of[i];
        std::copy(nfa.out_ids.begin() + nfa.out_off[s], nfa.out_ids.begin() + nfa.out_off[s + 1],
                  d.out_ids.begin() + d.out_off[i]);
    }
    d.outinfo.assign(S, 0ull);
    for (std::uint32_t i = 0; i < S; ++i) {
        const std::uint32_t lo = d.out_off[i], cnt = d.out_off[i + 1] - lo;
        if (!cnt) continue;
        const std::uint64_t first = d.out_ids[lo];
        d.outinfo[i] = lo | (static_cast<std::uint64_t>(std::min<std::uint32_t>(cnt, 255)) << 32) |
                       ((first < (1u << 24) ? first : 0ull) << 40);
    }
    d.hot16.assign(static_cast<std::size_t>(H + 1) * K, 0xFFFF);
    for (std::size_t i = 0; i < static_cast<std::size_t>(H) * K; ++i)
        if (d.next[i] < H) d.hot16[i] = static_cast<std::uint16_t>(d.next[i]);

    // Truncated automaton A_H: valid when the hot set is a BFS prefix (closed
    // under longest-hot-suffix) and the alphabet is dna4 (4 columns, 8-byte rows).
    d.sparse_ok = !(visits && visits->size() == S) && d.mode == kAlphaDna4 && H <= 0x7FFF;
    if (d.sparse_ok) {
        d.hotH.assign(static_cast<std::size_t>(H) * K, 0);
        for (std::uint32_t i = 0; i < H; ++i) {
            for (std::uint32_t c = 0; c < K; ++c) {
                const std::uint32_t t = d.next[static_cast<std::size_t>(i) * K + c];  // true target (device id)
                std::uint32_t h = d.nfa_of[t];
                while (d.dev_of[h] >= H) h = nfa.fail[h];  // first hot state on t's fail chain
                const bool attn = t >= H || has_out(d.nfa_of[t]);
                d.hotH[static_cast<std::size_t>(i) * K + c] =
                    static_cast<std::uint16_t>(d.dev_of[h] | (attn ? 0x8000u : 0u));
            }
        }
    }
    d.id_bits = 1;
    while ((1ull << d.id_bits) < nfa.n_patterns) ++d.id_bits;
    d.halo = (nfa.max_len + 15u) & ~15u;
    d.max_len = nfa.max_len;
    compile_qfilter(nfa, d);
}

}  // namespace acg
