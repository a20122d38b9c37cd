// Host-side pattern-matching machine (NFA view) and its dense-DFA image.
//
// The NFA is built with the reference's algorithm so that every public
// observable matches it: DFS-preorder state numbering with children in
// insertion order, BFS failure links, sorted suffix-closed output sets
// (reference: proj/include/acmatch/aho_corasick.hpp:130-233). The DFA image is
// the device's private representation: a dense transition table over symbol
// classes, states renumbered for locality, plus a CSR of output ids. Its
// numbering never leaks through the API.
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace acg {

using StateId = std::uint32_t;

struct Nfa {
    // CSR goto edges sorted by byte (aho_corasick.hpp:104-105)
    std::vector<std::uint32_t> edge_off;  // S+1
    std::vector<std::uint8_t> edge_byte;
    std::vector<StateId> edge_to;
    std::vector<StateId> fail;         // aho_corasick.hpp:106
    std::vector<std::uint32_t> depth;  // :107
    std::vector<std::uint32_t> out_off;  // S+1, suffix-closed, ascending (:108)
    std::vector<std::uint32_t> out_ids;
    std::vector<std::uint32_t> bfs;      // states in BFS order (root first)
    StateId root_row[256];               // :115-117
    std::uint32_t n_patterns = 0;
    std::uint32_t max_len = 0;
    std::uint32_t min_len = 0;
    std::vector<std::uint8_t> pat_bytes;  // the dictionary as given (q-gram prefilter build)
    std::vector<std::uint64_t> pat_off;   // n_patterns + 1
    // Dense image built level by level with the failure links (NFA numbering):
    // columns = symbol classes of the pattern alphabet (Dfa::mode / K / symmap).
    int mode = 1;                         // AlphaMode
    std::uint32_t K = 0, n_sym = 0;
    std::uint8_t symmap[256] = {};
    std::vector<int> col_byte;            // column -> byte (-1: escape column)
    std::vector<StateId> delta;           // S*K: next_state(s, byte of column c)
    std::vector<std::uint16_t> fol;       // S*K: failure links the reference walk follows (saturating)
    std::vector<std::uint16_t> fesc;      // S: ... for a byte outside the alphabet (dna4 mode)

    std::uint32_t state_count() const { return static_cast<std::uint32_t>(fail.size()); }
    bool goto_transition(StateId s, std::uint8_t b, StateId* out) const;
    StateId next_state(StateId s, std::uint8_t b) const;
};

// Error codes shared with the C ABI (include/acg.h).
enum : int {
    kOk = 0,
    kErrEmptyDictionary = 1,
    kErrEmptyPattern = 2,
    kErrInvalid = 3,
    kErrInvalidWorkerCount = 4,
    kErrCuda = 5,
    kErrOutOfMemory = 6,
    kErrNoDevice = 7,
    kErrTooLarge = 8,  // dictionary of >= 4 GiB: more states than a u32 StateId numbers (maps to kErrInvalid)
};

// build: reference aho_corasick.hpp:130-233. Returns an error code.
int build_nfa(const std::uint8_t* concat, const std::uint64_t* offs, std::uint32_t count, Nfa& out);

// Alphabet modes of the device scan.
enum AlphaMode : int {
    kAlphaDna4 = 0,     // pattern bytes ⊆ {A,C,G,T}: column = (byte>>1)&3, others escape
    kAlphaGeneric = 1,  // column = symmap[byte]; escape column K maps every state to the root
};

struct Dfa {
    int mode = kAlphaGeneric;
    std::uint32_t K = 0;        // table row stride (columns); generic mode includes the escape column
    std::uint32_t n_sym = 0;    // distinct pattern bytes
    std::uint8_t symmap[256];   // byte -> column (generic mode); escape = K-1
    std::uint32_t S = 0;
    // device numbering: [0,Hn) hot non-output, [Hn,H) hot output, [H,Cn) cold output, [Cn,S) cold non-output
    // (the output states [Hn,Cn) are contiguous: output rank = s - Hn)
    std::uint32_t H = 0, Hn = 0, Cn = 0;
    std::vector<std::uint32_t> dev_of;   // NFA id -> device id
    std::vector<std::uint32_t> nfa_of;   // device id -> NFA id
    std::vector<std::uint32_t> next;     // S*K, device ids
    std::vector<std::uint16_t> hot16;    // (H+1)*K, u16 device ids, 0xFFFF = consult `next`; row H all 0xFFFF
    // Truncated automaton over the hot set (sparse mode; dna4, BFS-ordered hot
    // set only): hotH[s*K+c] = longest hot suffix of s.c, | 0x8000 when the
    // true target is cold or has outputs (the step must be replayed exactly).
    std::vector<std::uint16_t> hotH;     // H*K
    bool sparse_ok = false;
    // Generic alphabets (SPARSE-G walk): H*K u16 = longest hot suffix of the
    // target | 0x8000 when the true target is cold (empty = not available).
    std::vector<std::uint16_t> hotG;
    // Compressed hot automaton (ctab.hpp; generic alphabets of <= 31 columns
    // whose states do not all fit the dense hot rows): the shared-memory image
    // = ct_slots row-displaced exception entries, then the K^ct_D default table.
    std::vector<std::uint32_t> ctab;
    std::uint32_t ct_slots = 0, ct_D = 0, ct_hot = 0;  // slots (= id space), default depth, hot states
    bool ct_cnt = false;                 // counted state words (output count in bits 17-24, ctab.hpp)
    bool ct_deep = false;                // the default takes one more level from the rows of the depth-D states
    std::vector<std::uint16_t> ct_rank;  // ct_slots: id -> output rank (kCtNoRank: none)
    std::vector<std::uint32_t> ct_sw;    // S: device state -> state word
    std::vector<std::uint32_t> ct_next;  // S*K: the dense table with state-word targets (cold steps: one load)
    std::vector<std::uint32_t> depth;    // S, device order
    std::vector<std::uint32_t> out_off;  // S+1 in device order
    std::vector<std::uint32_t> out_ids;  // ascending per state
    std::vector<std::uint16_t> follows;  // S*K failure follows taken by the reference scan on (s, column)
    std::vector<std::uint16_t> follows_esc;  // per state, for bytes outside the pattern alphabet (dna4 mode)
    // per device state: outputs packed for one load in the scan's emission —
    // out_off (32 bits) | count << 32 (8 bits, 255 = more) | first id << 40 (24 bits)
    std::vector<std::uint64_t> outinfo;
    std::uint32_t id_bits = 1;           // bits for a pattern id in a packed record
    std::uint32_t halo = 0;              // round_up(max_len, 16): warm-up bytes before each chunk
    std::uint32_t max_len = 0;
    // Sampled q-gram prefilter (filter mode; qfilter.hpp): dna4 dictionaries
    // whose shortest pattern has at least kQMinQ + kQSample - 1 bytes.
    bool filter_ok = false;
    std::uint32_t q = 0;
    // shared-memory image of level 1: the blocked Bloom filter of the (pattern,
    // offset) q-grams (kQWords words), or with qbm a 2^20-bit bitmap of their
    // 10-gram prefixes followed by that Bloom filter (kQBitmapWords + kQWordsBM)
    std::vector<std::uint32_t> qbloom;
    bool qbm = false;
    std::uint32_t qtab_bits = 0;         // exact table: 2^qtab_bits slots of (code, bucket start | kQEmpty)
    std::vector<std::uint32_t> qtab;     // 2 * 2^qtab_bits
    std::vector<std::uint32_t> qb_off;   // bucket offsets (keys + 1)
    std::vector<std::uint32_t> qb_ent;   // entries: pattern id << 2 | offset
    std::vector<std::uint32_t> pat_off32;  // pattern byte offsets (n_patterns + 1) into Nfa::pat_bytes
    std::vector<std::uint64_t> pat_code;   // per pattern 2 words: 2-bit codes of bytes 0..31, 32..63
    double filter_fp = 1.0;              // fraction of random q-grams passing the Bloom filter(s)
    // Level 2 (large dictionaries): when the shared-memory filter alone passes
    // too many q-grams, the ones it passes probe a second, L2-resident blocked
    // Bloom filter of the same keys (empty = single level).
    std::vector<std::uint32_t> qbloom2;
    double filter_fp1 = 1.0;             // pass rate of level 1 alone
};

// Fold the NFA into the dense DFA image. `hot_budget_bytes` bounds the u16 hot
// table kept in shared memory. `visits` (optional, NFA order) gives
// profile-guided hotness; otherwise BFS order is used.
// `ctab_budget_bytes` (0 = hot_budget_bytes) bounds the compressed hot
// automaton's image (ctab.hpp).
void compile_dfa(const Nfa& nfa, std::size_t hot_budget_bytes, const std::vector<std::uint64_t>* visits, Dfa& out,
                 std::uint32_t hot_limit = 0, std::size_t ctab_budget_bytes = 0);

}  // namespace acg
