/*
 * ORACLE — test infrastructure, NOT the product.
 *
 * A plain-C restatement of the reference's Aho-Corasick algorithm, used only
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker. Nothing in paper_1403_7294_b200/ links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks this restatement against
 *   (1) the reference's own known-answer vectors (SHERS, AA/AAAA, the
 *       full-byte alphabet case, ABCABC, the classic machine shape), and
 *   (2) the reference itself compiled from /root/reference by
 *       oracle/Makefile into oracle/_ref/ (randomised trials, seeds of the
 *       reference acceptance runner), and
 *   (3) committed golden fixtures in tests/golden/ made by
 *       oracle/make_goldens.py from that compiled reference.
 *
 * Each function cites the reference code it restates
 * (paths relative to /root/reference/proj).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint32_t state_t;

typedef struct {
    uint32_t n_states;
    uint32_t n_patterns;
    uint32_t max_len;
    /* goto edges, CSR sorted by byte: include/acmatch/aho_corasick.hpp:104-105 */
    uint32_t *edge_off; /* n_states + 1 */
    uint8_t *edge_byte;
    state_t *edge_to;
    state_t *fail;      /* :106 */
    uint32_t *depth;    /* :107 */
    uint32_t *out_off;  /* n_states + 1, suffix-closed sorted outputs :108 */
    uint32_t *out_ids;
    state_t root_row[256]; /* :115-117 */
} orc_automaton;

/* ---- growable arrays ---------------------------------------------------- */
typedef struct { uint32_t *v; size_t n, cap; } u32vec;
static int u32_push(u32vec *a, uint32_t x) {
    if (a->n == a->cap) {
        size_t c = a->cap ? a->cap * 2 : 16;
        uint32_t *p = (uint32_t *)realloc(a->v, c * sizeof(uint32_t));
        if (!p) return -1;
        a->v = p;
        a->cap = c;
    }
    a->v[a->n++] = x;
    return 0;
}

/* Trie node with children kept in insertion order (a sibling list), as the
 * reference's phase 1 keeps `kids` in insertion order
 * (include/acmatch/aho_corasick.hpp:139-166). */
typedef struct {
    uint32_t first_kid, last_kid, next_sib; /* 0 = none (root is never a kid) */
    uint32_t depth;
    uint32_t own_head; /* index into own list chain, 0 = none */
    uint8_t byte;
} tnode;

typedef struct { uint32_t id, next; } ownlink;

void orc_free(orc_automaton *a) {
    if (!a) return;
    free(a->edge_off); free(a->edge_byte); free(a->edge_to);
    free(a->fail); free(a->depth); free(a->out_off); free(a->out_ids);
    free(a);
}

static int cmp_edge(const void *x, const void *y) {
    const uint64_t a = *(const uint64_t *)x, b = *(const uint64_t *)y;
    return (a > b) - (a < b);
}

/* Sorted-edge goto lookup: include/acmatch/aho_corasick.hpp:67-74. */
static int orc_goto(const orc_automaton *a, state_t s, uint8_t b, state_t *out) {
    uint32_t lo = a->edge_off[s], hi = a->edge_off[s + 1];
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (a->edge_byte[mid] < b) lo = mid + 1; else hi = mid;
    }
    if (lo < a->edge_off[s + 1] && a->edge_byte[lo] == b) { *out = a->edge_to[lo]; return 1; }
    return 0;
}

/*
 * build: include/acmatch/aho_corasick.hpp:130-233.
 *   errors (return codes): 1 = empty dictionary (:131), 2 = empty pattern (:133-134).
 *   Ids are implicitly dense (pattern i has id i), the reference's :135-136 check.
 */
int orc_build(const uint8_t *concat, const uint64_t *offs, uint32_t count, orc_automaton **out) {
    *out = NULL;
    if (count == 0) return 1;
    for (uint32_t i = 0; i < count; ++i)
        if (offs[i + 1] == offs[i]) return 2;

    /* Phase 1: keyword trie (:139-166). */
    size_t cap = 1024, n = 1;
    tnode *trie = (tnode *)calloc(cap, sizeof(tnode));
    ownlink *own = (ownlink *)malloc(sizeof(ownlink) * (count + 1));
    uint32_t *own_tail = NULL;
    uint32_t max_len = 0;
    if (!trie || !own) { free(trie); free(own); return -1; }
    for (uint32_t p = 0; p < count; ++p) {
        uint32_t node = 0;
        const uint64_t len = offs[p + 1] - offs[p];
        if (len > max_len) max_len = (uint32_t)len;
        for (uint64_t k = 0; k < len; ++k) {
            const uint8_t b = concat[offs[p] + k];
            uint32_t kid = trie[node].first_kid, found = 0;
            for (; kid; kid = trie[kid].next_sib)
                if (trie[kid].byte == b) { found = kid; break; }
            if (found) { node = found; continue; }
            if (n == cap) {
                cap *= 2;
                tnode *t = (tnode *)realloc(trie, cap * sizeof(tnode));
                if (!t) { free(trie); free(own); return -1; }
                trie = t;
            }
            const uint32_t child = (uint32_t)n++;
            memset(&trie[child], 0, sizeof(tnode));
            trie[child].byte = b;
            trie[child].depth = trie[node].depth + 1;
            if (trie[node].last_kid) trie[trie[node].last_kid].next_sib = child;
            else trie[node].first_kid = child;
            trie[node].last_kid = child;
            node = child;
        }
        /* own ids appended in id order, so each list is ascending (:165, :192) */
        own[p + 1].id = p;
        own[p + 1].next = 0;
        if (!trie[node].own_head) trie[node].own_head = p + 1;
        else {
            uint32_t t = trie[node].own_head;
            while (own[t].next) t = own[t].next;
            own[t].next = p + 1;
        }
    }
    (void)own_tail;

    /* Phase 2: DFS preorder numbering, children in insertion order (:170-183). */
    uint32_t *order = (uint32_t *)malloc(n * sizeof(uint32_t));
    uint32_t *renum = (uint32_t *)malloc(n * sizeof(uint32_t));
    u32vec stack = {0}, kids = {0};
    size_t no = 0;
    u32_push(&stack, 0);
    while (stack.n) {
        const uint32_t v = stack.v[--stack.n];
        order[no++] = v;
        kids.n = 0;
        for (uint32_t k = trie[v].first_kid; k; k = trie[k].next_sib) u32_push(&kids, k);
        for (size_t j = kids.n; j-- > 0;) u32_push(&stack, kids.v[j]);
    }
    for (uint32_t s = 0; s < n; ++s) renum[order[s]] = s;

    orc_automaton *a = (orc_automaton *)calloc(1, sizeof(orc_automaton));
    a->n_states = (uint32_t)n;
    a->n_patterns = count;
    a->max_len = max_len;
    a->edge_off = (uint32_t *)calloc(n + 1, sizeof(uint32_t));
    a->edge_byte = (uint8_t *)malloc(n > 1 ? n - 1 : 1);
    a->edge_to = (state_t *)malloc((n > 1 ? n - 1 : 1) * sizeof(state_t));
    a->fail = (state_t *)calloc(n, sizeof(state_t));
    a->depth = (uint32_t *)calloc(n, sizeof(uint32_t));

    /* freeze: edges re-sorted by byte (:185-196) */
    uint64_t *tmp = (uint64_t *)malloc(257 * sizeof(uint64_t));
    uint32_t e = 0;
    for (uint32_t s = 0; s < n; ++s) {
        const tnode *t = &trie[order[s]];
        a->depth[s] = t->depth;
        a->edge_off[s] = e;
        uint32_t m = 0;
        for (uint32_t k = t->first_kid; k; k = trie[k].next_sib)
            tmp[m++] = ((uint64_t)trie[k].byte << 32) | renum[k];
        qsort(tmp, m, sizeof(uint64_t), cmp_edge);
        for (uint32_t j = 0; j < m; ++j) {
            a->edge_byte[e] = (uint8_t)(tmp[j] >> 32);
            a->edge_to[e] = (uint32_t)tmp[j];
            ++e;
        }
    }
    a->edge_off[n] = e;
    free(tmp);

    /* Phase 3: BFS failure links; outputs merged with the fail state's
     * (:201-226). Outputs are built into per-state vectors, then packed. */
    u32vec *outs = (u32vec *)calloc(n, sizeof(u32vec));
    for (uint32_t s = 0; s < n; ++s)
        for (uint32_t o = trie[order[s]].own_head; o; o = own[o].next) u32_push(&outs[s], own[o].id);
    uint32_t *queue = (uint32_t *)malloc(n * sizeof(uint32_t));
    size_t qh = 0, qt = 0;
    for (uint32_t j = a->edge_off[0]; j < a->edge_off[1]; ++j) {
        a->fail[a->edge_to[j]] = 0;
        queue[qt++] = a->edge_to[j];
    }
    while (qh < qt) {
        const uint32_t u = queue[qh++];
        for (uint32_t j = a->edge_off[u]; j < a->edge_off[u + 1]; ++j) {
            const uint8_t b = a->edge_byte[j];
            const uint32_t child = a->edge_to[j];
            uint32_t f = a->fail[u], target = 0;
            int has = 0;
            for (;;) {
                has = orc_goto(a, f, b, &target);
                if (has || f == 0) break;
                f = a->fail[f];
            }
            a->fail[child] = has ? target : 0;
            const u32vec *inh = &outs[a->fail[child]];
            if (inh->n) { /* std::merge of two ascending lists (:219-225) */
                u32vec merged = {0};
                size_t x = 0, y = 0;
                const u32vec *mine = &outs[child];
                while (x < mine->n || y < inh->n) {
                    if (y >= inh->n || (x < mine->n && !(inh->v[y] < mine->v[x])))
                        u32_push(&merged, mine->v[x++]);
                    else
                        u32_push(&merged, inh->v[y++]);
                }
                free(outs[child].v);
                outs[child] = merged;
            }
            queue[qt++] = child;
        }
    }
    size_t tot = 0;
    for (uint32_t s = 0; s < n; ++s) tot += outs[s].n;
    a->out_off = (uint32_t *)malloc((n + 1) * sizeof(uint32_t));
    a->out_ids = (uint32_t *)malloc((tot ? tot : 1) * sizeof(uint32_t));
    tot = 0;
    for (uint32_t s = 0; s < n; ++s) {
        a->out_off[s] = (uint32_t)tot;
        if (outs[s].n) memcpy(a->out_ids + tot, outs[s].v, outs[s].n * sizeof(uint32_t));
        tot += outs[s].n;
        free(outs[s].v);
    }
    a->out_off[n] = (uint32_t)tot;

    /* dense root row (:230-231) */
    for (int b = 0; b < 256; ++b) a->root_row[b] = 0;
    for (uint32_t j = a->edge_off[0]; j < a->edge_off[1]; ++j) a->root_row[a->edge_byte[j]] = a->edge_to[j];

    free(outs); free(queue); free(order); free(renum); free(stack.v); free(kids.v);
    free(trie); free(own);
    *out = a;
    return 0;
}

/* ---- accessors (include/acmatch/aho_corasick.hpp:60-101) ----------------- */
uint32_t orc_state_count(const orc_automaton *a) { return a->n_states; }
uint32_t orc_max_len(const orc_automaton *a) { return a->max_len; }
state_t orc_failure(const orc_automaton *a, state_t s) { return a->fail[s]; }
uint32_t orc_depth(const orc_automaton *a, state_t s) { return a->depth[s]; }
int orc_goto_transition(const orc_automaton *a, state_t s, uint8_t b, state_t *out) { return orc_goto(a, s, b, out); }
uint32_t orc_outputs(const orc_automaton *a, state_t s, const uint32_t **ids) {
    *ids = a->out_ids + a->out_off[s];
    return a->out_off[s + 1] - a->out_off[s];
}
uint32_t orc_transitions(const orc_automaton *a, state_t s, const uint8_t **bytes, const state_t **to) {
    *bytes = a->edge_byte + a->edge_off[s];
    *to = a->edge_to + a->edge_off[s];
    return a->edge_off[s + 1] - a->edge_off[s];
}

/* next_state: include/acmatch/aho_corasick.hpp:238-245 */
state_t orc_next_state(const orc_automaton *a, state_t s, uint8_t b) {
    for (;;) {
        state_t t;
        if (orc_goto(a, s, b, &t)) return t;
        if (s == 0) return 0;
        s = a->fail[s];
    }
}

/*
 * scan: include/acmatch/aho_corasick.hpp:250-272, generalised to the window
 * [start, n) of `text` (start scanning at byte `start` from the root) while
 * emitting only records with end >= emit_from and counting failure follows
 * only on steps at positions >= emit_from. With start = 0 and emit_from = 0
 * this is exactly the reference scan. Records are written when ids/ends are
 * non-NULL (capacity cap); the return value is the full record count.
 */
uint64_t orc_scan_window(const orc_automaton *a, const uint8_t *text, uint64_t n, uint64_t start,
                         uint64_t emit_from, uint64_t *follows, uint32_t *ids, uint64_t *ends,
                         uint64_t cap, uint64_t *counts) {
    uint64_t m = 0, fol = 0;
    state_t s = 0;
    for (uint64_t i = start; i < n; ++i) {
        const uint8_t b = text[i];
        const int owned = i >= emit_from;
        for (;;) {
            if (s == 0) { s = a->root_row[b]; break; }
            state_t t;
            if (orc_goto(a, s, b, &t)) { s = t; break; }
            s = a->fail[s];
            fol += owned;
        }
        if (!owned) continue;
        for (uint32_t j = a->out_off[s]; j < a->out_off[s + 1]; ++j) {
            if (ids && m < cap) { ids[m] = a->out_ids[j]; ends[m] = i; }
            if (counts) counts[a->out_ids[j]]++;
            ++m;
        }
    }
    if (follows) *follows = fol;
    return m;
}

uint64_t orc_scan(const orc_automaton *a, const uint8_t *text, uint64_t n, uint64_t *follows,
                  uint32_t *ids, uint64_t *ends, uint64_t cap) {
    return orc_scan_window(a, text, n, 0, 0, follows, ids, ends, cap, NULL);
}

/* Brute force: tests/support/oracle.hpp:31-43 (every (pattern, offset) pair),
 * records sorted by (end, id) (include/acmatch/aho_corasick.hpp:38-41). */
typedef struct { uint64_t end; uint32_t id; } rec;
static int cmp_rec(const void *x, const void *y) {
    const rec *a = (const rec *)x, *b = (const rec *)y;
    if (a->end != b->end) return (a->end > b->end) - (a->end < b->end);
    return (a->id > b->id) - (a->id < b->id);
}
uint64_t orc_naive_find_all(const uint8_t *concat, const uint64_t *offs, uint32_t count, const uint8_t *text,
                            uint64_t n, uint32_t *ids, uint64_t *ends, uint64_t cap) {
    uint64_t m = 0;
    rec *buf = NULL;
    size_t bcap = 0;
    for (uint32_t p = 0; p < count; ++p) {
        const uint64_t len = offs[p + 1] - offs[p];
        if (len == 0 || len > n) continue;
        for (uint64_t off = 0; off + len <= n; ++off)
            if (memcmp(text + off, concat + offs[p], len) == 0) {
                if (m == bcap) {
                    bcap = bcap ? bcap * 2 : 256;
                    buf = (rec *)realloc(buf, bcap * sizeof(rec));
                }
                buf[m].end = off + len - 1;
                buf[m].id = p;
                ++m;
            }
    }
    qsort(buf, m, sizeof(rec), cmp_rec);
    for (uint64_t i = 0; i < m && i < cap; ++i) { ids[i] = buf[i].id; ends[i] = buf[i].end; }
    free(buf);
    return m;
}

/* ---- record digest shared with the golden fixtures ----------------------- */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
/* order-independent digest of a record set: key = end * 2^20 + id */
void orc_digest(const uint32_t *ids, const uint64_t *ends, uint64_t m, uint64_t *dsum, uint64_t *dxor) {
    uint64_t s = 0, x = 0;
    for (uint64_t i = 0; i < m; ++i) {
        const uint64_t h = mix64((ends[i] << 20) + ids[i]);
        s += h;
        x ^= h;
    }
    *dsum = s;
    *dxor = x;
}

/* ---- std::mt19937_64 and the reference's random trial generators --------
 * The engine is the published MT19937-64 algorithm (parameters of
 * std::mt19937_64). The draws restate tests/support/oracle.hpp:46-67 so the
 * randomised trials of tests/acceptance/acceptance_main.cpp:116-169 can be
 * replayed bit-for-bit. */
typedef struct { uint64_t mt[312]; int mti; } orc_mt64;

void orc_mt64_seed(orc_mt64 *r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = 312;
}

uint64_t orc_mt64_next(orc_mt64 *r) {
    static const uint64_t mag01[2] = {0ull, 0xB5026F5AA96619E9ull};
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    uint64_t x;
    if (r->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ mag01[x & 1];
        }
        for (; i < 311; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[x & 1];
        }
        x = (r->mt[311] & UM) | (r->mt[0] & LM);
        r->mt[311] = r->mt[155] ^ (x >> 1) ^ mag01[x & 1];
        r->mti = 0;
    }
    x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    return x;
}

size_t orc_mt64_size(void) { return sizeof(orc_mt64); }

/* testsupport::random_dictionary (tests/support/oracle.hpp:46-60).
 * Writes up to max_count words into concat/offs; returns the word count. */
uint32_t orc_random_dictionary(orc_mt64 *r, uint32_t max_count, uint32_t min_len, uint32_t max_len,
                               const char *alphabet, uint32_t asize, uint8_t *concat, uint64_t *offs) {
    const uint64_t count = 1 + orc_mt64_next(r) % max_count;
    uint32_t have = 0;
    uint8_t word[4096];
    offs[0] = 0;
    while (have < count) {
        const uint64_t len = min_len + orc_mt64_next(r) % (uint64_t)(max_len - min_len + 1);
        for (uint64_t k = 0; k < len; ++k) word[k] = (uint8_t)alphabet[orc_mt64_next(r) % asize];
        int dup = 0;
        for (uint32_t w = 0; w < have && !dup; ++w)
            if (offs[w + 1] - offs[w] == len && memcmp(concat + offs[w], word, len) == 0) dup = 1;
        if (!dup) {
            memcpy(concat + offs[have], word, len);
            offs[have + 1] = offs[have] + len;
            ++have;
        } else if (orc_mt64_next(r) % 4 == 0) {
            break;
        }
    }
    return have;
}

/* testsupport::random_input (tests/support/oracle.hpp:62-67); returns length. */
uint64_t orc_random_input(orc_mt64 *r, uint64_t max_len, const char *alphabet, uint32_t asize, uint8_t *out) {
    const uint64_t len = orc_mt64_next(r) % (max_len + 1);
    for (uint64_t i = 0; i < len; ++i) out[i] = (uint8_t)alphabet[orc_mt64_next(r) % asize];
    return len;
}
