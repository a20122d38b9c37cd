/*
 * acg.h — C ABI of the B200 Aho-Corasick text scan (libacg.so).
 *
 * The reference (/root/reference, header-only C++20 `acmatch`) has no FFI; its
 * scan path is the inline C++ API in proj/include/acmatch/aho_corasick.hpp.
 * Each entry point below replaces one piece of that API (cited file:line,
 * relative to /root/reference/proj). The C++ drop-in headers in
 * include/acmatch/ are a thin inline layer over these functions, and
 * INTEGRATION.md shows the ctypes binding.
 *
 * Conventions: functions returning int return ACG_OK (0) or an ACG_ERR_*
 * code; the thread-local message of the last failure is acg_last_error().
 * Plain pointers and sizes only. All handles are opaque and freed by the
 * caller. An acg_automaton is immutable after acg_build and may be scanned
 * from any number of threads concurrently (aho_corasick.hpp:50-52); an
 * acg_scanner is single-user.
 */
#ifndef ACG_H_
#define ACG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ACG_OK = 0,
    ACG_ERR_EMPTY_DICTIONARY = 1,     /* acmatch::EmptyDictionaryError (errors.hpp:21-24) */
    ACG_ERR_EMPTY_PATTERN = 2,        /* acmatch::EmptyPatternError (errors.hpp:15-18) */
    ACG_ERR_INVALID = 3,              /* acmatch::Error (errors.hpp:9-12) */
    ACG_ERR_INVALID_WORKER_COUNT = 4, /* acmatch::InvalidWorkerCountError (errors.hpp:27-30) */
    ACG_ERR_CUDA = 5,                 /* new: CUDA failure (acmatch::DeviceError) */
    ACG_ERR_OUT_OF_MEMORY = 6,        /* new: device allocation failure */
    ACG_ERR_NO_DEVICE = 7,            /* new: no usable sm_100 device */
    ACG_ERR_IO = 9                    /* acmatch::IoError (errors.hpp; io.hpp:27-29, 71-76) */
};

/* scan flags */
enum {
    ACG_SCAN_LIST = 1u,   /* produce the (end, id) match list */
    ACG_SCAN_COUNTS = 2u, /* produce per-pattern occurrence counts */
    ACG_SCAN_STATS = 4u,  /* count failure follows exactly as the reference scan (ScanStats) */
    ACG_SCAN_PROFILE = 8u /* record CUDA events around each kernel stage (acg_scanner_kernel_ms) */
};

typedef struct acg_automaton acg_automaton;
typedef struct acg_result acg_result;
typedef struct acg_scanner acg_scanner;

const char* acg_last_error(void);
const char* acg_version(void);

/* ---- build: replaces acmatch::build (aho_corasick.hpp:130-233) ----------
 * Pattern i (id i, dense by construction) is concat[offsets[i], offsets[i+1]).
 * Errors: ACG_ERR_EMPTY_DICTIONARY (:131), ACG_ERR_EMPTY_PATTERN (:133-134).
 * Host-only; no device is touched until the first scan. */
int acg_build(const uint8_t* concat, const uint64_t* offsets, uint32_t n_patterns, acg_automaton** out);
void acg_automaton_destroy(acg_automaton* a);

/* ---- accessors: Automaton (aho_corasick.hpp:58-101), NFA numbering ------- */
uint32_t acg_state_count(const acg_automaton* a);                       /* :60 */
uint32_t acg_pattern_count(const acg_automaton* a);                     /* :62 patterns().size() */
uint32_t acg_max_pattern_length(const acg_automaton* a);
/* goto_transition (:67-74): 1 and *to set when the edge exists, else 0 */
int acg_goto_transition(const acg_automaton* a, uint32_t s, uint8_t b, uint32_t* to);
/* transitions (:77-80): edge count; *bytes/*targets point into the automaton */
uint32_t acg_transitions(const acg_automaton* a, uint32_t s, const uint8_t** bytes, const uint32_t** targets);
uint32_t acg_failure(const acg_automaton* a, uint32_t s);               /* :84-87 */
uint32_t acg_outputs(const acg_automaton* a, uint32_t s, const uint32_t** ids); /* :92-95 */
uint32_t acg_depth(const acg_automaton* a, uint32_t s);                 /* :98-101 */
/* The whole NFA at once (the accessors above for every state): CSR views
 * into the automaton, valid while it lives. Edges of state s are
 * [edge_off[s], edge_off[s+1]) sorted by byte; outputs [out_off[s],
 * out_off[s+1]) ascending. Any pointer argument may be NULL. */
int acg_nfa_arrays(const acg_automaton* a, const uint32_t** fail, const uint32_t** depth, const uint32_t** edge_off,
                   const uint8_t** edge_byte, const uint32_t** edge_to, const uint32_t** out_off, const uint32_t** out_ids);
/* next_state (:238-245) */
uint32_t acg_next_state(const acg_automaton* a, uint32_t s, uint8_t b);

/* Optional profile-guided layout: renumber the device DFA so that the states
 * most visited on `sample` are the shared-memory-resident ones. Results are
 * unaffected; only speed. Must be called before the first scan. */
int acg_optimize_layout(acg_automaton* a, const uint8_t* sample, uint64_t n);

/* Diagnostics: cap the number of shared-memory-resident DFA rows (0 = as
 * many as fit). Exercises the cold paths on small automata. Must be called
 * before the first scan. */
int acg_set_hot_limit(acg_automaton* a, uint32_t max_hot_rows);

/* ---- one-shot host scan: replaces acmatch::scan (aho_corasick.hpp:250-277) -
 * Host text in, host results out (H2D, device scan, D2H inside).
 * Records are ordered by (end, pattern_id) (aho_corasick.hpp:38-41). */
int acg_scan(const acg_automaton* a, const uint8_t* text, uint64_t n, uint32_t flags, acg_result** out);
uint64_t acg_result_match_count(const acg_result* r);       /* match_count (:280-282) */
const uint32_t* acg_result_ids(const acg_result* r);        /* MatchRecord::pattern_id, M entries */
const uint64_t* acg_result_ends(const acg_result* r);       /* MatchRecord::end, M entries */
const uint64_t* acg_result_pattern_counts(const acg_result* r); /* P entries (ACG_SCAN_COUNTS) */
uint64_t acg_result_failure_follows(const acg_result* r);   /* ScanStats::failure_follows (:46-48) */
void acg_result_destroy(acg_result* r);

/* ---- device-resident scanning (benchmarks, shards) ----------------------
 * A scanner owns the device workspace for one automaton on one device and
 * reuses it across runs. `d_text` is a device pointer (16-byte aligned) to n
 * bytes; bytes [0, emit_from) are warm-up context only (emit_from must be a
 * multiple of 16, and should be >= the automaton's halo for shard exactness);
 * records carry end = base_offset + position. Runs are enqueued on `stream`
 * (a cudaStream_t, NULL = the scanner's own stream) without host syncs. */
int acg_scanner_create(const acg_automaton* a, int device, uint32_t flags, acg_scanner** out);
void acg_scanner_destroy(acg_scanner* s);
int acg_scanner_run(acg_scanner* s, const uint8_t* d_text, uint64_t n, uint64_t emit_from, uint64_t base_offset,
                    void* stream);
/* End-to-end: copy host text (pinned for full speed) into the scanner's
 * device buffer, then scan it (one copy, then the run, both on `stream`; for
 * copy/scan overlap on large inputs see acg_scan_pipelined). */
int acg_scanner_run_host(acg_scanner* s, const uint8_t* h_text, uint64_t n, void* stream);
/* Waits for the last run; grows the record buffer and re-emits if it overflowed. */
int acg_scanner_sync(acg_scanner* s);
uint64_t acg_scanner_match_count(acg_scanner* s);            /* after sync */
int acg_scanner_records(acg_scanner* s, uint32_t* ids, uint64_t* ends, uint64_t cap);   /* D2H + widen */
int acg_scanner_packed_records(acg_scanner* s, uint64_t* host, uint64_t cap, uint32_t* id_bits);
int acg_scanner_pattern_counts(acg_scanner* s, uint64_t* host_counts);           /* P entries */
/* Packed records [first, first+count) of the list (a window of it; e.g. to
 * stream a long list out in pieces). ACG_ERR_INVALID past the list's end. */
int acg_scanner_copy_records(acg_scanner* s, uint64_t first, uint64_t count, uint64_t* host_packed);
/* device pointers (valid until the next run / destroy) */
const uint64_t* acg_scanner_device_pattern_counts(acg_scanner* s);
const uint64_t* acg_scanner_device_records(acg_scanner* s, uint32_t* id_bits);
uint64_t acg_scanner_failure_follows(acg_scanner* s);
/* Order-independent digest of the record set (key = end*2^20 + id; sum and
 * xor of splitmix64(key)) plus the number of adjacent pairs out of strict
 * (end, id) order. Verification helper. */
int acg_scanner_digest(acg_scanner* s, uint64_t* dsum, uint64_t* dxor, uint64_t* unsorted_pairs);
/* Per-stage device time of the last run in ms: [K1 count walk (K1s or K1x),
 * K1f excursion fix-up (sparse mode; 0 in exact mode), K2 prefix, K3
 * compact+write, K4 pattern counts] (scanner created with ACG_SCAN_PROFILE). */
int acg_scanner_kernel_ms(acg_scanner* s, float* ms5);
/* Turns the per-stage event timing (ACG_SCAN_PROFILE) on or off for the next
 * runs (events are recorded between the stages, so leave it off for timing
 * whole runs). No reference counterpart (the reference times with
 * std::chrono around whole calls, partition.hpp:110-111). */
int acg_scanner_set_profiling(acg_scanner* s, int on);
/* Scan mode. SPARSE walks the truncated hot automaton from shared memory and
 * replays the rare cold excursions exactly; EXACT walks the full DFA in
 * lockstep (hot rows in shared memory, cold rows from L2); FILTER streams the
 * text through a sampled q-gram Bloom prefilter and walks only the 64-byte
 * blocks where a match can end (DNA dictionaries whose shortest pattern has
 * >= 13 bytes and a selective filter). AUTO picks FILTER, else SPARSE, else
 * EXACT from the automaton and the previous run's candidate / excursion
 * rates. All are bit-exact; ACG_SCAN_STATS always runs EXACT. */
enum { ACG_MODE_AUTO = 0, ACG_MODE_SPARSE = 1, ACG_MODE_EXACT = 2, ACG_MODE_FILTER = 3 };
int acg_scanner_set_mode(acg_scanner* s, int mode);
/* Mode of the last run (ACG_MODE_SPARSE / _EXACT / _FILTER) and its event
 * rate: sparse, excursion events per walked byte; filter, passing samples per
 * text byte (-1 before the first sync of that mode). */
int acg_scanner_last_mode(acg_scanner* s, double* event_rate);
/* Which walk kernel the last EXACT run used (diagnostics): 0 = the dense hot
 * rows (KE, or the inline-emission walk), 1 = the compressed hot automaton
 * (KC, csrc/ctab.hpp), 2 = SPARSE-G; -1 for a null scanner. */
int acg_scanner_last_walk(const acg_scanner* s);
/* Copies the P per-pattern counts (u64) into a caller device buffer, enqueued
 * on `stream` (NULL = the stream of the last run) — e.g. for an NCCL all-reduce.
 * Enqueued without a host wait: if the run is later replayed at sync (an
 * overflowed workspace; acg_scanner_replays grows), copy again after the sync.
 * Repeating a synced run on the same input does not replay. */
int acg_scanner_copy_pattern_counts(acg_scanner* s, void* d_dst, void* stream);
/* Number of runs this scanner had to replay (or re-emit) at sync because a
 * workspace buffer sized from earlier runs overflowed; results are exact
 * either way. A benchmark checks it is unchanged across its timed runs. */
uint64_t acg_scanner_replays(const acg_scanner* s);
/* Geometry of the last run: chunks, chunk bytes, and launches issued. */
int acg_scanner_last_geometry(acg_scanner* s, uint64_t* n_chunks, uint64_t* chunk_bytes, uint32_t* launches);
/* Filter-mode eligibility (diagnostics): returns 1 when the sampled q-gram
 * prefilter applies, with its q-gram length and the fraction of random
 * q-grams that pass all Bloom stages; 0 otherwise. */
int acg_automaton_filter_info(const acg_automaton* a, uint32_t* q, double* pass_rate);
/* Device layout of the automaton (diagnostics): states, hot rows in smem, columns. */
int acg_automaton_layout(const acg_automaton* a, uint32_t* n_states, uint32_t* hot_rows, uint32_t* columns,
                         uint32_t* halo, int* alphabet_mode);

/* Compressed hot automaton of the EXACT walk (diagnostics; host only, no
 * device needed): info[5] = {slots, default depth D, hot states,
 * exception entries, 1 if the default takes one more level from the table}; when `text` is given, walks it on the host both with the dense
 * transition table and with the compressed tables exactly as the device walk
 * (KC) does, and returns in *mismatches the positions where the two states
 * differ (0 = the compressed automaton is exact on this text) and in
 * *cold_steps the steps taken from cold state words. Returns 1 when the
 * automaton has a compressed table, 0 when the scheme does not apply. */
int acg_automaton_ctab_check(const acg_automaton* a, const uint8_t* text, uint64_t n, uint32_t* info,
                             uint64_t* mismatches, uint64_t* cold_steps);

/* ---- the paper's dictionary-partitioned run, GPU-native: replaces
 * acmatch::run_partitioned + split_patterns + merge_matches
 * (proj/include/acmatch/partition.hpp:29-170). Same split (contiguous chunks,
 * sizes differ by at most one), one worker per non-empty chunk (machines built
 * concurrently on host threads), the input copied to the device once and
 * scanned by every worker on its own stream, the workers' lists merged ON THE
 * DEVICE (global ids, merge-path rounds) and read back once. Errors:
 * ACG_ERR_INVALID_WORKER_COUNT (worker_count < 1), ACG_ERR_EMPTY_DICTIONARY,
 * else the lowest failing chunk's error. Timings: per launched worker the
 * host build and scan seconds (the reference's fields) and the scan's device
 * time; the whole call's wall time; device times of the H2D copy and merge. */
typedef struct acg_partitioned acg_partitioned;
int acg_run_partitioned(const uint8_t* concat, const uint64_t* offsets, uint32_t n_patterns, const uint8_t* text,
                        uint64_t n, uint32_t worker_count, int device, acg_partitioned** out);
uint64_t acg_partitioned_match_count(const acg_partitioned* r);
const uint32_t* acg_partitioned_ids(const acg_partitioned* r);
const uint64_t* acg_partitioned_ends(const acg_partitioned* r);
int acg_partitioned_timings(const acg_partitioned* r, uint32_t* worker_count, uint32_t* workers_launched,
                            const double** build_s, const double** scan_s, const double** gpu_scan_ms, double* total_s,
                            double* h2d_ms, double* merge_ms, double* d2h_ms);
void acg_partitioned_destroy(acg_partitioned* r);

/* ---- output step: replaces cmd_match's output loop (proj/include/acmatch/
 * cli.hpp:58-76), formatted on the GPU from the device match list ----------
 * ACG_FORMAT_TSV:  "<end>\t<pattern_id>\t<pattern bytes>\n" per record (:71-74)
 * ACG_FORMAT_JSON: the nlohmann dump(-1) of [{"end":..,"pattern":"..",
 *                  "pattern_id":..},...] plus "\n" (:63-69): compact, keys in
 *                  order, strings escaped, invalid UTF-8 replaced by U+FFFD.
 * acg_scanner_format: records [first, first+count) of the last run's list
 * (JSON: "[" before record 0, "]\n" after the last, "," between); *bytes =
 * the text size; host_out NULL = size query; cap < *bytes = ACG_ERR_INVALID.
 * acg_scanner_write_matches: the whole list to a file descriptor, formatted
 * in windows of 2^24 records (*bytes written). */
enum { ACG_FORMAT_TSV = 0, ACG_FORMAT_JSON = 1 };
int acg_scanner_format(acg_scanner* s, int format, uint64_t first, uint64_t count, uint8_t* host_out, uint64_t cap,
                       uint64_t* bytes);
int acg_scanner_write_matches(acg_scanner* s, int format, int fd, uint64_t* bytes);

/* ---- streamed host scan: the match list of a host text of any size handed
 * to a callback window by window, in canonical order, while the next pieces
 * are copied and scanned — for lists larger than host or device memory
 * (cfg4: ~1.7e10 records per 4 GiB). format -1: packed records (count =
 * records, end << *id_bits | id); ACG_FORMAT_TSV / _JSON: cmd_match's output
 * (cli.hpp:58-76) formatted on the GPU (count = bytes; JSON framed across
 * windows). The sink returns 0 to go on; anything else stops the scan
 * (ACG_ERR_INVALID). Per-pattern counts into h_counts (NULL: none). */
typedef int (*acg_sink)(void* user, const void* data, uint64_t count);
int acg_scan_stream(const acg_automaton* a, int device, const uint8_t* h_text, uint64_t n, uint64_t piece_bytes,
                    int format, acg_sink sink, void* user, uint64_t* h_counts, uint64_t* m_out, uint32_t* id_bits);

/* ---- input path: replaces acmatch::load_input / load_patterns
 * (proj/include/acmatch/io.hpp:25-31, :37-65) --------------------------------
 * acg_load_input: the whole file as raw bytes in page-locked host memory
 * (parallel reads; pageable if pinning fails), *n bytes; free with
 * acg_host_free. Errors: ACG_ERR_IO ("cannot open <path>", "read failed"). */
int acg_load_input(const char* path, uint8_t** data, uint64_t* n);
/* acg_load_patterns: one pattern per line — LF split, one trailing CR
 * stripped, empty lines skipped (*skipped_empty), repeated lines dropped
 * keeping the first (*duplicates), dense ids in load order; the dictionary as
 * acg_build takes it (*concat, *offsets[*count+1]; free both with
 * acg_host_free). ACG_ERR_EMPTY_DICTIONARY when no line is left (io.hpp:62-63). */
int acg_load_patterns(const char* path, uint8_t** concat, uint64_t** offsets, uint32_t* count, uint64_t* duplicates,
                      uint64_t* skipped_empty);
void acg_host_free(void* p);

/* ---- pipelined host scan: acmatch::scan (aho_corasick.hpp:250-277) of a
 * host text of any size, with the PCIe copies overlapped: the text is cut into
 * pieces of piece_bytes (0 = 256 MiB) scanned as windows with maxlen-1 bytes
 * of context on two scanners / two streams, so piece k+1's H2D copy and scan
 * run while piece k's records come back. Outputs: *m_out matches; the first
 * min(m, cap) packed records (end << *id_bits | id, canonical order) into
 * h_packed (NULL: counts only); per-pattern counts into h_counts (NULL: none);
 * ScanStats::failure_follows with ACG_SCAN_STATS in flags. Windows as
 * acg_scanner_run: bytes [0, emit_from) are context only (a multiple of 16,
 * >= the halo for shard exactness), ends are base_offset + position. Host
 * buffers are best page-locked (acg_load_input); pageable text is staged. */
int acg_scan_pipelined(const acg_automaton* a, int device, const uint8_t* h_text, uint64_t n, uint64_t emit_from,
                       uint64_t base_offset, uint64_t piece_bytes, uint32_t flags, uint64_t* h_packed, uint64_t cap,
                       uint64_t* h_counts, uint64_t* m_out, uint32_t* id_bits, uint64_t* failure_follows);

/* Tuning knobs (diagnostics / benchmarks): streams per thread U in {1,2,4,8}
 * and threads per block; 0 = default. */
int acg_scanner_set_geometry(acg_scanner* s, uint32_t streams_per_thread, uint32_t threads_per_block,
                             uint64_t chunk_bytes);

#ifdef __cplusplus
}
#endif

#endif /* ACG_H_ */
