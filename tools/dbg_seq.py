"""Debug: replay the GPU test order that precedes the dense filter case, then diagnose it."""
import os
import sys
import numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle
from paper_1403_7294_b200 import acmatch as am, synth, _lib
import test_gpu_filter as tf

pre = sys.argv[1] if len(sys.argv) > 1 else "all"
if pre in ("all", "events"):
    import test_gpu_events as te
    te.test_homopolymer_dense_output_overflows_pool_then_replays()
    for sd in range(3):
        try:
            te.test_density_shift_between_runs_uses_pool_blocks(sd)
        except TypeError:
            pass
if pre in ("all", "filter"):
    for sd in range(6):
        tf.test_filter_random_dictionary_with_planted_matches(sd)
    tf.test_filter_matches_at_text_edges_and_odd_lengths()
    tf.test_filter_shortest_eligible_patterns()
    tf.test_filter_non_acgt_bytes_in_and_near_matches()
print("pre done", pre, flush=True)
rng = np.random.default_rng(9)
words = [tf.rand_dna(rng, 16).tobytes() for _ in range(8)] + [b"A" * 16, b"A" * 17, b"A" * 20]
reps = (24 << 20) // 16
text = np.frombuffer(b"".join(words[int(i)] for i in rng.integers(0, len(words), reps)), np.uint8).copy()
concat, offs = synth.pack_patterns(words)
a = am.Automaton.from_arrays(concat, offs)
oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
okey = oe.astype(np.uint64) * 16 + oi
s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
s.set_mode(am.MODE_FILTER)
for rep in range(3):
    s.run_host(text)
    ids, ends = s.records()
    key = ends.astype(np.uint64) * 16 + ids
    ok = np.array_equal(key, okey)
    print('rep', rep, 'replays', _lib.acg().acg_scanner_replays(s._h), 'gpu', key.size, 'ora', okey.size, 'equal', ok,
          'unsorted', int(np.sum(key[1:] <= key[:-1])), 'dups', key.size - np.unique(key).size,
          'missing', np.setdiff1d(okey, key).size, 'extra', np.setdiff1d(key, okey).size,
          'counts_eq', np.array_equal(s.pattern_counts(), cnt), flush=True)
    if not ok:
        m = min(key.size, okey.size)
        d = np.nonzero(key[:m] != okey[:m])[0]
        if d.size:
            i = int(d[0])
            print('  first diff', i, 'gpu', [(int(k >> 4), int(k & 15)) for k in key[i-3:i+4]])
            print('             ora', [(int(k >> 4), int(k & 15)) for k in okey[i-3:i+4]])
        ex = np.setdiff1d(key, okey)
        print('  extra', [(int(k >> 4), int(k & 15)) for k in ex[:12]], 'last', [(int(k >> 4), int(k & 15)) for k in ex[-4:]])
        mi = np.setdiff1d(okey, key)
        print('  missing', [(int(k >> 4), int(k & 15)) for k in mi[:12]])
        u, c = np.unique(key, return_counts=True)
        print('  dup sample', [(int(k >> 4), int(k & 15), int(n)) for k, n in zip(u[c > 1][:8], c[c > 1][:8])])
