"""Debug: FILTER mode on the dense back-to-back-pattern text (test_filter_dense_matches_grow_record_buffer)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import oracle
from paper_1403_7294_b200 import acmatch as am, synth, _lib

rng = np.random.default_rng(9)
def rand_dna(rng, n):
    return np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, n)]
words = [rand_dna(rng, 16).tobytes() for _ in range(8)] + [b"A" * 16, b"A" * 17, b"A" * 20]
reps = (24 << 20) // 16
text = np.frombuffer(b"".join(words[int(i)] for i in rng.integers(0, len(words), reps)), np.uint8).copy()
concat, offs = synth.pack_patterns(words)
a = am.Automaton.from_arrays(concat, offs)
o = oracle.OracleAutomaton(concat, offs)
oi, oe, _, cnt = o.scan(text, counts=True)
okey = oe.astype(np.uint64) * 16 + oi
for mode in (am.MODE_FILTER, am.MODE_EXACT, am.MODE_SPARSE):
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.set_mode(mode)
    for rep in range(2):
        s.run_host(text)
        ids, ends = s.records()
        key = ends.astype(np.uint64) * 16 + ids
        print(mode, rep, s.last_mode(), 'replays', _lib.acg().acg_scanner_replays(s._h) if hasattr(s, '_h') else '?',
              'gpu', key.size, 'oracle', okey.size, 'equal', np.array_equal(key, okey),
              'unsorted', int(np.sum(key[1:] <= key[:-1])), 'dups', key.size - np.unique(key).size,
              'missing', np.setdiff1d(okey, key).size, 'extra', np.setdiff1d(key, okey).size,
              'counts_eq', np.array_equal(s.pattern_counts(), cnt))
        if not np.array_equal(key, okey):
            d = np.nonzero(key[:min(key.size, okey.size)] != okey[:min(key.size, okey.size)])[0]
            if d.size:
                i = d[0]
                print('  first diff', i, 'gpu', [(int(k >> 4), int(k & 15)) for k in key[i-3:i+3]], 'ora', [(int(k >> 4), int(k & 15)) for k in okey[i-3:i+3]])
            ex = np.setdiff1d(key, okey)
            print('  extra sample', [(int(k >> 4), int(k & 15)) for k in ex[:10]])
