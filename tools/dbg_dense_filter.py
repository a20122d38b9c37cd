"""Debug: FILTER mode only on the dense text, repeated (for compute-sanitizer)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import oracle
from paper_1403_7294_b200 import acmatch as am, synth, _lib

rng = np.random.default_rng(9)
words = [np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, 16)].tobytes() for _ in range(8)] + [b"A" * 16, b"A" * 17, b"A" * 20]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else (24 << 20) // 16
text = np.frombuffer(b"".join(words[int(i)] for i in rng.integers(0, len(words), reps)), np.uint8).copy()
concat, offs = synth.pack_patterns(words)
a = am.Automaton.from_arrays(concat, offs)
oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
okey = oe.astype(np.uint64) * 16 + oi
s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
s.set_mode(am.MODE_FILTER)
s.run_host(text)
ids, ends = s.records()
key = ends.astype(np.uint64) * 16 + ids
print('replays', _lib.acg().acg_scanner_replays(s._h), 'n', text.size, 'equal', np.array_equal(key, okey), key.size, okey.size)
