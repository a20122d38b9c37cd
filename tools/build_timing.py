"""Host build time (acg_build: NFA + dense DFA + filter) per BASELINE config dictionary."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_7294_b200 import acmatch as am, synth

cfgs = [int(x) for x in sys.argv[1:]] or [0, 1, 2, 3, 4]
for k in cfgs:
    w = synth.CONFIGS[k]
    concat, offs = synth.patterns(w)
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        a = am.Automaton.from_arrays(concat, offs)
        best = min(best, time.perf_counter() - t)
    print(f"cfg{k}: patterns {w.patterns} states {a.state_count()} build {best * 1e3:.1f} ms (best of 3, "
          f"{os.cpu_count()} cpus)")
