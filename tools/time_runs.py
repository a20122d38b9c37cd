"""Experiments: host vs device time of back-to-back scanner runs (cfg1)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1403_7294_b200 import acmatch as am, synth

w = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
concat, offs = synth.patterns(w)
a = am.Automaton.from_arrays(concat, offs)
h = torch.empty(w.n, dtype=torch.uint8, pin_memory=True)
synth.text(w, out=h.numpy())
d = h.cuda()
sc = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS | am.SCAN_PROFILE)
st = torch.cuda.Stream()
for _ in range(3):
    sc.run(d.data_ptr(), d.numel(), stream=st.cuda_stream)
    sc.sync()
print("mode", sc.last_mode(), "kernel_ms", [round(x, 4) for x in sc.kernel_ms()])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for reps in (1, 5, 20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(reps):
        sc.run(d.data_ptr(), d.numel(), stream=st.cuda_stream)
    t1 = time.perf_counter()
    e1.record(st)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"reps {reps}: host enqueue {(t1-t0)/reps*1e3:.3f} ms/run, device {e0.elapsed_time(e1)/reps:.3f} ms/run, wall {(t2-t0)/reps*1e3:.3f}")
