"""Experiments: back-to-back vs individually synced scanner runs (exact mode)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1403_7294_b200 import acmatch as am, synth

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mib = int(sys.argv[2]) if len(sys.argv) > 2 else 512
w = synth.CONFIGS[cfg].scaled(mib << 20)
concat, offs = synth.patterns(w)
a = am.Automaton.from_arrays(concat, offs)
h = torch.empty(w.n, dtype=torch.uint8, pin_memory=True)
synth.text(w, out=h.numpy())
d = h.cuda()
order = (am.SCAN_LIST | am.SCAN_COUNTS | am.SCAN_PROFILE, am.SCAN_LIST | am.SCAN_COUNTS)
if len(sys.argv) > 3 and sys.argv[3] == "swap":
    order = order[::-1]
for flags in order + order:
    sc = am.Scanner(a, 0, flags)
    st = torch.cuda.Stream()
    for _ in range(4):
        sc.run(d.data_ptr(), d.numel(), stream=st.cuda_stream)
        sc.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(10):
        sc.run(d.data_ptr(), d.numel(), stream=st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) / 10
    synced = []
    for _ in range(5):
        e0.record(st)
        sc.run(d.data_ptr(), d.numel(), stream=st.cuda_stream)
        e1.record(st)
        sc.sync()
        torch.cuda.synchronize()
        synced.append(e0.elapsed_time(e1))
    km = sc.kernel_ms() if flags & am.SCAN_PROFILE else None
    print(f"flags {flags}: back-to-back {b2b:.3f} ms/run, synced {np.round(synced, 3)} ms, stages {km}, mode {sc.last_mode()}")
    del sc
