"""Experiments: per-run device time of one scan configuration.
usage: python tools/exact_probe.py CFG MIB MODE [list|counts|both] [bfs|profile] [U] [TPB]
Prints back-to-back and individually synced run times and the stage split."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1403_7294_b200 import acmatch as am, synth

cfg, mib, mode = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
what = sys.argv[4] if len(sys.argv) > 4 else "both"
layout = sys.argv[5] if len(sys.argv) > 5 else "bfs"
U = int(sys.argv[6]) if len(sys.argv) > 6 else 0
tpb = int(sys.argv[7]) if len(sys.argv) > 7 else 0
w = synth.CONFIGS[cfg].scaled(mib << 20) if mib else synth.CONFIGS[cfg]
concat, offs = synth.patterns(w)
a = am.Automaton.from_arrays(concat, offs)
h = torch.empty(w.n, dtype=torch.uint8, pin_memory=True)
synth.text(w, out=h.numpy())
if layout == "profile":
    a.optimize_layout(h.numpy()[: 1 << 20])
d = h.cuda()
flags = {"list": am.SCAN_LIST, "counts": am.SCAN_COUNTS, "both": am.SCAN_LIST | am.SCAN_COUNTS}[what]
sc = am.Scanner(a, 0, flags)
sc.set_mode({"auto": 0, "sparse": 1, "exact": 2, "filter": 3}[mode])
sc.set_geometry(U, tpb, 0)
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
for _ in range(3):
    e0.record(st)
    sc.run(d.data_ptr(), d.numel(), stream=st.cuda_stream)
    e1.record(st)
    sc.sync()
    torch.cuda.synchronize()
    synced.append(e0.elapsed_time(e1))
sc.set_profiling(True)
sc.run(d.data_ptr(), d.numel(), stream=st.cuda_stream)
sc.sync()
km = [round(x, 3) for x in sc.kernel_ms()]
m = sc.match_count() if flags & am.SCAN_LIST else -1
print(f"cfg{cfg} {mib}MiB {mode} {what} {layout} U={U} tpb={tpb}: b2b {b2b:.3f} ms/run, synced {np.round(synced, 3)} ms,"
      f" stages {km}, mode {sc.last_mode()}, m={m}, layout {a.layout()}, replays {sc.replays()}", flush=True)
