"""Experiments: time the pipelined host scan (acg_scan_pipelined) per call and per phase."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1403_7294_b200 import acmatch as am, synth

cfg, mib, piece = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 256
w = synth.CONFIGS[cfg].scaled(mib << 20) if mib else synth.CONFIGS[cfg]
concat, offs = synth.patterns(w)
a = am.Automaton.from_arrays(concat, offs)
h = torch.empty(w.n, dtype=torch.uint8, pin_memory=True)
synth.text(w, out=h.numpy())
t = time.perf_counter()
_, _, _, m, _ = am.scan_pipelined(a, h.numpy(), piece_bytes=piece << 20)
print("counts-only first call", time.perf_counter() - t, "m", m, flush=True)
out = torch.empty(m + 1024, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
for i in range(3):
    t = time.perf_counter()
    am.scan_pipelined(a, h.numpy(), piece_bytes=piece << 20, out=out)
    dt = time.perf_counter() - t
    print(f"list call {i}: {dt*1e3:.1f} ms  {w.n/dt/1e9:.2f} GB/s text, {8*m/dt/1e9:.2f} GB/s records", flush=True)
