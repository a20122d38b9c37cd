"""Output step: cmd_match's TSV / JSON output of a full
match list formatted on the GPU (acg_scanner_format windows; device time per
window with CUDA events, plus the D2H of the text) against the reference's
own formatting loop (oracle/_ref: the reference scan printed as cmd_match's
TSV, timed end to end on a bounded sample).
usage: python tools/output_bench.py [cfg] [MiB]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_1403_7294_b200 import acmatch as am, synth, _lib
import ctypes as C

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mib = int(sys.argv[2]) if len(sys.argv) > 2 else 0
w = synth.CONFIGS[cfg] if not mib else synth.CONFIGS[cfg].scaled(mib << 20)
concat, offs = synth.patterns(w)
a = am.Automaton.from_arrays(concat, offs)
h = torch.empty(w.n, dtype=torch.uint8, pin_memory=True)
synth.text(w, out=h.numpy())
d = h.cuda()
s = am.Scanner(a, 0, am.SCAN_LIST)
for _ in range(2):
    s.run(d.data_ptr(), w.n)
    s.sync()
m = s.match_count()
res = {"workload": w.name, "matches": m}
for fmt, f in (("tsv", 0), ("json", 1)):
    win = 1 << 24
    nb_tot, dev_ms = 0, 0.0
    t0 = time.perf_counter()
    for first in range(0, m, win):
        cnt = min(win, m - first)
        nb = C.c_uint64()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = _lib.acg().acg_scanner_format(s._h, f, first, cnt, None, 0, C.byref(nb))  # format on the device
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0
        dev_ms += e0.elapsed_time(e1)
        nb_tot += nb.value
    host_s = time.perf_counter() - t0
    res[fmt] = {"bytes": nb_tot, "format_s_incl_sync": round(host_s, 4),
                "GBps_text_out": round(nb_tot / host_s / 1e9, 2), "records_per_s": round(m / host_s / 1e6, 1)}
# the whole output step to a file descriptor (GPU format + D2H through pinned staging + write())
for fmt in ("tsv", "json"):
    t0 = time.perf_counter()
    nb = s.write_matches("/dev/null", fmt)
    dt = time.perf_counter() - t0
    res[fmt]["write_matches_s"] = round(dt, 4)
    res[fmt]["write_matches_GBps"] = round(nb / dt / 1e9, 2)
# the reference: scan + cmd_match's TSV loop on a bounded sample
sample = min(w.n, 16 << 20)
r = oracle.RefAutomaton(concat, offs)
t0 = time.perf_counter()
ref_tsv = r.match_tsv(h.numpy()[:sample])
ref_s = time.perf_counter() - t0
t0 = time.perf_counter()
recs = r.scan(h.numpy()[:sample])
scan_s = time.perf_counter() - t0
res["reference_tsv_sample"] = {"sample_bytes": sample, "bytes": len(ref_tsv), "scan_plus_format_s": round(ref_s, 3),
                               "scan_only_s": round(scan_s, 3),
                               "format_records_per_s": round(len(recs[0]) / max(ref_s - scan_s, 1e-9) / 1e6, 2)}
print(json.dumps(res), flush=True)
