"""run_partitioned wall time: the GPU-native drop-in (acg_run_partitioned,
device merge) against the reference's own run_partitioned (oracle/_ref: host
threads, heap merge) on the same dictionary/text, per worker count."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle
from paper_1403_7294_b200 import acmatch as am, synth

cfg, mib = int(sys.argv[1]), int(sys.argv[2])
workers = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,4,16").split(",")]
w = synth.CONFIGS[cfg].scaled(mib << 20)
text = synth.text(w)
concat, offs = synth.patterns(w)
pats = am.make_patterns(synth.pattern_list(concat, offs))
am.run_partitioned(pats, text[: 1 << 20], 2, records=False)  # warm-up (device init, pools)
for k in workers:
    t = time.perf_counter()
    r = am.run_partitioned(pats, text, k, records=False)
    ours = time.perf_counter() - t
    cap = len(r.ids) + 16
    ids = np.zeros(cap, np.uint32)
    ends = np.zeros(cap, np.uint64)
    m, wall, launched = C.c_uint64(), C.c_double(), C.c_uint32()
    t = time.perf_counter()
    rc = oracle.ref().ref_run_partitioned(oracle._ptr(concat), oracle._ptr(offs), len(offs) - 1, oracle._ptr(text),
                                          text.size, k, oracle._ptr(ids), oracle._ptr(ends), cap, C.byref(m),
                                          C.byref(wall), C.byref(launched))
    ref = time.perf_counter() - t
    same = rc == 0 and m.value == len(r.ids) and np.array_equal(ids[:m.value], r.ids) and np.array_equal(ends[:m.value], r.ends)
    print(f"cfg{cfg} {mib} MiB workers {k}: matches {len(r.ids)}; GPU-native total {r.total_wall_s*1e3:.1f} ms "
          f"(slowest build {max(r.per_worker_build_s)*1e3:.1f} ms, slowest device scan "
          f"{max(r.per_worker_gpu_scan_s)*1e3:.2f} ms, H2D {r.h2d_gpu_s*1e3:.2f} ms, device merge "
          f"{r.merge_gpu_s*1e3:.2f} ms, read-back {r.d2h_s*1e3:.1f} ms; call {ours*1e3:.1f} ms) | reference "
          f"total_wall_s {wall.value*1e3:.1f} ms (call {ref*1e3:.1f} ms) | identical {same}", flush=True)
