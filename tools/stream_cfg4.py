"""The FULL cfg4 match list (4 GiB text, ~1.7e10 records: larger than HBM)
through the public streamed scan (acg_scan_stream), checked against the
reference's full-size golden (tests/golden/configs_full.json: count,
order-independent digest of (end, id), per-pattern counts sha256) and for
canonical order across windows. The digest of each window is computed on the
GPU (torch) from the packed records the sink receives.
usage: python tools/stream_cfg4.py [cfg] [MiB (0 = full)]"""
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_7294_b200 import acmatch as am, synth

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mib = int(sys.argv[2]) if len(sys.argv) > 2 else 0
w = synth.CONFIGS[cfg] if not mib else synth.CONFIGS[cfg].scaled(mib << 20)
concat, offs = synth.patterns(w)
a = am.Automaton.from_arrays(concat, offs)
h = torch.empty(w.n, dtype=torch.uint8, pin_memory=True)
synth.text(w, out=h.numpy())

M64 = (1 << 64) - 1


def signed(c):
    return c - (1 << 64) if c >= 1 << 63 else c


C1, C2 = signed(0xBF58476D1CE4E5B9), signed(0x94D049BB133111EB)


def lshr(z, k):  # logical shift right of int64
    return (z >> k) & ((1 << (64 - k)) - 1)


def mix(z):
    z = (z ^ lshr(z, 30)) * C1
    z = (z ^ lshr(z, 27)) * C2
    return z ^ lshr(z, 31)


state = {"dsum": 0, "dxor": 0, "m": 0, "last": -1, "unsorted": 0}
dev = torch.device("cuda")


def consume(packed, id_bits):
    t = torch.from_numpy(packed.view(np.int64)).to(dev, non_blocking=False)
    ids = t & ((1 << id_bits) - 1)
    ends = lshr(t, id_bits)
    key = ends * (1 << 20) + ids
    z = mix(key)
    state["dsum"] = (state["dsum"] + int(z.sum().item())) & M64
    x = z
    while x.numel() > 1:
        half = x.numel() // 2
        rest = x[2 * half:]
        x = torch.cat([x[:half] ^ x[half:2 * half], rest])
    state["dxor"] ^= int(x[0].item()) & M64 if x.numel() else 0
    first, last = int(packed[0]), int(packed[-1])
    if first <= state["last"]:
        state["unsorted"] += 1
    state["unsorted"] += int((t[1:] <= t[:-1]).sum().item())
    state["last"] = last
    state["m"] += packed.size
    return False


t0 = time.perf_counter()
m, counts = am.scan_stream(a, h.numpy(), consume, counts=True)
dt = time.perf_counter() - t0
sha = hashlib.sha256(np.asarray(counts, dtype="<u8").tobytes()).hexdigest()
g = next(c for c in json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "configs_full.json")))["cases"]
         if c["name"] == w.name and c["n"] == w.n) if not mib else None
res = {"workload": w.name, "text_bytes": w.n, "matches": m, "records_seen": state["m"],
       "seconds": round(dt, 3), "text_GBps": round(w.n / dt / 1e9, 3), "records_GBps": round(8 * m / dt / 1e9, 2),
       "unsorted_pairs": state["unsorted"], "dsum": state["dsum"], "dxor": state["dxor"], "counts_sha256": sha}
if g:
    res["golden"] = ("bit-exact vs reference (count, digest, per-pattern counts)"
                     if (m, state["dsum"], state["dxor"], sha) == (g["m"], g["dsum"], g["dxor"], g["counts_sha256"])
                     else "MISMATCH vs reference golden")
print(json.dumps(res), flush=True)
