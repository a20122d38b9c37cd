"""GPU parity against the committed golden fixtures (tests/golden/, generated
from the REFERENCE itself by oracle/make_goldens.py).

  * known_answers.json — full match lists and failure follows;
  * configs_small.json — every BASELINE config at 2 MiB;
  * configs_full.json  — every BASELINE config at its FULL size (16 MiB ..
    8 GiB): record count, order-independent digest of the (end, id) list,
    per-pattern counts (sha256) and failure follows. The text is generated
    and scanned in overlapping windows (the multi-GPU shard decomposition,
    paper_1403_7294_b200/shards.py) so match lists far larger than one
    window's record buffer are still checked record by record via the digest;
    every window's list is also checked to be strictly (end, id) ordered.

Both scan modes are covered: SPARSE (truncated automaton + exact excursion
replay) for records/counts and EXACT (STATS) for the failure-follow count.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from paper_1403_7294_b200 import acmatch as am
from paper_1403_7294_b200 import shards, synth

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name: str) -> list[dict]:
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        return []
    with open(path) as f:
        return json.load(f)["cases"]


KNOWN = _load("known_answers.json")
SMALL = _load("configs_small.json")
FULL = _load("configs_full.json")


@pytest.mark.parametrize("case", KNOWN, ids=[c["name"] for c in KNOWN])
def test_gpu_known_answers(case):
    words = [bytes.fromhex(w) for w in case["patterns"]]
    text = bytes.fromhex(case["text"])
    a = am.build(am.make_patterns(words))
    st = am.ScanStats()
    got = am.scan(a, text, st)
    assert [[r.pattern_id, r.end] for r in got] == case["records"]
    assert st.failure_follows == case["follows"]
    assert [[r.pattern_id, r.end] for r in am.scan(a, text)] == case["records"]  # sparse-capable path


def _workload(case: dict) -> synth.Workload:
    base = next(x for x in synth.CONFIGS if case["name"].startswith(x.name))
    w = base.scaled(case["n"]) if case["n"] != base.n else base
    assert (w.kind, w.patterns, w.len_lo, w.len_hi, w.seed) == \
        (case["kind"], case["patterns"], case["len_lo"], case["len_hi"], case["seed"])
    return w


def _windowed_stats(w: synth.Workload, window: int, mode: int, stats: bool) -> dict:
    import torch
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    halo = a.layout()["halo"]
    flags = am.SCAN_LIST | am.SCAN_COUNTS | (am.SCAN_STATS if stats else 0)
    sc = am.Scanner(a, 0, flags)
    sc.set_mode(mode)
    n_win = -(-w.n // window)
    h = torch.empty(window + halo, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(window + halo, dtype=torch.uint8, device="cuda")
    counts = np.zeros(a.pattern_count(), np.uint64)
    m = dsum = dxor = follows = 0
    for r in range(n_win):
        lo = r * window
        sh = shards.Shard(r, max(0, lo - halo), lo, min(w.n, lo + window))
        synth.text(w, sh.start, sh.hi, out=h.numpy())
        d[: sh.window].copy_(h[: sh.window], non_blocking=False)
        shards.run_shard(sc, d.data_ptr(), sh)
        m += sc.match_count()
        s, x, unsorted = sc.digest()
        assert unsorted == 0, f"window {r}: records not in (end, id) order"
        dsum = (dsum + s) & 0xFFFFFFFFFFFFFFFF
        dxor ^= x
        counts += sc.pattern_counts()
        if stats:
            follows += sc.failure_follows()
    out = dict(m=m, dsum=dsum, dxor=dxor, states=a.state_count(),
               counts_sha256=hashlib.sha256(counts.astype("<u8").tobytes()).hexdigest())
    if stats:
        out["follows"] = follows
    return out


def _check(case: dict, got: dict, stats: bool) -> None:
    assert got["states"] == case["states"]
    assert got["m"] == case["m"]
    assert (got["dsum"], got["dxor"]) == (case["dsum"], case["dxor"])
    assert got["counts_sha256"] == case["counts_sha256"]
    if stats:
        assert got["follows"] == case["follows"]


@pytest.mark.parametrize("mode", [am.MODE_AUTO, am.MODE_SPARSE, am.MODE_EXACT], ids=["auto", "sparse", "exact"])
@pytest.mark.parametrize("case", SMALL, ids=[c["name"] for c in SMALL])
def test_gpu_configs_small(case, mode):
    w = _workload(case)
    _check(case, _windowed_stats(w, w.n, mode, stats=False), stats=False)
    if mode == am.MODE_EXACT:
        _check(case, _windowed_stats(w, w.n, mode, stats=True), stats=True)


@pytest.mark.parametrize("case", FULL, ids=[c["name"] for c in FULL])
def test_gpu_configs_full_size(case):
    """BASELINE sizes, checked against the reference's own statistics."""
    w = _workload(case)
    window = min(w.n, 256 << 20)
    _check(case, _windowed_stats(w, window, am.MODE_AUTO, stats=False), stats=False)
    _check(case, _windowed_stats(w, window, am.MODE_EXACT, stats=True), stats=True)
