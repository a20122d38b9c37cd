"""GPU parity of the EXACT walk over the compressed hot automaton (KC,
csrc/ctab.hpp + exact_kernels.cuh: ctab_event_kernel, E1's payload -> rank
mapping): full (end, id) lists and per-pattern counts against the oracle
(reference semantics: acmatch::scan, proj/include/acmatch/
aho_corasick.hpp:250-272), with the hot set capped so that cold state words,
cold output states and T_D defaults that are cold all occur, on texts with
bytes outside the alphabet, at every stream interleave, through shard windows
and after a profile-guided relayout.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1403_7294_b200 import acmatch as am
from paper_1403_7294_b200 import synth

pytestmark = pytest.mark.gpu


def protein(n, patterns):
    w = synth.CONFIGS[3].scaled(n, patterns)
    return synth.text(w), synth.patterns(w)


def check(a, text, concat, offs, walk="ctab", u=0):
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.set_mode(am.MODE_EXACT)
    if u:
        s.set_geometry(streams_per_thread=u)
    oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    for _ in range(2):  # second run: per-chunk event slabs from the first run's counts
        s.run_host(text)
        ids, ends = s.records()
        assert s.last_walk() == walk
        assert np.array_equal(ends, oe) and np.array_equal(ids, oi)
        assert np.array_equal(s.pattern_counts(), cnt)


@pytest.mark.parametrize("limit", [0, 1, 40, 3000])
def test_protein_hot_limits(limit):
    text, (concat, offs) = protein(3 << 20, 5000)
    a = am.Automaton.from_arrays(concat, offs)
    if limit:
        a.set_hot_limit(limit)
    check(a, text, concat, offs)


@pytest.mark.parametrize("u", [1, 2, 4])
def test_protein_interleaves_and_foreign_bytes(u):
    text, (concat, offs) = protein(1 << 20, 3000)
    text = text.copy()
    rng = np.random.default_rng(u)
    text[rng.integers(0, text.size, 3000)] = rng.integers(0, 256, 3000).astype(np.uint8)
    a = am.Automaton.from_arrays(concat, offs)
    a.set_hot_limit(700)
    check(a, text, concat, offs, u=u)


def test_profile_guided_layout():
    text, (concat, offs) = protein(2 << 20, 5000)
    a = am.Automaton.from_arrays(concat, offs)
    a.optimize_layout(text[: 1 << 18])
    check(a, text, concat, offs)


@pytest.mark.parametrize("nsym", [3, 22, 30])
def test_other_alphabets_default_depth_2_and_3(nsym):
    rng = np.random.default_rng(nsym)
    alpha = np.arange(97, 97 + nsym, dtype=np.uint8)
    words = list(dict.fromkeys(alpha[rng.integers(0, nsym, rng.integers(1, 9))].tobytes() for _ in range(4000)))
    concat, offs = synth.pack_patterns(words)
    a = am.Automaton.from_arrays(concat, offs)
    a.set_hot_limit(60)
    text = alpha[rng.integers(0, nsym, 1 << 20)]
    check(a, text, concat, offs)


def test_ragged_sizes_and_shard_windows():
    import torch
    text, (concat, offs) = protein((1 << 20) + 12345, 4000)
    a = am.Automaton.from_arrays(concat, offs)
    a.set_hot_limit(2000)
    for n in (1, 15, 16, 17, 4097, text.size):
        check(a, text[:n], concat, offs)
    halo = a.layout()["halo"]
    d = torch.from_numpy(text).cuda()
    oi, oe, _, _ = oracle.OracleAutomaton(concat, offs).scan(text)
    s = am.Scanner(a, 0, am.SCAN_LIST)
    s.set_mode(am.MODE_EXACT)
    got_i, got_e = [], []
    cuts = [0, 300000 // 16 * 16, 700000 // 16 * 16, text.size]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        start = max(0, lo - halo)
        s.run(d.data_ptr() + start, hi - start, emit_from=lo - start, base_offset=start)
        i, e = s.records()
        assert s.last_walk() == "ctab"
        got_i.append(i)
        got_e.append(e)
    assert np.array_equal(np.concatenate(got_e), oe) and np.array_equal(np.concatenate(got_i), oi)


def test_dense_rows_when_everything_fits(monkeypatch):
    text, (concat, offs) = protein(1 << 19, 300)
    a = am.Automaton.from_arrays(concat, offs)  # all states in the dense hot rows: KE
    check(a, text, concat, offs, walk="dense")
