"""GPU parity of the EXACT mode's event pipeline (csrc/exact_kernels.cuh:
KE walk -> E1 per-chunk record counts -> K2 prefix -> E2 expansion), on the
inputs that stress its storage: dense output that overflows the first run's
uniform event slabs into the block pool (and the pool itself: replay at sync),
chunks whose density changes between runs of the same geometry (per-chunk
slabs sized from the previous run, overflow into linked pool blocks), states
with long output lists (the warp expansion's binary search), and generic
alphabets. Reference semantics: acmatch::scan (proj/include/acmatch/
aho_corasick.hpp:250-272) — full (end, id) lists and per-pattern counts are
compared with the oracle.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1403_7294_b200 import acmatch as am
from paper_1403_7294_b200 import synth

pytestmark = pytest.mark.gpu


def rand(rng, alpha: bytes, n):
    return np.frombuffer(alpha, np.uint8)[rng.integers(0, len(alpha), n)]


def run(scanner, text):
    scanner.run_host(text)
    ids, ends = scanner.records()
    return ids, ends, scanner.pattern_counts()


def expect(concat, offs, text, got):
    oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    ids, ends, counts = got
    assert np.array_equal(ends, oe) and np.array_equal(ids, oi)
    assert np.array_equal(counts, cnt)


def test_homopolymer_dense_output_overflows_pool_then_replays():
    """A^n with patterns A, AA, ..., A^40: one event per byte, 40 records per
    byte. The first run's uniform slabs (chunk/16) overflow the pool; the run
    is replayed at sync and the result is exact."""
    words = [b"A" * k for k in range(1, 41)] + [b"C" * 3, b"ACGT"]
    concat, offs = synth.pack_patterns(words)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0)
    s.set_mode(am.MODE_EXACT)
    text = np.full(1 << 20, ord("A"), np.uint8)
    text[1000:1004] = np.frombuffer(b"ACGT", np.uint8)
    r0 = s.replays()
    got = run(s, text)
    assert s.last_mode()[0] == "exact"
    expect(concat, offs, text, got)
    assert s.replays() > r0  # the pool overflowed at least once
    r1 = s.replays()
    expect(concat, offs, text, run(s, text))  # second run: per-chunk slabs, no replay
    assert s.replays() == r1


@pytest.mark.parametrize("seed", range(3))
def test_density_shift_between_runs_uses_pool_blocks(seed):
    """Same geometry, different text: slabs sized from run 1's per-chunk counts
    are wrong for run 2 (dense where run 1 was sparse): chunks continue in
    linked pool blocks."""
    rng = np.random.default_rng(seed)
    words = sorted({rand(rng, b"ACGT", int(rng.integers(2, 7))).tobytes() for _ in range(300)})
    words += [b"A" * k for k in range(8, 30)]
    concat, offs = synth.pack_patterns(words)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0)
    s.set_mode(am.MODE_EXACT)
    n = 2 << 20
    t1 = rand(rng, b"ACGT", n)
    t1[: n // 2] = ord("C")  # first half: almost no matches
    expect(concat, offs, t1, run(s, t1))
    t2 = rand(rng, b"ACGT", n)
    t2[: n // 2] = ord("A")  # first half now maximal density
    t2[n // 2:] = ord("T")
    expect(concat, offs, t2, run(s, t2))
    expect(concat, offs, t1, run(s, t1))


def test_long_output_lists_generic_alphabet():
    """Suffix-closed output sets of up to 60 ids (a pattern and all its
    suffixes), protein alphabet, dense in a planted region."""
    rng = np.random.default_rng(5)
    base = rand(rng, b"ACDEFGHIKLMNPQRSTVWY", 60).tobytes()
    words = [base[i:] for i in range(60)] + [rand(rng, b"ACDEFGHIKLMNPQRSTVWY", 3).tobytes() for _ in range(100)]
    words = list(dict.fromkeys(words))
    concat, offs = synth.pack_patterns(words)
    text = rand(rng, b"ACDEFGHIKLMNPQRSTVWY", 1 << 20)
    for p in range(5000, 900_000, 9973):
        text[p:p + 60] = np.frombuffer(base, np.uint8)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0)
    s.set_mode(am.MODE_EXACT)
    expect(concat, offs, text, run(s, text))
    expect(concat, offs, text, run(s, text))


@pytest.mark.parametrize("flags", [am.SCAN_COUNTS, am.SCAN_LIST, am.SCAN_LIST | am.SCAN_COUNTS])
def test_event_pipeline_flags(flags):
    w = synth.CONFIGS[4].scaled(3 << 20)
    concat, offs = synth.patterns(w)
    text = synth.text(w)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0, flags)
    s.set_mode(am.MODE_EXACT)
    s.run_host(text)
    oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    if flags & am.SCAN_LIST:
        ids, ends = s.records()
        assert np.array_equal(ends, oe) and np.array_equal(ids, oi)
        assert s.digest()[2] == 0
    if flags & am.SCAN_COUNTS:
        assert np.array_equal(s.pattern_counts(), cnt)


def test_record_buffer_regrowth_reexpands_events():
    """A later, denser input outgrows the record buffer sized by earlier runs:
    the list is re-expanded from the (intact) events at sync."""
    words = [b"A" * k for k in range(1, 33)]
    concat, offs = synth.pack_patterns(words)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0)
    s.set_mode(am.MODE_EXACT)
    rng = np.random.default_rng(2)
    t1 = rand(rng, b"ACGT", 1 << 20)
    expect(concat, offs, t1, run(s, t1))
    t2 = np.full(1 << 20, ord("A"), np.uint8)
    expect(concat, offs, t2, run(s, t2))
