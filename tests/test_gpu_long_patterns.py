"""GPU parity for dictionaries with LONG patterns (any length is legal:
reference SPEC.md:110; acmatch::scan, proj/include/acmatch/aho_corasick.hpp:
250-272, has no length limit).

Two input classes the round-1 suite did not cover:
  * FILTER mode with DNA patterns longer than one KQ output region (2 KiB for
    texts under ~4.8 MB): a match found from one region's survivors can end
    many regions later; it must still land in its end's slot range.
  * SPARSE mode with a halo past the 17-bit walk offsets of its event log
    (a ~140 KB pattern): the scan must fall back to EXACT, not corrupt events.
Every case compares the FULL (end, id) list with the oracle, the per-pattern
counts, and the device's own order check (unsorted_pairs == 0).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1403_7294_b200 import acmatch as am
from paper_1403_7294_b200 import synth

pytestmark = pytest.mark.gpu

MODES = {"auto": am.MODE_AUTO, "filter": am.MODE_FILTER, "sparse": am.MODE_SPARSE, "exact": am.MODE_EXACT}


def rand_dna(rng, n):
    return np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, n)]


def check(words, text, mode, expect_mode=None, emit_from=0):
    concat, offs = synth.pack_patterns(words)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.set_mode(MODES[mode])
    s.run_host(text)
    ids, ends = s.records()
    if expect_mode:
        assert s.last_mode()[0] == expect_mode
    _, _, unsorted = s.digest()
    assert unsorted == 0
    oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    assert np.array_equal(ends, oe) and np.array_equal(ids, oi)
    assert np.array_equal(s.pattern_counts(), cnt)
    return len(oi)


def long_dictionary(seed, long_lens=(3000, 6000, 20000)):
    rng = np.random.default_rng(seed)
    words = sorted({rand_dna(rng, int(rng.integers(13, 65))).tobytes() for _ in range(50)})
    longs = [rand_dna(rng, L).tobytes() for L in long_lens]
    text = rand_dna(rng, 1 << 20)
    for w in words + longs:
        for _ in range(3):
            p = int(rng.integers(0, text.size - len(w)))
            text[p:p + len(w)] = np.frombuffer(w, np.uint8)
    # a long pattern's prefix and suffix are also patterns (overlapping ends)
    words += longs + [longs[0][:40], longs[1][-40:]]
    return words, text


@pytest.mark.parametrize("mode", ["filter", "auto"])
@pytest.mark.parametrize("seed", range(3))
def test_filter_patterns_longer_than_a_region(mode, seed):
    words, text = long_dictionary(seed)
    a = am.Automaton.from_arrays(*synth.pack_patterns(words))
    assert a.filter_info()["eligible"]
    concat, offs = synth.pack_patterns(words)
    m = check(words, text, mode, expect_mode="filter")
    ids, _, _, _ = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    assert m > 0 and {len(words) - 5, len(words) - 4, len(words) - 3} <= set(ids.tolist())  # the long ones occur


def test_filter_long_pattern_spanning_many_regions_at_text_end():
    rng = np.random.default_rng(7)
    long = rand_dna(rng, 9000)
    text = rand_dna(rng, 64 << 10)
    text[-9000:] = long
    text[100:9100] = long
    words = [long.tobytes()] + [rand_dna(rng, 20).tobytes() for _ in range(20)]
    check(words, text, "filter", expect_mode="filter")


@pytest.mark.parametrize("mode", ["sparse", "auto", "exact"])
def test_pattern_longer_than_sparse_walk(mode):
    """One ~140 KB DNA pattern (halo > 2^17 - 320) plus short ones: sparse mode
    cannot encode the walk offsets and must run EXACT."""
    rng = np.random.default_rng(3)
    big = rand_dna(rng, 140_000)
    shorts = sorted({rand_dna(rng, int(rng.integers(6, 12))).tobytes() for _ in range(40)})
    text = rand_dna(rng, 1 << 20)
    for p in (5, 400_000, text.size - big.size):
        text[p:p + big.size] = big
    for w in shorts:
        p = int(rng.integers(0, text.size - len(w)))
        text[p:p + len(w)] = np.frombuffer(w, np.uint8)
    words = shorts + [big.tobytes(), big[:1000].tobytes()]
    check(words, text, mode, expect_mode="exact")


def test_pattern_just_inside_sparse_walk():
    """A halo just below the sparse limit still runs SPARSE, bit-exact."""
    rng = np.random.default_rng(4)
    big = rand_dna(rng, (1 << 17) - 320 - 16)
    shorts = sorted({rand_dna(rng, 8).tobytes() for _ in range(30)})
    text = rand_dna(rng, 1 << 20)
    text[1000:1000 + big.size] = big
    check(shorts + [big.tobytes()], text, "sparse", expect_mode="sparse")


def test_generic_alphabet_long_patterns_exact():
    rng = np.random.default_rng(9)
    alpha = np.frombuffer(b"ACDEFGHIKLMNPQRSTVWY", np.uint8)
    big = alpha[rng.integers(0, 20, 50_000)]
    text = alpha[rng.integers(0, 20, 1 << 20)]
    text[777:777 + big.size] = big
    words = [big.tobytes(), big[:5].tobytes()] + [alpha[rng.integers(0, 20, 4)].tobytes() for _ in range(50)]
    check(words, text, "auto", expect_mode="exact")


def test_pattern_over_16_mib_builds_and_scans():
    """round 1 rejected patterns over 16 MiB; the reference accepts any length."""
    rng = np.random.default_rng(1)
    big = rand_dna(rng, (16 << 20) + 5)
    words = [big.tobytes(), b"ACGT", big[:30].tobytes()]
    a = am.Automaton.from_arrays(*synth.pack_patterns(words))
    assert a.max_pattern_length() == big.size
    text = rand_dna(rng, 1 << 20)
    text[5000:5030] = big[:30]
    check(words, text, "auto")
