"""GPU parity of the FILTER scan mode (sampled q-gram Bloom prefilter + exact
block walks; paper_1403_7294_b200/csrc/qfilter.hpp) against the oracle, on
dictionaries where the filter is eligible (DNA, shortest pattern >= 13), with
the cases that stress its exactness argument: matches straddling 64-byte
blocks, 8 KiB chunks and text edges, non-ACGT bytes inside and next to
matches, unaligned lengths, dense matches (many dirty blocks, record-buffer
growth), shard windows, and the shortest eligible patterns (q = 10).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1403_7294_b200 import acmatch as am
from paper_1403_7294_b200 import synth

pytestmark = pytest.mark.gpu


def recs(ids, ends):
    return list(zip(np.asarray(ends).tolist(), np.asarray(ids).tolist()))


def run_filter(words_or_arrays, text, expect_filter=True, emit_from=0):
    if isinstance(words_or_arrays, tuple):
        concat, offs = words_or_arrays
    else:
        concat, offs = synth.pack_patterns(words_or_arrays)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.set_mode(am.MODE_FILTER)
    s.run_host(text)
    ids, ends = s.records()
    if expect_filter:
        assert s.last_mode()[0] == "filter"
    o = oracle.OracleAutomaton(concat, offs)
    oi, oe, _, cnt = o.scan(text, counts=True)
    assert recs(ids, ends) == recs(oi, oe), diff_report(s, ids, ends, oi, oe)
    assert np.array_equal(s.pattern_counts(), cnt)
    return len(oi)


def diff_report(s, ids, ends, oi, oe) -> str:
    """Why two match lists differ (duplicates, missing, extra, first difference)."""
    from paper_1403_7294_b200 import _lib
    key = np.asarray(ends, np.uint64) * np.uint64(1 << 20) + np.asarray(ids, np.uint64)
    okey = np.asarray(oe, np.uint64) * np.uint64(1 << 20) + np.asarray(oi, np.uint64)
    m = min(key.size, okey.size)
    d = np.nonzero(key[:m] != okey[:m])[0]
    first = int(d[0]) if d.size else m
    fmt = lambda ks: [(int(k) >> 20, int(k) & 0xFFFFF) for k in ks]
    return (f"gpu {key.size} oracle {okey.size} replays {_lib.acg().acg_scanner_replays(s._h)} "
            f"mode {s.last_mode()} dups {key.size - np.unique(key).size} "
            f"missing {np.setdiff1d(okey, key).size} extra {np.setdiff1d(key, okey).size} "
            f"unsorted {int(np.sum(key[1:] <= key[:-1]))} first diff {first}: gpu {fmt(key[first:first + 4])} "
            f"oracle {fmt(okey[first:first + 4])} extra {fmt(np.setdiff1d(key, okey)[:6])} "
            f"missing {fmt(np.setdiff1d(okey, key)[:6])}")


def rand_dna(rng, n):
    return np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, n)]


@pytest.mark.parametrize("seed", range(6))
def test_filter_random_dictionary_with_planted_matches(seed):
    rng = np.random.default_rng(seed)
    words = sorted({rand_dna(rng, int(rng.integers(16, 65))).tobytes() for _ in range(500)})
    text = rand_dna(rng, 3 << 20)
    # plant every pattern a few times at random offsets (incl. block/chunk straddles)
    for w in words:
        for _ in range(3):
            p = int(rng.integers(0, text.size - len(w)))
            text[p:p + len(w)] = np.frombuffer(w, np.uint8)
    m = run_filter(words, text)
    assert m >= len(words)


def test_filter_matches_at_text_edges_and_odd_lengths():
    rng = np.random.default_rng(11)
    words = [rand_dna(rng, L).tobytes() for L in (13, 14, 16, 31, 64)]
    for n in (13, 15, 16, 17, 63, 64, 65, 100, 4097, 8191, 8192, 8193, 70001):
        text = rand_dna(rng, n)
        w = words[0]
        text[:13] = np.frombuffer(w, np.uint8)          # match at the very start
        if n >= 26:
            text[n - 13:] = np.frombuffer(w, np.uint8)  # and at the very end
        run_filter(words, text)


def test_filter_shortest_eligible_patterns():
    """min length 13 -> q = 10: the least selective eligible filter."""
    rng = np.random.default_rng(5)
    words = sorted({rand_dna(rng, 13).tobytes() for _ in range(200)})
    text = rand_dna(rng, 1 << 20)
    for i, w in enumerate(words):
        p = (i * 5237) % (text.size - 13)
        text[p:p + 13] = np.frombuffer(w, np.uint8)
    run_filter(words, text)


def test_filter_non_acgt_bytes_in_and_near_matches():
    rng = np.random.default_rng(3)
    words = sorted({rand_dna(rng, int(rng.integers(16, 40))).tobytes() for _ in range(100)})
    text = rand_dna(rng, 1 << 20)
    for i, w in enumerate(words):
        p = 97 + i * 9973
        text[p:p + len(w)] = np.frombuffer(w, np.uint8)
        text[p - 1] = ord("N")                       # escape right before
        if i % 3 == 0:
            text[p + len(w) // 2] = ord("n")          # breaks this occurrence
        if i % 5 == 0:
            text[p + len(w)] = 0                      # NUL right after
    bad = rng.integers(0, text.size, 5000)
    text[bad] = np.frombuffer(b"NRYacgt\x00\xff", np.uint8)[rng.integers(0, 9, bad.size)]
    run_filter(words, text)


def test_filter_dense_matches_grow_record_buffer():
    """Text made of back-to-back pattern copies: nearly every block is dirty
    and > 1M records force the record-buffer growth path."""
    rng = np.random.default_rng(9)
    words = [rand_dna(rng, 16).tobytes() for _ in range(8)] + [b"A" * 16, b"A" * 17, b"A" * 20]
    reps = (24 << 20) // 16
    text = np.frombuffer(b"".join(words[int(i)] for i in rng.integers(0, len(words), reps)), np.uint8).copy()
    m = run_filter(words, text)
    assert m > 1_500_000


def test_filter_cfg1_scaled_vs_oracle():
    w = synth.CONFIGS[1].scaled(8 << 20)
    concat, offs = synth.patterns(w)
    m = run_filter((concat, offs), synth.text(w))
    assert m > 0


def test_filter_shard_windows():
    """emit_from / base_offset windows (the multi-GPU shards) in filter mode."""
    import torch
    w = synth.CONFIGS[1].scaled(6 << 20)
    text = synth.text(w)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    halo = a.layout()["halo"]
    d = torch.from_numpy(text).cuda()
    parts = []
    bounds = [0, 1 << 20, (3 << 20) + 4096, 6 << 20]
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        start = max(0, lo - halo)
        s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
        s.set_mode(am.MODE_FILTER)
        s.run(d[start:hi].data_ptr(), hi - start, emit_from=lo - start, base_offset=start)
        parts.append(s.records())
        assert s.last_mode()[0] == "filter"
    oi, oe, _, _ = oracle.OracleAutomaton(concat, offs).scan(text)
    got_i = np.concatenate([p[0] for p in parts])
    got_e = np.concatenate([p[1] for p in parts])
    assert recs(got_i, got_e) == recs(oi, oe)


def test_filter_not_eligible_falls_back():
    """Short patterns (cfg0: 8..32) are not filter-eligible: FILTER requests run another exact mode."""
    w = synth.CONFIGS[0].scaled(1 << 20, 300)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0, am.SCAN_LIST)
    s.set_mode(am.MODE_FILTER)
    s.run_host(synth.text(w))
    s.sync()
    assert s.last_mode()[0] in ("sparse", "exact")


def test_auto_picks_filter_for_cfg1():
    w = synth.CONFIGS[1].scaled(4 << 20)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0, am.SCAN_LIST)
    s.run_host(synth.text(w))
    s.sync()
    assert s.last_mode()[0] == "filter"


def test_filter_region_sort_paths():
    """Per-region match counts across ORDER's paths: a bitonic round in
    registers (<= 32 per region) and the warp sort in shared memory (33..1024),
    with matches straddling region boundaries (owned by the next region)."""
    rng = np.random.default_rng(21)
    words = sorted({rand_dna(rng, int(rng.integers(16, 30))).tobytes() for _ in range(40)})
    text = rand_dna(rng, 1 << 20)
    p = 0
    while p < text.size - 64:
        w = words[int(rng.integers(0, len(words)))]
        text[p:p + len(w)] = np.frombuffer(w, np.uint8)
        # dense (about 60 per 2 KiB region) in the first half, sparse after
        p += int(rng.integers(len(w), 48)) if p < text.size // 2 else int(rng.integers(200, 900))
    m = run_filter(words, text)
    assert m > 10000


def test_filter_region_too_dense_replays_chunk_pipeline():
    """A homopolymer run gives every region > 1024 matches: the scanner
    replays the run through the per-chunk pipeline, with the same result."""
    rng = np.random.default_rng(22)
    words = [b"A" * 16, b"A" * 24] + [rand_dna(rng, 20).tobytes() for _ in range(10)]
    text = rand_dna(rng, 1 << 20)
    text[100_000:300_000] = ord("A")
    run_filter(words, text)


def test_filter_two_level_cfg2_dictionary():
    """cfg2's 100,000 patterns: the shared-memory filter alone passes too many
    q-grams, so its survivors probe the L2-resident level-2 filter. Parity on
    a scaled text with the full dictionary, planted matches included."""
    w = synth.CONFIGS[2].scaled(8 << 20, 100_000)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    info = a.filter_info()
    assert info["eligible"] and info["q"] == 16
    m = run_filter((concat, offs), synth.text(w))
    assert m > 0


def test_filter_no_phantom_survivors_past_the_text_end():
    """KQ reads the partial last block with zero bytes past the end, whose
    2-bit codes are 'A': an A-homopolymer pattern must not make those samples
    survivors (they were counted but never stored, so V1/V0 read stale slots:
    duplicate records after an earlier scanner left positions in that memory)."""
    rng = np.random.default_rng(21)
    words = [b"A" * 16, b"A" * 23]
    for n in (100, 2048 * 3 + 100, (1 << 20) + 1000):
        text = np.frombuffer(b"CGT", np.uint8)[rng.integers(0, 3, n)].copy()
        text[n // 2:n // 2 + 20] = ord("A")  # one real run: 5 + 0 matches
        m = run_filter(words, text)
        assert m == 5
        concat, offs = synth.pack_patterns(words)
        s = am.Scanner(am.Automaton.from_arrays(concat, offs), 0, am.SCAN_LIST)
        s.set_mode(am.MODE_FILTER)
        s.run_host(text)
        s.sync()
        mode, rate = s.last_mode()
        assert mode == "filter" and rate * n <= 8  # survivors: samples inside the one A-run only
