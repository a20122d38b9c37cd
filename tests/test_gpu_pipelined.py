"""GPU parity of the pipelined host scan (acg_scan_pipelined: pieces scanned
as windows on two scanners/streams, H2D of piece k+1 overlapped with the
read-back of piece k) against the oracle: piece boundaries everywhere (tiny
pieces, pieces that are not a multiple of the halo, a text shorter than one
piece, the empty text), pinned and pageable inputs, counts-only and STATS runs,
a list capacity smaller than the match count, and the file loader feeding it.
Reference semantics: acmatch::scan (proj/include/acmatch/aho_corasick.hpp:250-277)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1403_7294_b200 import acmatch as am
from paper_1403_7294_b200 import synth

pytestmark = pytest.mark.gpu


def unpack(packed, id_bits):
    packed = np.asarray(packed, np.uint64)
    return (packed & np.uint64((1 << id_bits) - 1)).astype(np.uint32), (packed >> np.uint64(id_bits))


@pytest.mark.parametrize("cfg,mib", [(0, 4), (3, 4), (4, 2), (1, 4)])
@pytest.mark.parametrize("piece", [4096, 65552, 1 << 20, 0])
def test_pipelined_matches_oracle(cfg, mib, piece):
    w = synth.CONFIGS[cfg].scaled(mib << 20, min(synth.CONFIGS[cfg].patterns, 2000))
    text = synth.text(w)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    recs, ib, counts, m, _ = am.scan_pipelined(a, text, piece_bytes=piece, list_cap=len(oi) + 5)
    assert m == len(oi)
    ids, ends = unpack(recs, ib)
    assert np.array_equal(ends, oe) and np.array_equal(ids, oi)
    assert np.array_equal(counts, cnt)


def test_pipelined_pinned_input_stats_and_counts_only():
    import torch
    w = synth.CONFIGS[3].scaled(3 << 20, 1500)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    h = torch.empty(w.n - 5, dtype=torch.uint8, pin_memory=True)  # odd length
    synth.text(w, 0, w.n - 5, out=h.numpy())
    text = h.numpy()
    oi, oe, fol, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    recs, ib, counts, m, f = am.scan_pipelined(a, text, piece_bytes=1 << 19, list_cap=len(oi), stats=True)
    ids, ends = unpack(recs, ib)
    assert m == len(oi) and np.array_equal(ends, oe) and np.array_equal(ids, oi)
    assert f == fol and np.array_equal(counts, cnt)
    r2, _, c2, m2, _ = am.scan_pipelined(a, text, piece_bytes=1 << 20)  # counts only, no list
    assert r2 is None and m2 == m and np.array_equal(c2, cnt)
    r3, _, _, m3, _ = am.scan_pipelined(a, text, list_cap=100, counts=False)  # capacity below m
    assert m3 == m and np.array_equal(unpack(r3, ib)[1], oe[:100])


@pytest.mark.parametrize("n", [0, 1, 15, 17, 4095])
def test_pipelined_short_texts(n):
    words = [b"A", b"AC", b"CGT", b"T" * 20]
    concat, offs = synth.pack_patterns(words)
    a = am.Automaton.from_arrays(concat, offs)
    text = np.frombuffer(b"ACGT", np.uint8)[np.random.default_rng(n).integers(0, 4, n)].copy()
    oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    recs, ib, counts, m, _ = am.scan_pipelined(a, text, piece_bytes=64, list_cap=len(oi) + 1)
    ids, ends = unpack(recs, ib)
    assert m == len(oi) and np.array_equal(ends, oe) and np.array_equal(ids, oi) and np.array_equal(counts, cnt)


def test_file_loaders_feed_the_pipelined_scan(tmp_path):
    w = synth.CONFIGS[0].scaled(2 << 20, 300)
    text = synth.text(w)
    concat, offs = synth.patterns(w)
    words = synth.pattern_list(concat, offs)
    (tmp_path / "in.bin").write_bytes(text.tobytes())
    (tmp_path / "p.txt").write_bytes(b"\n".join(words) + b"\n")
    f = am.load_patterns(str(tmp_path / "p.txt"))
    a = am.build(f.patterns)
    inp = am.load_input(str(tmp_path / "in.bin"))
    recs, ib, counts, m, _ = am.scan_pipelined(a, inp, piece_bytes=1 << 18, list_cap=1 << 20)
    oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    ids, ends = unpack(recs, ib)
    assert np.array_equal(ends, oe) and np.array_equal(ids, oi) and np.array_equal(counts, cnt)


@pytest.mark.parametrize("fmt", [None, "tsv", "json"])
@pytest.mark.parametrize("piece", [1 << 16, 0])
def test_streamed_scan_equals_the_whole_list(fmt, piece):
    """acg_scan_stream: windows handed to a callback in canonical order; their
    concatenation is the whole list (packed records) or the whole cmd_match
    output (TSV / JSON framed across windows), for any piece size."""
    w = synth.CONFIGS[3].scaled(1 << 20, 400)
    text = synth.text(w)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    got = []
    m, counts = am.scan_stream(a, text, lambda *x: got.append(x[0].copy() if fmt is None else x[0]) and False,
                               fmt=fmt, piece_bytes=piece, counts=True)
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.run_host(text)
    assert m == s.match_count() and np.array_equal(counts, s.pattern_counts())
    if fmt is None:
        packed, _ = s.packed_records()
        assert np.array_equal(np.concatenate(got) if got else np.zeros(0, np.uint64), packed)
    else:
        assert b"".join(got) == s.format(fmt)


def test_streamed_scan_empty_list_and_stop():
    concat, offs = synth.pack_patterns([b"ZZZZ"])
    a = am.Automaton.from_arrays(concat, offs)
    got = []
    m, _ = am.scan_stream(a, b"ACGT" * 1000, lambda b: got.append(b) and False, fmt="json")
    assert m == 0 and b"".join(got) == b"[]\n"
    w = synth.CONFIGS[3].scaled(1 << 20, 400)
    a2 = am.Automaton.from_arrays(*synth.patterns(w))
    with pytest.raises(am.Error):
        am.scan_stream(a2, synth.text(w), lambda *x: True, piece_bytes=1 << 16)  # the sink stops the scan
