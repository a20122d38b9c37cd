"""CPU: pin the oracle (oracle/ac_oracle.c, the plain-C restatement) against
the reference's known answers and against the reference itself.

Pins, in order of strength:
  * tests/golden/known_answers.json — full match lists + failure follows the
    reference produced (oracle/make_goldens.py), incl. the reference's worked
    example and its randomized trials;
  * tests/golden/configs_small.json — every BASELINE config at 2 MiB: record
    count, digest, follows, per-pattern counts from the reference;
  * live comparison with oracle/_ref/libacref.so (the reference compiled from
    /root/reference) on fresh randomized trials, when the library is present.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from paper_1403_7294_b200 import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name: str) -> list[dict]:
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)["cases"]


KNOWN = _load("known_answers.json")
SMALL = _load("configs_small.json")


@pytest.mark.parametrize("case", KNOWN, ids=[c["name"] for c in KNOWN])
def test_oracle_known_answers(case):
    words = [bytes.fromhex(w) for w in case["patterns"]]
    text = bytes.fromhex(case["text"])
    a = oracle.OracleAutomaton.from_words(words)
    assert a.state_count() == case["states"]
    ids, ends, fol, _ = a.scan(text)
    assert [[int(i), int(e)] for i, e in zip(ids, ends)] == case["records"]
    assert fol == case["follows"]
    # the brute-force matcher agrees on the match list
    nid, nend = oracle.naive_find_all(words, text)
    assert np.array_equal(nid, ids) and np.array_equal(nend, ends)


def test_known_answer_classic_example():
    """The reference's worked example (test_aho_corasick.cpp Scan.FindsOverlappingKeywords shape)."""
    case = next(c for c in KNOWN if c["name"] == "classic-ushers")
    assert case["records"] == [[1, 3], [2, 5]]  # SHE ends at 3, HERS at 5 in "USHERS"
    assert case["states"] == 10


@pytest.mark.parametrize("case", SMALL, ids=[c["name"] for c in SMALL])
def test_oracle_configs_small(case):
    w = next(x for x in synth.CONFIGS if case["name"].startswith(x.name)).scaled(case["n"])
    concat, offs = synth.patterns(w)
    t = synth.text(w)
    a = oracle.OracleAutomaton(concat, offs)
    ids, ends, fol, counts = a.scan(t, counts=True)
    assert a.state_count() == case["states"]
    assert len(ids) == case["m"]
    assert fol == case["follows"]
    assert oracle.digest(ids, ends) == (case["dsum"], case["dxor"])
    assert hashlib.sha256(counts.astype("<u8").tobytes()).hexdigest() == case["counts_sha256"]
    if "counts" in case:
        assert [int(x) for x in counts] == case["counts"]


def test_oracle_windowed_scan_composes():
    """Windows with a max_len halo reproduce the whole-text scan (the chunking
    rule the GPU path and the golden generator rely on)."""
    w = synth.CONFIGS[4].scaled(1 << 18)
    concat, offs = synth.patterns(w)
    t = synth.text(w)
    a = oracle.OracleAutomaton(concat, offs)
    ids, ends, fol, _ = a.scan(t)
    halo = a.max_len()
    parts_i, parts_e, fsum = [], [], 0
    step = 10_007
    for lo in range(0, t.size, step):
        start = max(0, lo - halo)
        i, e, f, _ = a.scan(t[:min(lo + step, t.size)], start=start, emit_from=lo)
        parts_i.append(i)
        parts_e.append(e)
        _, _, fpre, _ = a.scan(t[:lo], start=start, emit_from=lo) if lo else (None, None, 0, None)
        fsum += f - fpre
    assert np.array_equal(np.concatenate(parts_i), ids)
    assert np.array_equal(np.concatenate(parts_e), ends)
    assert fsum == fol


needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("seed", range(0, 400, 7))
def test_oracle_matches_reference_random_trials(seed):
    words, text = oracle.oracle_trial(seed)
    a = oracle.OracleAutomaton.from_words(words)
    r = oracle.RefAutomaton.from_words(words)
    ids, ends, fol, _ = a.scan(text)
    rids, rends, rfol = r.scan(text)
    assert np.array_equal(ids, rids) and np.array_equal(ends, rends) and fol == rfol
    assert a.state_count() == r.state_count()
    for s in range(a.state_count()):
        assert a.failure(s) == r.failure(s)
        assert a.depth(s) == r.depth(s)
        assert a.outputs(s) == r.outputs(s)
        assert a.transitions(s) == r.transitions(s)


@needs_ref
def test_oracle_mt64_replays_reference_trial_generator():
    """The oracle's std::mt19937_64 replay draws the reference's own trials."""
    for seed in (1, 17, 12345):
        words, text = oracle.oracle_trial(seed)
        rwords, rtext = oracle.ref_random_trial(seed)
        assert words == rwords and text == rtext


@needs_ref
def test_oracle_full_byte_alphabet_against_reference():
    rng = np.random.default_rng(7)
    words = sorted({bytes(rng.integers(0, 256, rng.integers(1, 6), dtype=np.uint8)) for _ in range(300)})
    text = rng.integers(0, 256, 200_000, dtype=np.uint8).tobytes() + b"".join(words[:50])
    a = oracle.OracleAutomaton.from_words(words)
    r = oracle.RefAutomaton.from_words(words)
    ids, ends, fol, _ = a.scan(text)
    rids, rends, rfol = r.scan(text)
    assert np.array_equal(ids, rids) and np.array_equal(ends, rends) and fol == rfol


def test_golden_fixtures_cover_every_config():
    full = _load("configs_full.json")
    assert {c["name"] for c in full} == {w.name for w in synth.CONFIGS}
    assert all(c["n"] == w.n for c, w in zip(full, synth.CONFIGS))
    small = {c["name"].split("@")[0] for c in SMALL}
    assert small == {w.name for w in synth.CONFIGS}
