"""GPU parity: the CUDA scan (through the C ABI) against the oracle.

Mirrors the reference's own tests (paths relative to /root/reference/proj):
known answers of tests/unit/test_aho_corasick.cpp:129-189, the randomised
acceptance criteria 3 and 5 (tests/acceptance/acceptance_main.cpp:116-169),
plus chunk-boundary, escape-byte and shard-window properties the GPU design
adds. The oracle is oracle/ac_oracle.c (pinned to the reference in
tests/test_oracle.py).
"""
import numpy as np
import pytest

import oracle
from paper_1403_7294_b200 import acmatch as am
from paper_1403_7294_b200 import synth

pytestmark = pytest.mark.gpu


def recs(ids, ends):
    return list(zip(np.asarray(ends).tolist(), np.asarray(ids).tolist()))


def gpu_vs_oracle(words, text, stats=True, counts=True):
    a = am.build(am.make_patterns(words))
    flags = am.SCAN_LIST | (am.SCAN_STATS if stats else 0) | (am.SCAN_COUNTS if counts else 0)
    res = am.scan_arrays(a, text, flags)
    o = oracle.OracleAutomaton.from_words(words)
    ids, ends, fol, cnt = o.scan(text, counts=True)
    assert recs(res.ids, res.ends) == recs(ids, ends)
    if stats:
        assert res.failure_follows == fol
    if counts:
        assert np.array_equal(res.counts, cnt)
    return res


# ---- known answers (test_aho_corasick.cpp, test_partition.cpp) -------------
def test_shers_classic():
    a = am.build(am.make_patterns(["HIS", "SHE", "HERS"]))
    assert am.scan(a, b"SHERS") == [am.MatchRecord(1, 2), am.MatchRecord(2, 4)]
    assert am.match_count(am.scan(a, b"SHERS")) == 2


def test_empty_input():
    a = am.build(am.make_patterns(["HIS", "SHE", "HERS"]))
    assert am.scan(a, b"") == []
    st = am.ScanStats()
    assert am.scan(a, b"", st) == [] and st.failure_follows == 0


def test_self_overlapping():
    a = am.build(am.make_patterns(["AA"]))
    assert am.scan(a, b"AAAA") == [am.MatchRecord(0, 1), am.MatchRecord(0, 2), am.MatchRecord(0, 3)]


def test_full_byte_alphabet():
    nul, high = b"\x00\xff", b"\xfe\xff\x80"
    a = am.build(am.make_patterns([nul, high, b"his"]))
    text = high + nul + b"HIS" + nul
    assert am.scan(a, text) == [am.MatchRecord(1, 2), am.MatchRecord(0, 4), am.MatchRecord(0, 9)]


def test_abcabc():
    a = am.build(am.make_patterns(["AB", "BC"]))
    assert am.scan(a, b"ABCABC") == [am.MatchRecord(0, 1), am.MatchRecord(1, 2), am.MatchRecord(0, 4),
                                     am.MatchRecord(1, 5)]


def test_deterministic_repeats():
    r = oracle.MT64(7)
    words = r.random_dictionary(30, 1, 8)
    text = r.random_input(5000)
    a = am.build(am.make_patterns(words))
    assert am.scan(a, text) == am.scan(a, text)


# ---- randomised trials (acceptance criteria 3 and 5) ------------------------
def test_acceptance_oracle_trials():
    """acceptance_main.cpp:116-169: 1000 trials, seeds 0x5eed0000+t; records
    equal the naive oracle; failure follows equal the reference scan's and
    stay <= n."""
    for t in range(1000):
        words, text = oracle.oracle_trial(0x5eed0000 + t)
        a = am.build(am.make_patterns(words))
        res = am.scan_arrays(a, text, am.SCAN_LIST | am.SCAN_STATS)
        nid, nend = oracle.naive_find_all(words, text)
        assert recs(res.ids, res.ends) == recs(nid, nend), f"trial {t}"
        _, _, fol, _ = oracle.OracleAutomaton.from_words(words).scan(text, with_records=False)
        assert res.failure_follows == fol, f"trial {t}"
        assert res.failure_follows <= len(text)


def test_unit_seeds_match_naive():
    """test_aho_corasick.cpp:150-163: seeds 100..159, <=2000 bytes."""
    for seed in range(100, 160):
        r = oracle.MT64(seed)
        words = r.random_dictionary(50, 1, 8)
        text = r.random_input(2000)
        gpu_vs_oracle(words, text)


# ---- alphabet modes and escapes --------------------------------------------
def test_generic_alphabet_random_bytes():
    rng = np.random.default_rng(1)
    for trial in range(20):
        words = list({bytes(rng.integers(0, 256, rng.integers(1, 6), dtype=np.uint8)) for _ in range(40)})
        text = rng.integers(0, 256, 30000, dtype=np.uint8).tobytes()
        # plant some occurrences
        t = bytearray(text)
        for w in words[:10]:
            p = int(rng.integers(0, len(t) - len(w)))
            t[p:p + len(w)] = w
        gpu_vs_oracle(words, bytes(t))


def test_dna_with_escape_bytes():
    """DNA dictionary (dna4 column mode) over text containing N, lowercase, NUL."""
    rng = np.random.default_rng(2)
    alpha = np.frombuffer(b"ACGT", np.uint8)
    text = alpha[rng.integers(0, 4, 100_000)].copy()
    junk = np.frombuffer(b"NacgtX\x00\xff", np.uint8)
    pos = rng.integers(0, text.size, 2000)
    text[pos] = junk[rng.integers(0, junk.size, pos.size)]
    words = [alpha[rng.integers(0, 4, int(rng.integers(3, 9)))].tobytes() for _ in range(200)]
    words = list(dict.fromkeys(words))
    res = gpu_vs_oracle(words, text.tobytes())
    assert len(res.ids) > 0


def test_protein_alphabet():
    w = synth.CONFIGS[3].scaled(2 << 20, 500)
    text = synth.text(w)
    words = synth.pattern_list(*synth.patterns(w))
    gpu_vs_oracle(words, text, stats=False)


# ---- chunking and shard properties ------------------------------------------
MODES = [am.MODE_SPARSE, am.MODE_EXACT, am.MODE_FILTER]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("U", [1, 2, 4, 8])
@pytest.mark.parametrize("chunk", [16, 48, 256, 0])
def test_chunk_geometry_invariance(mode, U, chunk):
    """Any chunk size / interleave / scan mode gives the identical record list (halo exactness)."""
    w = synth.CONFIGS[0].scaled(1 << 20, 300)
    text = synth.text(w)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.set_geometry(U, 0, chunk)
    s.set_mode(mode)
    s.run_host(text)
    ids, ends = s.records()
    want = {am.MODE_SPARSE: ("sparse",), am.MODE_EXACT: ("exact",)}.get(mode, ("sparse", "exact", "filter"))
    assert s.last_mode()[0] in want
    o = oracle.OracleAutomaton(concat, offs)
    oi, oe, fol, cnt = o.scan(text, counts=True)
    assert recs(ids, ends) == recs(oi, oe)
    assert np.array_equal(s.pattern_counts(), cnt)
    st = am.Scanner(a, 0, am.SCAN_COUNTS | am.SCAN_STATS)
    st.set_geometry(0, 0, chunk)
    st.run_host(text)
    assert st.failure_follows() == fol


@pytest.mark.parametrize("mode", MODES)
def test_small_hot_set_forces_cold_excursions(mode):
    """A dictionary whose automaton far exceeds the shared-memory hot set:
    long cold excursions (planted long patterns) replayed exactly."""
    w = synth.CONFIGS[1].scaled(2 << 20, 4000)
    text = synth.text(w)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.set_mode(mode)
    s.run_host(text)
    ids, ends = s.records()
    oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    assert len(oi) > 1000
    assert recs(ids, ends) == recs(oi, oe)
    assert np.array_equal(s.pattern_counts(), cnt)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("hot", [1, 2, 7, 64, 1000])
@pytest.mark.parametrize("k", [0, 3, 4])
def test_tiny_hot_sets(k, hot, mode):
    """Hot set capped to a few rows: nearly every step is a cold excursion
    (event-log overflow -> exact fallback in sparse mode)."""
    w = synth.CONFIGS[k].scaled(256 << 10, 300)
    text = synth.text(w)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    a.set_hot_limit(hot)
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.set_mode(mode)
    s.run_host(text)
    ids, ends = s.records()
    oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    assert recs(ids, ends) == recs(oi, oe)
    assert np.array_equal(s.pattern_counts(), cnt)


def test_shard_windows_concatenate_to_full_scan():
    """Text sharded with a halo (the multi-GPU decomposition) reproduces the
    full scan by plain concatenation, failure follows included."""
    import torch
    w = synth.CONFIGS[4].scaled(3 << 20, 300)
    text = synth.text(w)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    halo = a.layout()["halo"]
    d = torch.from_numpy(text).cuda()
    full = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS | am.SCAN_STATS)
    full.run(d.data_ptr(), text.size)
    fid, fend = full.records()
    parts_i, parts_e, tot_counts, tot_fol = [], [], 0, 0
    bounds = [0, 1 << 20, 1 << 21, 3 << 20]
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        start = max(0, lo - halo)
        buf = d[start:hi]
        s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS | am.SCAN_STATS)
        s.run(buf.data_ptr(), hi - start, emit_from=lo - start, base_offset=start)
        i, e = s.records()
        parts_i.append(i)
        parts_e.append(e)
        tot_counts = tot_counts + s.pattern_counts()
        tot_fol += s.failure_follows()
    assert recs(np.concatenate(parts_i), np.concatenate(parts_e)) == recs(fid, fend)
    assert np.array_equal(tot_counts, full.pattern_counts())
    assert tot_fol == full.failure_follows()


@pytest.mark.parametrize("mode", MODES + [am.MODE_AUTO])
@pytest.mark.parametrize("k", [0, 1, 2, 3, 4])
def test_scaled_configs_vs_oracle(k, mode):
    """Every BASELINE config at a size the oracle finishes in seconds, every mode."""
    w = synth.CONFIGS[k].scaled(4 << 20, min(synth.CONFIGS[k].patterns, 2000))
    text = synth.text(w)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.set_mode(mode)
    s.run_host(text)
    ids, ends = s.records()
    o = oracle.OracleAutomaton(concat, offs)
    oi, oe, _, cnt = o.scan(text, counts=True)
    assert len(ids) == len(oi)
    assert np.array_equal(ids, oi) and np.array_equal(ends, oe)
    assert np.array_equal(s.pattern_counts(), cnt)
    dsum, dxor, unsorted = s.digest()
    assert (dsum, dxor) == oracle.digest(oi, oe) and unsorted == 0


# ---- exact mode: single-pass slabs after the first run ------------------------
@pytest.mark.parametrize("cfg", [0, 3])
def test_exact_single_pass_repeat_runs(cfg):
    """The first EXACT run counts then writes; later runs (record density known)
    walk once into per-chunk slabs and copy them into place. Both must equal
    the oracle, run after run."""
    w = synth.CONFIGS[cfg].scaled(2 << 20, 300)
    text = synth.text(w)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.set_mode(am.MODE_EXACT)
    oi, oe, _, cnt = oracle.OracleAutomaton(concat, offs).scan(text, counts=True)
    for _ in range(3):
        s.run_host(text)
        ids, ends = s.records()
        assert recs(ids, ends) == recs(oi, oe)
        assert np.array_equal(s.pattern_counts(), cnt)


def test_exact_single_pass_slab_overflow():
    """A sparse first text sizes small slabs; a dense second text overflows
    them, and the overflowed chunks are re-walked by the WRITE pass."""
    rng = np.random.default_rng(31)
    dna = np.frombuffer(b"ACGT", np.uint8)
    words = [b"ACGTAC", b"AAAA", b"AAAAAAAA", b"CGCGT"] + sorted({rng.choice(dna, 7).tobytes() for _ in range(20)})
    o = oracle.OracleAutomaton.from_words(words)
    a = am.build(am.make_patterns(words))
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.set_mode(am.MODE_EXACT)
    sparse = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, 1 << 20)]
    dense = sparse.copy()
    dense[200_000:600_000] = ord("A")
    for text in (sparse, dense, sparse, dense):
        s.run_host(text)
        ids, ends = s.records()
        oi, oe, _, cnt = o.scan(text, counts=True)
        assert recs(ids, ends) == recs(oi, oe)
        assert np.array_equal(s.pattern_counts(), cnt)


def test_concurrent_scans_share_one_automaton():
    """Any number of concurrent scans on one immutable automaton
    (aho_corasick.hpp:50-52; SPEC: scan is reentrant): 8 host threads, each
    with its own text, through the one-shot API (scanner pool per automaton)."""
    import threading
    w = synth.CONFIGS[0].scaled(1 << 20, 300)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    o = oracle.OracleAutomaton(concat, offs)
    texts = [synth.text(w.scaled((1 << 20) + 4096 * k)) for k in range(8)]
    results = [None] * len(texts)
    errors = []

    def work(k):
        try:
            for _ in range(3):
                results[k] = am.scan_arrays(a, texts[k], am.SCAN_LIST | am.SCAN_COUNTS)
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(len(texts))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k, text in enumerate(texts):
        oi, oe, _, cnt = o.scan(text, counts=True)
        assert recs(results[k].ids, results[k].ends) == recs(oi, oe)
        assert np.array_equal(results[k].counts, cnt)
