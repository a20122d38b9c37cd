"""CPU: the C-ABI library and its host side, without a GPU.

  * lib/libacg.so loads and exports every function include/acg.h declares
    (and the ctypes table binds exactly those);
  * the host automaton build behind acg_build reproduces the reference's
    machine state by state (numbering, goto edges, failure links, depth,
    outputs, next_state) — checked against oracle/_ref (the reference
    compiled from /root/reference) and the oracle restatement;
  * error statuses map to the reference's exception types;
  * the product path has no CPU fallback: without the library it fails.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_1403_7294_b200 import _lib, acmatch as am, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared() -> set[str]:
    src = open(os.path.join(ROOT, "include", "acg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(acg_[a-z0-9_]+)\s*\(", src))


def test_header_declares_the_bound_symbols():
    assert _declared() == set(_lib.ACG_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(os.path.join(ROOT, "paper_1403_7294_b200", "lib", "libacg.so"))
    missing = [s for s in sorted(_declared()) if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_1403_7294_b200", "lib", "libacg.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert _declared() <= exported


def test_library_is_sm100a():
    """The CUDA kernels in libacg.so are sm_100a SASS (no PTX JIT, no other arch)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_1403_7294_b200", "lib", "libacg.so")],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, out


def test_version_and_last_error():
    assert am.version().startswith("acg ")
    h = C.c_void_p()
    offs = np.zeros(1, np.uint64)
    rc = _lib.acg().acg_build(None, offs.ctypes.data_as(C.c_void_p), 0, C.byref(h))
    assert rc == 1 and not h.value  # ACG_ERR_EMPTY_DICTIONARY
    assert "empty" in _lib.acg().acg_last_error().decode().lower()


def test_build_errors_map_to_reference_exceptions():
    with pytest.raises(am.EmptyDictionaryError):
        am.build([])
    with pytest.raises(am.EmptyPatternError):
        am.build(am.make_patterns([b"AC", b""]))
    with pytest.raises(am.Error):
        am.build([am.Pattern(1, b"AC")])  # ids must be dense, in load order
    assert issubclass(am.EmptyPatternError, am.Error) and issubclass(am.DeviceError, am.Error)


def _same_machine(a: am.Automaton, r) -> None:
    S = r.state_count()
    assert a.state_count() == S
    for s in range(S):
        assert a.failure(s) == r.failure(s), s
        assert a.depth(s) == r.depth(s), s
        assert a.outputs(s) == r.outputs(s), s
        assert a.transitions(s) == r.transitions(s), s
        for b in (0, 65, 67, 71, 84, 255):
            assert am.next_state(a, s, b) == r.next_state(s, b)
            assert a.goto_transition(s, b) == r.goto_transition(s, b)


def test_classic_machine():
    a = am.build(am.make_patterns([b"HIS", b"SHE", b"HERS"]))
    _same_machine(a, oracle.OracleAutomaton.from_words([b"HIS", b"SHE", b"HERS"]))
    assert a.state_count() == 10
    assert a.outputs(9) == [1]  # SHE
    assert a.max_pattern_length() == 4 and a.pattern_count() == 3


@pytest.mark.parametrize("seed", range(0, 300, 11))
def test_host_build_matches_reference_on_trials(seed):
    words, _ = oracle.oracle_trial(seed)
    a = am.build(am.make_patterns(words))
    _same_machine(a, oracle.RefAutomaton.from_words(words) if oracle.ref_available()
                  else oracle.OracleAutomaton.from_words(words))


@pytest.mark.parametrize("cfg", range(5))
def test_host_build_matches_oracle_on_config_dictionaries(cfg):
    w = synth.CONFIGS[cfg].scaled(1 << 20, patterns=min(synth.CONFIGS[cfg].patterns, 800))
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    o = oracle.OracleAutomaton(concat, offs)
    assert a.state_count() == o.state_count()
    rng = np.random.default_rng(cfg)
    for s in rng.integers(0, o.state_count(), 400):
        s = int(s)
        assert (a.failure(s), a.depth(s), a.outputs(s), a.transitions(s)) == \
            (o.failure(s), o.depth(s), o.outputs(s), o.transitions(s))


def test_layout_reports_dfa_geometry():
    w = synth.CONFIGS[1].scaled(1 << 20, patterns=2000)
    concat, offs = synth.patterns(w)
    a = am.Automaton.from_arrays(concat, offs)
    lay = a.layout()
    assert lay["halo"] % 16 == 0 and lay["halo"] >= a.max_pattern_length()
    assert 0 < lay["hot_rows"] <= a.state_count() and lay["alphabet"] == "dna4"


def test_synth_windows_are_consistent():
    """Counter-based generator: any window equals the slice of the whole text
    (what lets ranks and the golden generator produce only their windows)."""
    for w in synth.CONFIGS:
        ws = w.scaled(1 << 20)
        full = synth.text(ws)
        for lo, hi in ((0, 1), (12345, 67890), ((1 << 20) - 100, 1 << 20)):
            assert np.array_equal(synth.text(ws, lo, hi), full[lo:hi])
    dna = synth.text(synth.CONFIGS[1].scaled(1 << 16))
    assert set(np.unique(dna).tobytes()) == set(b"ACGT")


def test_no_cpu_fallback_without_library():
    """With the library missing, the product import fails loudly."""
    code = ("import os; os.environ['ACG_LIBRARY_OVERRIDE']='/nonexistent/libacg.so'\n"
            "from paper_1403_7294_b200 import acmatch as am\n"
            "try:\n    am.build(am.make_patterns([b'A']))\nexcept ImportError as e:\n    print('IMPORT-ERROR', e)\n")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert "IMPORT-ERROR" in p.stdout or "ImportError" in p.stderr, p.stdout + p.stderr


def test_scan_without_device_raises_device_error():
    """No GPU here: scanning reports DeviceError instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    a = am.build(am.make_patterns([b"HIS", b"SHE", b"HERS"]))
    with pytest.raises(am.DeviceError):
        am.scan(a, b"USHERS")


@pytest.mark.parametrize("cfg", range(5))
def test_full_machine_equals_reference_on_config_dictionaries(cfg):
    """The bulk (sort-based, level-parallel) build against the REFERENCE's own
    build (oracle/_ref), state by state over the whole machine — failure links,
    depths, sorted edges, suffix-closed output sets — on every BASELINE
    config's full dictionary (up to cfg2's 100,000 patterns, 1.85M states)."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref (the reference compiled here) is not built")
    concat, offs = synth.patterns(synth.CONFIGS[cfg])
    mine = am.Automaton.from_arrays(concat, offs).nfa_arrays()
    theirs = oracle.RefAutomaton(concat, offs).export()
    for k in ("fail", "depth", "edge_off", "edge_byte", "edge_to", "out_off", "out_ids"):
        assert np.array_equal(mine[k], theirs[k]), k


@pytest.mark.parametrize("seed", range(8))
def test_bulk_build_duplicates_prefixes_and_bytes(seed):
    """Duplicate patterns, patterns that are prefixes of others, ids whose
    insertion order disagrees with lexicographic order, the full byte range."""
    rng = np.random.default_rng(1000 + seed)
    alpha = [b"AB", b"ACGT", bytes(range(256))][seed % 3]
    words = []
    for _ in range(int(rng.integers(1, 400))):
        n = int(rng.integers(1, 9))
        words.append(bytes(alpha[int(i)] for i in rng.integers(0, len(alpha), n)))
    words += [w[: max(1, len(w) // 2)] for w in words[:50]] + words[:30]  # prefixes and duplicates
    rng.shuffle(words)
    concat, offs = oracle.pack(words)
    mine = am.Automaton.from_arrays(concat, offs).nfa_arrays()
    ref = (oracle.RefAutomaton(concat, offs).export() if oracle.ref_available() else None)
    if ref is None:
        pytest.skip("oracle/_ref is not built")
    for k in mine:
        assert np.array_equal(mine[k], ref[k]), k
