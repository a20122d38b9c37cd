"""Host logic of the compressed hot automaton (csrc/ctab.hpp, built by
compile_dfa): the device walk's per-step rule — one row-displaced exception
lookup, else the text-only default T_D — replayed on the host against the
dense transition table (reference semantics: next_state,
proj/include/acmatch/aho_corasick.hpp:238-245), state for state.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_1403_7294_b200 import acmatch as am
from paper_1403_7294_b200 import synth


def protein(n=1 << 20, patterns=5000):
    w = synth.CONFIGS[3].scaled(n, patterns)
    return synth.text(w), synth.patterns(w)


def test_cfg3_dictionary_walks_exactly():
    text, (concat, offs) = protein()
    a = am.Automaton.from_arrays(concat, offs)
    r = a.ctab_check(text)
    assert r["available"] and r["default_depth"] == 3
    assert r["mismatches"] == 0
    # the deep default makes the whole automaton hot (the dense rows hold a fifth of it)
    assert r["deep"] and r["hot_states"] == a.layout()["states"] and r["cold_steps"] == 0
    assert r["entries"] <= r["slots"]


def test_profile_order_and_hot_limits_walk_exactly():
    text, (concat, offs) = protein(1 << 19)
    for limit in (0, 1, 7, 300, 4000):
        a = am.Automaton.from_arrays(concat, offs)
        a.optimize_layout(text[: 1 << 16])
        if limit:
            a.set_hot_limit(limit)
        r = a.ctab_check(text)
        assert r["available"] and r["mismatches"] == 0
        if limit in (1, 7, 300):
            assert not r["deep"]  # every state of depth <= 3 must be hot for the deep default
        if limit:
            assert r["hot_states"] <= limit and r["cold_steps"] > 0


def test_bytes_outside_the_alphabet_reset_to_the_root():
    text, (concat, offs) = protein(1 << 18, 2000)
    text = text.copy()
    rng = np.random.default_rng(7)
    text[rng.integers(0, text.size, 4000)] = rng.integers(0, 256, 4000).astype(np.uint8)
    a = am.Automaton.from_arrays(concat, offs)
    a.set_hot_limit(500)
    assert a.ctab_check(text)["mismatches"] == 0


def test_not_built_when_it_does_not_apply():
    # DNA dictionaries use the 2-bit walk; small automata fit the dense hot rows
    w = synth.CONFIGS[0].scaled(1 << 16, 100)
    a = am.Automaton.from_arrays(*synth.patterns(w))
    assert not a.ctab_check()["available"]
    a = am.build(am.make_patterns(["HIS", "SHE", "HERS"]))
    assert not a.ctab_check()["available"]
    # 40 distinct symbols: more columns than the 5-bit column field holds
    words = [bytes([65 + (i * 7 + j) % 40 for j in range(6)]) for i in range(3000)]
    a = am.build(am.make_patterns(words))
    a.set_hot_limit(8)
    assert not a.ctab_check()["available"]


@pytest.mark.parametrize("nsym", [2, 5, 22, 30])
def test_alphabet_sizes(nsym):
    rng = np.random.default_rng(nsym)
    alpha = np.arange(97, 97 + nsym, dtype=np.uint8)
    words = [alpha[rng.integers(0, nsym, rng.integers(2, 10))].tobytes() + b"" for _ in range(3000)]
    words = list(dict.fromkeys(words))
    if nsym == 2:
        words.append(b"z")  # not a DNA alphabet anyway; keeps the generic mode explicit
    a = am.build(am.make_patterns(words))
    a.set_hot_limit(50)
    text = alpha[rng.integers(0, nsym, 1 << 17)]
    r = a.ctab_check(text)
    assert r["available"], r
    assert r["default_depth"] == (3 if (nsym + 1 + (nsym == 2)) ** 3 * 4 <= 40 * 1024 else 2)
    assert r["mismatches"] == 0
