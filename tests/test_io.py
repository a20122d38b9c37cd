"""Input path: acg_load_input / acg_load_patterns against
the REFERENCE's own loaders (oracle/_ref: acmatch::load_input / load_patterns,
proj/include/acmatch/io.hpp:25-65) on the cases its unit tests pin (CRLF, empty
lines, duplicates, missing final newline, NUL bytes, empty and missing files)
plus random byte files. Host-only: these run without a GPU."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from paper_1403_7294_b200 import acmatch as am

CASES = {
    "plain": b"HIS\nSHE\nHERS\n",
    "crlf": b"HIS\r\nSHE\r\nHERS\r\n",
    "no_final_newline": b"HIS\nSHE\nHERS",
    "empties_and_dups": b"\n\nA\nB\n\nA\r\nB\nC\n\n",
    "cr_only_inside": b"A\rB\nC\r\r\n\r\n",
    "nul_bytes": b"\x00A\x00\nB\x00\n\x00\n",
    "high_bytes": bytes(range(1, 10)) + b"\n" + bytes(range(200, 256)) + b"\n",
    "blank": b"\n\r\n\n",
    "zero": b"",
}


def write(tmp_path, name, data):
    p = tmp_path / name
    p.write_bytes(data)
    return str(p)


@pytest.mark.parametrize("name", sorted(CASES))
def test_load_patterns_matches_reference(tmp_path, name):
    path = write(tmp_path, name, CASES[name])
    if not oracle.ref_available():
        pytest.skip("oracle/_ref is not built")
    rc, words, dups, empty = oracle.ref_load_patterns(path)
    if rc:
        with pytest.raises(am.EmptyDictionaryError if rc == 1 else am.Error):
            am.load_patterns(path)
        return
    f = am.load_patterns(path)
    assert [p.bytes for p in f.patterns] == words
    assert [p.id for p in f.patterns] == list(range(len(words)))
    assert (f.duplicates, f.skipped_empty) == (dups, empty)


@pytest.mark.parametrize("seed", range(6))
def test_load_patterns_random_files(tmp_path, seed):
    rng = np.random.default_rng(seed)
    alpha = np.frombuffer(b"AB\r\n\x00C", np.uint8)
    data = alpha[rng.integers(0, alpha.size, int(rng.integers(1, 4000)))].tobytes()
    path = write(tmp_path, "r.txt", data)
    rc, words, dups, empty = oracle.ref_load_patterns(path)
    if rc:
        with pytest.raises(am.Error):
            am.load_patterns(path)
        return
    f = am.load_patterns(path)
    assert ([p.bytes for p in f.patterns], f.duplicates, f.skipped_empty) == (words, dups, empty)


@pytest.mark.parametrize("size", [0, 1, 5, 4096, (64 << 20) + 12345])
def test_load_input_matches_reference(tmp_path, size):
    data = np.random.default_rng(size).integers(0, 256, size, dtype=np.uint8).tobytes()
    path = write(tmp_path, "in.bin", data)
    got = am.load_input(path)
    assert got.n == size and got.array.tobytes() == data
    rc, ref = oracle.ref_load_input(path)
    assert rc == 0 and ref == data


def test_missing_files_are_io_errors(tmp_path):
    missing = str(tmp_path / "nope")
    with pytest.raises(am.IoError):
        am.load_input(missing)
    with pytest.raises(am.IoError):
        am.load_patterns(missing)
    assert oracle.ref_load_input(missing)[0] == 9 and oracle.ref_load_patterns(missing)[0] == 9


def test_loaded_dictionary_builds_the_same_machine(tmp_path):
    words = [b"HIS", b"SHE", b"HERS", b"SHE", b"", b"HE"]
    path = write(tmp_path, "p.txt", b"\n".join(words) + b"\n")
    f = am.load_patterns(path)
    a = am.build(f.patterns)
    r = oracle.RefAutomaton.from_words([p.bytes for p in f.patterns])
    assert a.nfa_arrays()["fail"].tolist() == r.export()["fail"].tolist()
