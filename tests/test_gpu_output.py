"""GPU parity of the output step (acg_scanner_format / acg_scanner_write_matches:
the match list formatted on the GPU as the reference's `acmatch match` output,
proj/include/acmatch/cli.hpp:58-76). TSV is compared byte for byte with the
REFERENCE's scan printed by cmd_match's loop (oracle/_ref); JSON with Python's
json module (nlohmann dump(-1) of the same records: compact, keys sorted,
ensure_ascii off) for valid UTF-8 patterns, and with oracle.json_escape's
restatement of nlohmann's error_handler::replace for invalid UTF-8 (unpinned:
nlohmann/json is not in this image). Windows of the list, the empty list and
tiles whose text exceeds the shared-memory staging (long patterns) included."""
from __future__ import annotations

import json

import numpy as np
import pytest

import oracle
from paper_1403_7294_b200 import acmatch as am
from paper_1403_7294_b200 import synth

pytestmark = pytest.mark.gpu


def scan(words, text):
    concat, offs = synth.pack_patterns(words)
    a = am.Automaton.from_arrays(concat, offs)
    s = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
    s.run_host(text)
    s.sync()
    return a, s, concat, offs


def expect_json(words, ids, ends) -> bytes:
    recs = [{"end": int(e), "pattern": words[int(i)].decode("utf-8"), "pattern_id": int(i)} for i, e in zip(ids, ends)]
    return json.dumps(recs, ensure_ascii=False, separators=(",", ":"), sort_keys=True).encode() + b"\n"


@pytest.mark.parametrize("cfg,mib", [(0, 2), (3, 2), (4, 1)])
def test_tsv_matches_reference_and_json_matches_json_module(cfg, mib):
    w = synth.CONFIGS[cfg].scaled(mib << 20, min(synth.CONFIGS[cfg].patterns, 1000))
    text = synth.text(w)
    a, s, concat, offs = scan(synth.pattern_list(*synth.patterns(w)), text)
    tsv = s.format("tsv")
    if oracle.ref_available():
        assert tsv == oracle.RefAutomaton(concat, offs).match_tsv(text)
    ids, ends = s.records()
    words = synth.pattern_list(concat, offs)
    lines = b"".join(b"%d\t%d\t" % (e, i) + words[i] + b"\n" for i, e in zip(ids.tolist(), ends.tolist()))
    assert tsv == lines
    assert s.format("json") == expect_json(words, ids, ends)


def test_windows_concatenate_to_the_whole_output():
    w = synth.CONFIGS[3].scaled(1 << 20, 500)
    text = synth.text(w)
    a, s, concat, offs = scan(synth.pattern_list(*synth.patterns(w)), text)
    m = s.match_count()
    for fmt in ("tsv", "json"):
        whole = s.format(fmt)
        cuts = [0, 1, 255, 256, 257, m // 3, m - 1, m]
        parts = b"".join(s.format(fmt, lo, hi - lo) for lo, hi in zip(cuts, cuts[1:]))
        assert parts == whole


def test_escaping_and_invalid_utf8_and_long_patterns(tmp_path):
    words = [b'a"b', b"c\\d", b"e\tf", b"\x01\x1fX", b"h\xc3\xa9!", b"\xff\xfe", b"\xe2\x82z", b"Q" * 3000]
    text = np.frombuffer(b"".join(w + b"  " for w in words) * 40, np.uint8).copy()
    a, s, concat, offs = scan(words, text)
    ids, ends = s.records()
    assert len(ids) >= 40 * len(words)
    body = b",".join(b'{"end":%d,"pattern":"' % e + oracle.json_escape(words[i]) + b'","pattern_id":%d}' % i
                     for i, e in zip(ids.tolist(), ends.tolist()))
    assert s.format("json") == b"[" + body + b"]\n"
    tsv = b"".join(b"%d\t%d\t" % (e, i) + words[i] + b"\n" for i, e in zip(ids.tolist(), ends.tolist()))
    assert s.format("tsv") == tsv
    if oracle.ref_available():
        assert tsv == oracle.RefAutomaton(concat, offs).match_tsv(text)
    p = tmp_path / "out.tsv"
    assert s.write_matches(str(p), "tsv") == len(tsv) and p.read_bytes() == tsv


def test_empty_list():
    a, s, _, _ = scan([b"ZZZ"], np.frombuffer(b"ACGT" * 100, np.uint8).copy())
    assert s.match_count() == 0
    assert s.format("tsv") == b"" and s.format("json") == b"[]\n"
