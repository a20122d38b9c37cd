"""TEST INFRASTRUCTURE: writes the golden fixtures under tests/golden/ from the
REFERENCE ITSELF — oracle/_ref/libacref.so, the unmodified reference headers
compiled where they lie under /root/reference (oracle/Makefile) — so the
fixtures pin both the C restatement (oracle/ac_oracle.c) and the GPU path.
Run in the build container (needs oracle/_ref):  python -m oracle.make_goldens

  known_answers.json   small dictionaries/texts with their full reference
                       match lists and failure-follow counts: the reference's
                       worked example (HIS/SHE/HERS), self-overlap, full byte
                       alphabet, escapes, and the reference's own randomized
                       trials (tests/support/oracle.hpp:46-67 draws, replayed
                       through std::mt19937_64 inside the reference build).
  configs_small.json   every BASELINE config scaled to 2 MiB of text (its own
                       dictionary regenerated at that size): record count,
                       order-independent digest, failure follows and
                       per-pattern counts.
  configs_full.json    the same statistics at every config's FULL size
                       (16 MiB .. 8 GiB), computed by the reference scanning
                       overlapping windows in parallel (halo = longest
                       pattern, so window states equal whole-text states).

Digest: key = end * 2^20 + pattern_id, mixed by splitmix64's finalizer;
dsum = sum of mixed keys mod 2^64, dxor = their xor (order independent).
counts_sha256 = sha256 of the per-pattern counts as little-endian uint64.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1403_7294_b200 import synth  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
MIB = 1 << 20


def _records(ra: "oracle.RefAutomaton", text: bytes) -> tuple[list[list[int]], int]:
    ids, ends, fol = ra.scan(text)
    return [[int(i), int(e)] for i, e in zip(ids, ends)], int(fol)


def known_answers() -> list[dict]:
    cases: list[tuple[str, list[bytes], bytes]] = [
        ("classic-ushers", [b"HIS", b"SHE", b"HERS"], b"USHERS"),
        ("classic-long", [b"HIS", b"SHE", b"HERS"], b"AHISHERSHESHISHERSXHERSHIS"),
        ("classic-empty-text", [b"HIS", b"SHE", b"HERS"], b""),
        ("self-overlap", [b"AA", b"A", b"AAA"], b"AAAAAAA"),
        ("nested-suffixes", [b"ACGTACGT", b"GTACGT", b"ACGT", b"CGT", b"T"], b"ACGTACGTACGTTTACGTACG"),
        ("single-byte-dictionary", [b"G"], b"GATTACAGG"),
        ("dna-with-escapes", [b"ACGT", b"GTAC", b"TTT"], b"ACGTNNACGTACxTTTTacgtTTT\x00ACGT"),
        ("full-byte-alphabet", [bytes([0, 255]), bytes([255]), bytes(range(250, 256)), b"\n\r", b"\x80\x81\x82"],
         bytes(range(256)) * 3 + b"\x00\xff\x00\xff\xff\n\r\x80\x81\x82"),
        ("pattern-longer-than-text", [b"ACGTACGTACGT", b"CG"], b"ACGTACG"),
    ]
    out = []
    for name, words, text in cases:
        ra = oracle.RefAutomaton.from_words(words)
        recs, fol = _records(ra, text)
        out.append(dict(name=name, patterns=[w.hex() for w in words], text=text.hex(), records=recs, follows=fol,
                        states=ra.state_count()))
    # the reference's randomized trials (acceptance_main.cpp:129-169 shape)
    for seed in range(12):
        for (mc, lo, hi, alpha) in ((50, 1, 8, b"ACGT"), (20, 2, 6, b"AB")):
            rng = oracle.MT64(1000 + seed)
            words = rng.random_dictionary(mc, lo, hi, alpha)
            text = rng.random_input(1500, alpha)
            ra = oracle.RefAutomaton.from_words(words)
            recs, fol = _records(ra, text)
            out.append(dict(name=f"mt64-{1000 + seed}-{alpha.decode()}", patterns=[w.hex() for w in words],
                            text=text.hex(), records=recs, follows=fol, states=ra.state_count()))
    return out


def config_stats(w: synth.Workload, threads: int, window: int = 32 * MIB) -> dict:
    t0 = time.time()
    concat, offs = synth.patterns(w)
    ra = oracle.RefAutomaton(concat, offs)
    P = len(offs) - 1
    maxlen = int(np.max(np.diff(offs.astype(np.int64))))
    spans = [(lo, min(lo + window, w.n)) for lo in range(0, w.n, window)]

    def job(span):
        lo, hi = span
        start = max(0, lo - maxlen)
        t = synth.text(w, start, hi, threads=1)
        counts = np.zeros(P, np.uint64)
        acc = dict(m=0, dsum=0, dxor=0, follows=0)
        rc = ra.window_digest(t, lo - start, start, counts, acc)
        if rc:
            raise RuntimeError(f"reference output out of order in window {span}")
        return counts, acc

    counts = np.zeros(P, np.uint64)
    m = dsum = dxor = follows = 0
    with ThreadPoolExecutor(threads) as ex:
        for c, acc in ex.map(job, spans):
            counts += c
            m += acc["m"]
            dsum = (dsum + acc["dsum"]) & 0xFFFFFFFFFFFFFFFF
            dxor ^= acc["dxor"]
            follows += acc["follows"]
    rec = dict(name=w.name, kind=w.kind, n=w.n, patterns=w.patterns, len_lo=w.len_lo, len_hi=w.len_hi, seed=w.seed,
               states=ra.state_count(), max_len=maxlen, m=m, dsum=dsum, dxor=dxor, follows=follows,
               counts_sha256=hashlib.sha256(counts.astype("<u8").tobytes()).hexdigest(),
               counts_nonzero=int(np.count_nonzero(counts)), counts_max=int(counts.max()),
               seconds=round(time.time() - t0, 1))
    if P <= 2000:
        rec["counts"] = [int(x) for x in counts]
    print(f"  {w.name}: n={w.n} m={m} follows={follows} ({rec['seconds']} s)", flush=True)
    return rec


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--skip-full", action="store_true")
    ap.add_argument("--only", default="", help="comma-separated fixture names (known,small,full)")
    args = ap.parse_args()
    if not oracle.ref_available():
        sys.exit("oracle/_ref/libacref.so missing: run `make -C oracle` with /root/reference present")
    os.makedirs(GOLDEN, exist_ok=True)
    only = set(filter(None, args.only.split(","))) or {"known", "small", "full"}
    meta = dict(generator="oracle/make_goldens.py", source="reference (oracle/_ref/libacref.so)",
                digest="key=end*2^20+id; mix=splitmix64 finalizer; dsum=sum mod 2^64; dxor=xor")

    def dump(name, payload):
        with open(os.path.join(GOLDEN, name), "w") as f:
            json.dump(dict(meta, cases=payload), f, indent=None if name == "known_answers.json" else 1,
                      separators=(",", ":") if name == "known_answers.json" else None)
            f.write("\n")

    if "known" in only:
        dump("known_answers.json", known_answers())
    if "small" in only:
        print("configs scaled to 2 MiB:")
        dump("configs_small.json", [config_stats(w.scaled(2 * MIB), args.threads) for w in synth.CONFIGS])
    if "full" in only and not args.skip_full:
        print("configs at full size:")
        dump("configs_full.json", [config_stats(w, args.threads) for w in synth.CONFIGS])


if __name__ == "__main__":
    main()
