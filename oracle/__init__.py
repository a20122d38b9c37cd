"""ORACLE — test infrastructure, NOT the product.

Python handles on
  * liboracle.so      the plain-C restatement of the reference algorithm
                      (oracle/ac_oracle.c), and
  * _ref/libacref.so  the unmodified reference headers compiled by
                      oracle/Makefile (absent when neither /root/reference nor
                      a prebuilt _ref/ is available).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker or the timed CPU
baseline — never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBORACLE = os.path.join(HERE, "liboracle.so")
LIBREF = os.path.join(HERE, "_ref", "libacref.so")

vp = C.c_void_p
u64 = C.c_uint64
u32 = C.c_uint32

_ORACLE_SYMS = {
    "orc_build": (C.c_int, [vp, vp, u32, C.POINTER(vp)]),
    "orc_free": (None, [vp]),
    "orc_state_count": (u32, [vp]),
    "orc_max_len": (u32, [vp]),
    "orc_failure": (u32, [vp, u32]),
    "orc_depth": (u32, [vp, u32]),
    "orc_goto_transition": (C.c_int, [vp, u32, C.c_uint8, C.POINTER(u32)]),
    "orc_outputs": (u32, [vp, u32, C.POINTER(C.POINTER(u32))]),
    "orc_transitions": (u32, [vp, u32, C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(C.POINTER(u32))]),
    "orc_next_state": (u32, [vp, u32, C.c_uint8]),
    "orc_scan": (u64, [vp, vp, u64, C.POINTER(u64), vp, vp, u64]),
    "orc_scan_window": (u64, [vp, vp, u64, u64, u64, C.POINTER(u64), vp, vp, u64, vp]),
    "orc_naive_find_all": (u64, [vp, vp, u32, vp, u64, vp, vp, u64]),
    "orc_digest": (None, [vp, vp, u64, C.POINTER(u64), C.POINTER(u64)]),
    "orc_mt64_seed": (None, [vp, u64]),
    "orc_mt64_next": (u64, [vp]),
    "orc_mt64_size": (C.c_size_t, []),
    "orc_random_dictionary": (u32, [vp, u32, u32, u32, C.c_char_p, u32, vp, vp]),
    "orc_random_input": (u64, [vp, u64, C.c_char_p, u32, vp]),
}

_REF_SYMS = {
    "ref_build": (C.c_int, [vp, vp, u32, C.POINTER(vp)]),
    "ref_free": (None, [vp]),
    "ref_state_count": (u32, [vp]),
    "ref_failure": (u32, [vp, u32]),
    "ref_depth": (u32, [vp, u32]),
    "ref_next_state": (u32, [vp, u32, C.c_uint8]),
    "ref_goto": (C.c_int, [vp, u32, C.c_uint8, C.POINTER(u32)]),
    "ref_outputs": (u32, [vp, u32, vp, u32]),
    "ref_transitions": (u32, [vp, u32, vp, vp, u32]),
    "ref_scan": (u64, [vp, vp, u64, C.POINTER(u64), vp, vp, u64]),
    "ref_scan_window_stats": (C.c_int, [vp, vp, u64, u64, u64, vp, C.POINTER(u64), C.POINTER(u64),
                                        C.POINTER(u64), C.POINTER(u64)]),
    "ref_window_digest": (C.c_int, [vp, vp, u64, u64, u64, vp, C.POINTER(u64), C.POINTER(u64),
                                    C.POINTER(u64), C.POINTER(u64)]),
    "ref_run_partitioned": (C.c_int, [vp, vp, u32, vp, u64, u32, vp, vp, u64, C.POINTER(u64),
                                      C.POINTER(C.c_double), C.POINTER(u32)]),
    "ref_partitioned_prepare": (vp, [vp, vp, u32, u32]),
    "ref_partitioned_scan": (C.c_double, [vp, vp, u64, C.POINTER(u64)]),
    "ref_partitioned_workers": (u32, [vp]),
    "ref_partitioned_free": (None, [vp]),
    "ref_random_trial": (u32, [u64, u32, u32, u32, u64, vp, vp, vp, C.POINTER(u64)]),
    "ref_naive_find_all": (u64, [vp, vp, u32, vp, u64, vp, vp, u64]),
    "ref_hardware_concurrency": (C.c_uint, []),
    "ref_export": (None, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "ref_load_patterns": (C.c_int, [C.c_char_p, vp, vp, vp]),
    "ref_load_input": (C.c_int, [C.c_char_p, C.POINTER(u64), vp]),
    "ref_match_tsv": (u64, [vp, vp, u64, vp, u64]),
}

_libs: dict = {}


def _load(path: str, syms: dict) -> C.CDLL:
    if path not in _libs:
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        lib = C.CDLL(path)
        for name, (res, args) in syms.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _libs[path] = lib
    return _libs[path]


def lib() -> C.CDLL:
    return _load(LIBORACLE, _ORACLE_SYMS)


def ref_available() -> bool:
    return os.path.exists(LIBREF)


def ref() -> C.CDLL:
    return _load(LIBREF, _REF_SYMS)


def _u8(x) -> np.ndarray:
    if isinstance(x, str):
        x = x.encode("latin-1")
    if isinstance(x, (bytes, bytearray)):
        return np.frombuffer(bytes(x) or b"\0", dtype=np.uint8)[: len(x)] if len(x) else np.zeros(1, np.uint8)[:0]
    return np.ascontiguousarray(x, dtype=np.uint8)


def pack(words: list[bytes]) -> tuple[np.ndarray, np.ndarray]:
    offs = np.zeros(len(words) + 1, dtype=np.uint64)
    if words:
        offs[1:] = np.cumsum([len(w) for w in words], dtype=np.uint64)
    concat = np.frombuffer(b"".join(words) + b"\0", dtype=np.uint8).copy()
    return concat, offs


def _ptr(a: np.ndarray) -> vp:
    return a.ctypes.data_as(vp)


class OracleAutomaton:
    """The C restatement (oracle/ac_oracle.c)."""

    def __init__(self, concat: np.ndarray, offs: np.ndarray):
        self._concat, self._offs = np.ascontiguousarray(concat, np.uint8), np.ascontiguousarray(offs, np.uint64)
        h = vp()
        rc = lib().orc_build(_ptr(self._concat), _ptr(self._offs), len(offs) - 1, C.byref(h))
        if rc:
            raise ValueError({1: "empty dictionary", 2: "empty pattern"}.get(rc, f"build failed {rc}"))
        self._h = h

    @classmethod
    def from_words(cls, words: list[bytes]) -> "OracleAutomaton":
        return cls(*pack(words))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_free(self._h)

    def state_count(self) -> int:
        return lib().orc_state_count(self._h)

    def max_len(self) -> int:
        return lib().orc_max_len(self._h)

    def failure(self, s: int) -> int:
        return lib().orc_failure(self._h, s)

    def depth(self, s: int) -> int:
        return lib().orc_depth(self._h, s)

    def goto_transition(self, s: int, b: int) -> Optional[int]:
        t = u32()
        return t.value if lib().orc_goto_transition(self._h, s, b, C.byref(t)) else None

    def outputs(self, s: int) -> list[int]:
        p = C.POINTER(u32)()
        n = lib().orc_outputs(self._h, s, C.byref(p))
        return [p[i] for i in range(n)]

    def transitions(self, s: int) -> list[tuple[int, int]]:
        bp, tp = C.POINTER(C.c_uint8)(), C.POINTER(u32)()
        n = lib().orc_transitions(self._h, s, C.byref(bp), C.byref(tp))
        return [(bp[i], tp[i]) for i in range(n)]

    def next_state(self, s: int, b: int) -> int:
        return lib().orc_next_state(self._h, s, b)

    def scan(self, text, start: int = 0, emit_from: int = 0, with_records: bool = True,
             counts: bool = False) -> tuple[np.ndarray, np.ndarray, int, Optional[np.ndarray]]:
        """(ids, ends, failure_follows, per-pattern counts) of the windowed scan."""
        t = _u8(text)
        fol = u64()
        P = len(self._offs) - 1
        cnt = np.zeros(P, np.uint64) if counts else None
        m = lib().orc_scan_window(self._h, _ptr(t), t.size, start, emit_from, C.byref(fol), None, None, 0,
                                  _ptr(cnt) if counts else None)
        ids = np.empty(m, np.uint32)
        ends = np.empty(m, np.uint64)
        if with_records and m:
            lib().orc_scan_window(self._h, _ptr(t), t.size, start, emit_from, C.byref(fol), _ptr(ids), _ptr(ends), m,
                                  None)
        return ids, ends, fol.value, cnt


def naive_find_all(words: list[bytes], text) -> tuple[np.ndarray, np.ndarray]:
    concat, offs = pack(words)
    t = _u8(text)
    m = lib().orc_naive_find_all(_ptr(concat), _ptr(offs), len(words), _ptr(t), t.size, None, None, 0)
    ids, ends = np.empty(m, np.uint32), np.empty(m, np.uint64)
    lib().orc_naive_find_all(_ptr(concat), _ptr(offs), len(words), _ptr(t), t.size, _ptr(ids), _ptr(ends), m)
    return ids, ends


def digest(ids: np.ndarray, ends: np.ndarray) -> tuple[int, int]:
    ids = np.ascontiguousarray(ids, np.uint32)
    ends = np.ascontiguousarray(ends, np.uint64)
    s, x = u64(), u64()
    lib().orc_digest(_ptr(ids), _ptr(ends), ids.size, C.byref(s), C.byref(x))
    return s.value, x.value


class MT64:
    """std::mt19937_64 replay (published MT19937-64)."""

    def __init__(self, seed: int):
        self._buf = C.create_string_buffer(lib().orc_mt64_size())
        lib().orc_mt64_seed(self._buf, seed)

    def __call__(self) -> int:
        return lib().orc_mt64_next(self._buf)

    def random_dictionary(self, max_count: int, min_len: int, max_len: int, alphabet: bytes = b"ACGT") -> list[bytes]:
        concat = np.zeros(max_count * max_len + 1, np.uint8)
        offs = np.zeros(max_count + 1, np.uint64)
        n = lib().orc_random_dictionary(self._buf, max_count, min_len, max_len, alphabet, len(alphabet), _ptr(concat),
                                        _ptr(offs))
        b = concat.tobytes()
        return [b[int(offs[i]):int(offs[i + 1])] for i in range(n)]

    def random_input(self, max_len: int, alphabet: bytes = b"ACGT") -> bytes:
        out = np.zeros(max_len + 1, np.uint8)
        n = lib().orc_random_input(self._buf, max_len, alphabet, len(alphabet), _ptr(out))
        return out[:n].tobytes()


def oracle_trial(seed: int, max_count: int = 50, min_len: int = 1, max_len: int = 8,
                 max_input: int = 10000) -> tuple[list[bytes], bytes]:
    """tests/acceptance/acceptance_main.cpp:120-126 replayed in the oracle."""
    r = MT64(seed)
    words = r.random_dictionary(max_count, min_len, max_len)
    return words, r.random_input(max_input)


class RefAutomaton:
    """The reference itself (oracle/_ref/libacref.so)."""

    def __init__(self, concat: np.ndarray, offs: np.ndarray):
        self._concat, self._offs = np.ascontiguousarray(concat, np.uint8), np.ascontiguousarray(offs, np.uint64)
        h = vp()
        rc = ref().ref_build(_ptr(self._concat), _ptr(self._offs), len(offs) - 1, C.byref(h))
        if rc:
            raise ValueError(f"reference build failed ({rc})")
        self._h = h
        self.P = len(offs) - 1

    @classmethod
    def from_words(cls, words: list[bytes]) -> "RefAutomaton":
        return cls(*pack(words))

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                ref().ref_free(self._h)
        except TypeError:  # interpreter shutdown: module globals already torn down
            pass

    def state_count(self) -> int:
        return ref().ref_state_count(self._h)

    def failure(self, s: int) -> int:
        return ref().ref_failure(self._h, s)

    def depth(self, s: int) -> int:
        return ref().ref_depth(self._h, s)

    def next_state(self, s: int, b: int) -> int:
        return ref().ref_next_state(self._h, s, b)

    def goto_transition(self, s: int, b: int) -> Optional[int]:
        t = u32()
        return t.value if ref().ref_goto(self._h, s, b, C.byref(t)) else None

    def outputs(self, s: int) -> list[int]:
        buf = np.zeros(4096, np.uint32)
        n = ref().ref_outputs(self._h, s, _ptr(buf), 4096)
        return buf[:n].tolist()

    def transitions(self, s: int) -> list[tuple[int, int]]:
        bb, tt = np.zeros(256, np.uint8), np.zeros(256, np.uint32)
        n = ref().ref_transitions(self._h, s, _ptr(bb), _ptr(tt), 256)
        return list(zip(bb[:n].tolist(), tt[:n].tolist()))

    def match_tsv(self, text) -> bytes:
        """The reference scan printed as `acmatch match` TSV (cli.hpp:71-74)."""
        t = _u8(text)
        n = ref().ref_match_tsv(self._h, _ptr(t), t.size, None, 0)
        out = np.zeros(max(n, 1), np.uint8)
        ref().ref_match_tsv(self._h, _ptr(t), t.size, _ptr(out), out.size)
        return out[:n].tobytes()

    def export(self) -> dict:
        """The whole machine through the reference's public accessors, as CSR arrays."""
        sizes = np.zeros(3, np.uint64)
        lib = ref()
        lib.ref_export(self._h, _ptr(sizes), *([None] * 7))
        S, E, O = (int(x) for x in sizes)
        out = {"fail": np.zeros(S, np.uint32), "depth": np.zeros(S, np.uint32),
               "edge_off": np.zeros(S + 1, np.uint32), "edge_byte": np.zeros(E, np.uint8),
               "edge_to": np.zeros(E, np.uint32), "out_off": np.zeros(S + 1, np.uint32),
               "out_ids": np.zeros(O, np.uint32)}
        lib.ref_export(self._h, _ptr(sizes), *[_ptr(out[k]) for k in ("fail", "depth", "edge_off", "edge_byte",
                                                                      "edge_to", "out_off", "out_ids")])
        return out

    def scan(self, text) -> tuple[np.ndarray, np.ndarray, int]:
        t = _u8(text)
        fol = u64()
        m = ref().ref_scan(self._h, _ptr(t), t.size, C.byref(fol), None, None, 0)
        ids, ends = np.empty(m, np.uint32), np.empty(m, np.uint64)
        ref().ref_scan(self._h, _ptr(t), t.size, C.byref(fol), _ptr(ids), _ptr(ends), m)
        return ids, ends, fol.value

    def window_stats(self, text, start: int, emit_from: int, counts: np.ndarray, acc: dict) -> int:
        t = _u8(text)
        m, s, x, f = u64(acc["m"]), u64(acc["dsum"]), u64(acc["dxor"]), u64(acc["follows"])
        rc = ref().ref_scan_window_stats(self._h, _ptr(t), t.size, start, emit_from, _ptr(counts), C.byref(m),
                                         C.byref(s), C.byref(x), C.byref(f))
        acc.update(m=m.value, dsum=s.value, dxor=x.value, follows=f.value)
        return rc

    def window_digest(self, window, emit_from: int, abs_base: int, counts: np.ndarray, acc: dict) -> int:
        """Reference scan of `window` (from the root) keeping ends >= emit_from;
        digest keys use absolute ends abs_base + end."""
        t = _u8(window)
        m, s, x, f = u64(acc["m"]), u64(acc["dsum"]), u64(acc["dxor"]), u64(acc["follows"])
        rc = ref().ref_window_digest(self._h, _ptr(t), t.size, emit_from, abs_base, _ptr(counts), C.byref(m),
                                     C.byref(s), C.byref(x), C.byref(f))
        acc.update(m=m.value, dsum=s.value, dxor=x.value, follows=f.value)
        return rc


def ref_random_trial(seed: int, max_count: int = 50, min_len: int = 1, max_len: int = 8,
                     max_input: int = 10000) -> tuple[list[bytes], bytes]:
    concat = np.zeros(max_count * max_len + 1, np.uint8)
    offs = np.zeros(max_count + 1, np.uint64)
    text = np.zeros(max_input + 1, np.uint8)
    tl = u64()
    n = ref().ref_random_trial(seed, max_count, min_len, max_len, max_input, _ptr(concat), _ptr(offs), _ptr(text),
                               C.byref(tl))
    b = concat.tobytes()
    return [b[int(offs[i]):int(offs[i + 1])] for i in range(n)], text[: tl.value].tobytes()


def ref_load_patterns(path: str):
    """The reference's acmatch::load_patterns: (rc, words, duplicates, skipped_empty)."""
    sizes = np.zeros(4, np.uint64)
    rc = ref().ref_load_patterns(os.fsencode(path), _ptr(sizes), None, None)
    if rc:
        return rc, None, 0, 0
    concat = np.zeros(max(int(sizes[1]), 1), np.uint8)
    offs = np.zeros(int(sizes[0]) + 1, np.uint64)
    ref().ref_load_patterns(os.fsencode(path), _ptr(sizes), _ptr(concat), _ptr(offs))
    b = concat.tobytes()
    return 0, [b[int(offs[i]):int(offs[i + 1])] for i in range(int(sizes[0]))], int(sizes[2]), int(sizes[3])


def ref_load_input(path: str):
    """The reference's acmatch::load_input: (rc, bytes)."""
    n = u64()
    rc = ref().ref_load_input(os.fsencode(path), C.byref(n), None)
    if rc:
        return rc, None
    out = np.zeros(max(n.value, 1), np.uint8)
    ref().ref_load_input(os.fsencode(path), C.byref(n), _ptr(out))
    return 0, out[:n.value].tobytes()


def json_escape(b: bytes) -> bytes:
    """Restatement of nlohmann::json's string dump with error_handler replace and
    ensure_ascii false (the reference's cmd_match JSON, cli.hpp:63-69): JSON
    escapes for '"', backslash, \\b \\f \\n \\r \\t, \\u00xx for other bytes < 0x20,
    valid UTF-8 as is, each invalid sequence -> U+FFFD. Parity of the invalid-UTF-8
    rule is UNPINNED (nlohmann/json is not in this image); valid text is pinned
    by Python's json module in the tests."""
    out = bytearray()
    i, n = 0, len(b)
    esc = {0x22: b'\\"', 0x5C: b"\\\\", 0x08: b"\\b", 0x0C: b"\\f", 0x0A: b"\\n", 0x0D: b"\\r", 0x09: b"\\t"}
    while i < n:
        c = b[i]
        if c < 0x80:
            out += esc.get(c, b"\\u%04x" % c if c < 0x20 else bytes([c]))
            i += 1
            continue
        need, lo, hi = 0, 0x80, 0xBF
        if 0xC2 <= c <= 0xDF: need = 1
        elif c == 0xE0: need, lo = 2, 0xA0
        elif 0xE1 <= c <= 0xEC or c in (0xEE, 0xEF): need = 2
        elif c == 0xED: need, hi = 2, 0x9F
        elif c == 0xF0: need, lo = 3, 0x90
        elif 0xF1 <= c <= 0xF3: need = 3
        elif c == 0xF4: need, hi = 3, 0x8F
        if need == 0:
            out += b"\xef\xbf\xbd"
            i += 1
            continue
        k = 1
        while k <= need and i + k < n:
            d = b[i + k]
            if not ((lo <= d <= hi) if k == 1 else (0x80 <= d <= 0xBF)):
                break
            k += 1
        if k == need + 1:
            out += b[i:i + need + 1]
            i += need + 1
        else:
            out += b"\xef\xbf\xbd"
            i += k
    return bytes(out)
