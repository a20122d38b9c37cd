"""Python binding of the `acmatch` API over the C ABI (include/acg.h).

Mirrors the reference's names and semantics (reference paths relative to
/root/reference/proj): `build` (include/acmatch/aho_corasick.hpp:130),
`next_state` (:238), `scan` (:250/:274), `match_count` (:280),
`match_before` (:38), the `Automaton` accessors (:58-101) and the error
hierarchy (include/acmatch/errors.hpp). The scan runs on the GPU through
lib/libacg.so; there is no CPU path. `Scanner` is the device-resident entry
used by the benchmark and the shard runner.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import NamedTuple, Optional, Sequence

import numpy as np

from . import _lib

SCAN_LIST, SCAN_COUNTS, SCAN_STATS, SCAN_PROFILE = 1, 2, 4, 8
MODE_AUTO, MODE_SPARSE, MODE_EXACT, MODE_FILTER = 0, 1, 2, 3


# ---- errors (include/acmatch/errors.hpp:9-48) ------------------------------
class Error(RuntimeError):
    pass


class EmptyPatternError(Error):
    pass


class EmptyDictionaryError(Error):
    pass


class InvalidWorkerCountError(Error):
    pass


class DeviceError(Error):
    """New in this build: CUDA failure or no usable device."""


class IoError(Error):
    """acmatch::IoError (reference errors.hpp; raised by the io.hpp loaders)."""


_ERRORS = {1: EmptyDictionaryError, 2: EmptyPatternError, 3: Error, 4: InvalidWorkerCountError,
           5: DeviceError, 6: DeviceError, 7: DeviceError, 9: IoError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.acg().acg_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, Error)(msg)


# ---- value types (aho_corasick.hpp:23-48) ----------------------------------
class Pattern(NamedTuple):
    id: int
    bytes: bytes


class MatchRecord(NamedTuple):
    pattern_id: int
    end: int


@dataclass
class ScanStats:
    failure_follows: int = 0


kRoot = 0


def match_before(a: MatchRecord, b: MatchRecord) -> bool:
    """aho_corasick.hpp:38-41: (end, pattern_id) ascending."""
    return (a.end, a.pattern_id) < (b.end, b.pattern_id)


def make_patterns(words: Sequence[bytes | str]) -> list[Pattern]:
    return [Pattern(i, w.encode("latin-1") if isinstance(w, str) else bytes(w)) for i, w in enumerate(words)]


def _pack(patterns: Sequence[Pattern]) -> tuple[np.ndarray, np.ndarray]:
    offs = np.zeros(len(patterns) + 1, dtype=np.uint64)
    if patterns:
        offs[1:] = np.cumsum([len(p.bytes) for p in patterns], dtype=np.uint64)
    concat = np.frombuffer(b"".join(p.bytes for p in patterns) or b"\0", dtype=np.uint8).copy()
    return concat, offs


class Automaton:
    """The pattern-matching machine (aho_corasick.hpp:58-121). NFA numbering:
    DFS preorder, children in insertion order, root = 0."""

    def __init__(self, handle: int, patterns: list[Pattern]):
        self._h = C.c_void_p(handle)
        self._patterns = patterns

    @classmethod
    def from_arrays(cls, concat: np.ndarray, offs: np.ndarray) -> "Automaton":
        """Build from a packed dictionary (pattern i = concat[offs[i]:offs[i+1]])."""
        concat = np.ascontiguousarray(concat, dtype=np.uint8)
        offs = np.ascontiguousarray(offs, dtype=np.uint64)
        h = C.c_void_p()
        _check(_lib.acg().acg_build(concat.ctypes.data_as(C.c_void_p), offs.ctypes.data_as(C.c_void_p),
                                    len(offs) - 1, C.byref(h)))
        a = cls.__new__(cls)
        a._h = h
        a._patterns = None
        a._packed = (concat, offs)
        return a

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:  # (module globals may be gone at interpreter exit)
            _lib.acg().acg_automaton_destroy(h)
            self._h = C.c_void_p()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def state_count(self) -> int:
        return _lib.acg().acg_state_count(self._h)

    def patterns(self) -> list[Pattern]:
        if self._patterns is None:
            concat, offs = self._packed
            b = concat.tobytes()
            self._patterns = [Pattern(i, b[int(offs[i]):int(offs[i + 1])]) for i in range(len(offs) - 1)]
        return self._patterns

    def pattern_count(self) -> int:
        return _lib.acg().acg_pattern_count(self._h)

    def max_pattern_length(self) -> int:
        return _lib.acg().acg_max_pattern_length(self._h)

    def goto_transition(self, s: int, b: int) -> Optional[int]:
        to = C.c_uint32()
        return to.value if _lib.acg().acg_goto_transition(self._h, s, b, C.byref(to)) else None

    def transitions(self, s: int) -> list[tuple[int, int]]:
        bp, tp = _lib.u8p(), _lib.u32p()
        n = _lib.acg().acg_transitions(self._h, s, C.byref(bp), C.byref(tp))
        return [(bp[i], tp[i]) for i in range(n)]

    def failure(self, s: int) -> int:
        return _lib.acg().acg_failure(self._h, s)

    def outputs(self, s: int) -> list[int]:
        ip = _lib.u32p()
        n = _lib.acg().acg_outputs(self._h, s, C.byref(ip))
        return [ip[i] for i in range(n)]

    def depth(self, s: int) -> int:
        return _lib.acg().acg_depth(self._h, s)

    def nfa_arrays(self) -> dict:
        """The whole NFA as numpy CSR arrays (copies): fail, depth, edge_off,
        edge_byte, edge_to, out_off, out_ids (acg_nfa_arrays)."""
        S = self.state_count()
        ptrs = [C.c_void_p() for _ in range(7)]
        _check(_lib.acg().acg_nfa_arrays(self._h, *[C.byref(p) for p in ptrs]))

        def view(p, n, ct, dt):
            if n == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), shape=(n,)).astype(dt, copy=True)

        edge_off = view(ptrs[2], S + 1, C.c_uint32, np.uint32)
        out_off = view(ptrs[5], S + 1, C.c_uint32, np.uint32)
        return {
            "fail": view(ptrs[0], S, C.c_uint32, np.uint32),
            "depth": view(ptrs[1], S, C.c_uint32, np.uint32),
            "edge_off": edge_off,
            "edge_byte": view(ptrs[3], int(edge_off[-1]), C.c_uint8, np.uint8),
            "edge_to": view(ptrs[4], int(edge_off[-1]), C.c_uint32, np.uint32),
            "out_off": out_off,
            "out_ids": view(ptrs[6], int(out_off[-1]), C.c_uint32, np.uint32),
        }

    def optimize_layout(self, sample: bytes | np.ndarray) -> None:
        """Profile-guided device layout from a text sample (speed only)."""
        arr = np.frombuffer(sample, dtype=np.uint8) if isinstance(sample, (bytes, bytearray)) else sample
        arr = np.ascontiguousarray(arr, dtype=np.uint8)
        _check(_lib.acg().acg_optimize_layout(self._h, arr.ctypes.data_as(C.c_void_p), arr.size))

    def set_hot_limit(self, max_hot_rows: int) -> None:
        """Diagnostics: cap the shared-memory-resident rows (exercises cold paths)."""
        _check(_lib.acg().acg_set_hot_limit(self._h, max_hot_rows))

    def filter_info(self) -> dict:
        """Filter-mode eligibility: q-gram length and Bloom pass rate."""
        q, fp = C.c_uint32(), C.c_double()
        ok = _lib.acg().acg_automaton_filter_info(self._h, C.byref(q), C.byref(fp))
        return {"eligible": bool(ok), "q": q.value, "pass_rate": fp.value}

    def ctab_check(self, text=None) -> dict:
        """Compressed hot automaton (csrc/ctab.hpp): its geometry and, with a
        text, the host replay of the device walk against the dense table."""
        info = (C.c_uint32 * 5)()
        mis, cold = C.c_uint64(), C.c_uint64()
        arr = None if text is None else _as_u8(text)
        ok = _lib.acg().acg_automaton_ctab_check(self._h, None if arr is None else arr.ctypes.data_as(C.c_void_p),
                                                 0 if arr is None else arr.size, info, C.byref(mis), C.byref(cold))
        return {"available": bool(ok), "slots": info[0], "default_depth": info[1], "hot_states": info[2],
                "entries": info[3], "deep": bool(info[4]), "mismatches": mis.value, "cold_steps": cold.value}

    def layout(self) -> dict:
        v = [C.c_uint32() for _ in range(4)]
        mode = C.c_int()
        _check(_lib.acg().acg_automaton_layout(self._h, *[C.byref(x) for x in v], C.byref(mode)))
        return {"states": v[0].value, "hot_rows": v[1].value, "columns": v[2].value, "halo": v[3].value,
                "alphabet": "dna4" if mode.value == 0 else "generic"}


def version() -> str:
    """Library version string (acg_version)."""
    return _lib.acg().acg_version().decode()


def build(patterns: Sequence[Pattern]) -> Automaton:
    """aho_corasick.hpp:130-233. Raises EmptyDictionaryError, EmptyPatternError,
    or Error when ids are not dense in load order (:135-136)."""
    patterns = list(patterns)
    if not patterns:
        raise EmptyDictionaryError("dictionary is empty")
    for i, p in enumerate(patterns):
        if len(p.bytes) == 0:
            raise EmptyPatternError(f"pattern {i} is empty")
        if p.id != i:
            raise Error("pattern ids must be dense and follow load order")
    concat, offs = _pack(patterns)
    h = C.c_void_p()
    _check(_lib.acg().acg_build(concat.ctypes.data_as(C.c_void_p), offs.ctypes.data_as(C.c_void_p),
                                len(patterns), C.byref(h)))
    return Automaton(h.value, patterns)


def next_state(a: Automaton, s: int, b: int) -> int:
    """aho_corasick.hpp:238-245 (total transition function)."""
    return _lib.acg().acg_next_state(a.handle, s, b)


def _as_u8(text) -> np.ndarray:
    if isinstance(text, str):
        text = text.encode("latin-1")
    if isinstance(text, (bytes, bytearray, memoryview)):
        return np.frombuffer(text, dtype=np.uint8) if len(text) else np.zeros(0, np.uint8)
    return np.ascontiguousarray(text, dtype=np.uint8)


@dataclass
class ScanResult:
    ids: np.ndarray          # uint32[M]
    ends: np.ndarray         # uint64[M]
    counts: Optional[np.ndarray] = None  # uint64[P]
    failure_follows: int = 0

    def records(self) -> list[MatchRecord]:
        return [MatchRecord(int(i), int(e)) for i, e in zip(self.ids, self.ends)]


def scan_arrays(a: Automaton, text, flags: int = SCAN_LIST) -> ScanResult:
    """One-shot host scan through acg_scan (H2D, GPU scan, D2H)."""
    arr = _as_u8(text)
    r = C.c_void_p()
    _check(_lib.acg().acg_scan(a.handle, arr.ctypes.data_as(C.c_void_p), arr.size, flags, C.byref(r)))
    try:
        L = _lib.acg()
        m = L.acg_result_match_count(r)
        ids = np.ctypeslib.as_array(L.acg_result_ids(r), shape=(m,)).copy() if m else np.zeros(0, np.uint32)
        ends = np.ctypeslib.as_array(L.acg_result_ends(r), shape=(m,)).copy() if m else np.zeros(0, np.uint64)
        counts = None
        if flags & SCAN_COUNTS:
            p = a.pattern_count()
            cp = L.acg_result_pattern_counts(r)
            counts = np.ctypeslib.as_array(cp, shape=(p,)).copy() if cp else np.zeros(p, np.uint64)
        return ScanResult(ids, ends, counts, L.acg_result_failure_follows(r))
    finally:
        _lib.acg().acg_result_destroy(r)


def scan(a: Automaton, input, stats: Optional[ScanStats] = None) -> list[MatchRecord]:
    """aho_corasick.hpp:250-277: every occurrence, ordered by (end, pattern_id).
    With `stats`, failure follows are counted exactly as the reference does."""
    res = scan_arrays(a, input, SCAN_LIST | (SCAN_STATS if stats is not None else 0))
    if stats is not None:
        stats.failure_follows += res.failure_follows
    return res.records()


def match_count(records) -> int:
    """aho_corasick.hpp:280-282: occurrence count."""
    return len(records)


FORMAT_TSV, FORMAT_JSON = 0, 1


class Scanner:
    """Device-resident scanning (acg_scanner_*): reusable workspace for one
    automaton on one device; `run` enqueues on a CUDA stream without host syncs."""

    def __init__(self, a: Automaton, device: int = 0, flags: int = SCAN_LIST | SCAN_COUNTS):
        self.automaton = a
        self.flags = flags
        h = C.c_void_p()
        _check(_lib.acg().acg_scanner_create(a.handle, device, flags, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            _lib.acg().acg_scanner_destroy(h)
            self._h = C.c_void_p()

    def set_geometry(self, streams_per_thread: int = 0, threads_per_block: int = 0, chunk_bytes: int = 0) -> None:
        _check(_lib.acg().acg_scanner_set_geometry(self._h, streams_per_thread, threads_per_block, chunk_bytes))

    def run(self, d_text_ptr: int, n: int, emit_from: int = 0, base_offset: int = 0, stream: int = 0) -> None:
        _check(_lib.acg().acg_scanner_run(self._h, C.c_void_p(d_text_ptr), n, emit_from, base_offset,
                                          C.c_void_p(stream or None)))

    def run_host(self, text, stream: int = 0) -> None:
        arr = _as_u8(text) if not isinstance(text, int) else None
        ptr, n = (arr.ctypes.data, arr.size)
        _check(_lib.acg().acg_scanner_run_host(self._h, C.c_void_p(ptr), n, C.c_void_p(stream or None)))

    def run_host_ptr(self, ptr: int, n: int, stream: int = 0) -> None:
        _check(_lib.acg().acg_scanner_run_host(self._h, C.c_void_p(ptr), n, C.c_void_p(stream or None)))

    def sync(self) -> None:
        _check(_lib.acg().acg_scanner_sync(self._h))

    def match_count(self) -> int:
        self.sync()
        return _lib.acg().acg_scanner_match_count(self._h)

    def records(self) -> tuple[np.ndarray, np.ndarray]:
        m = self.match_count()
        ids = np.empty(m, dtype=np.uint32)
        ends = np.empty(m, dtype=np.uint64)
        _check(_lib.acg().acg_scanner_records(self._h, ids.ctypes.data_as(C.c_void_p),
                                              ends.ctypes.data_as(C.c_void_p), m))
        return ids, ends

    def packed_records(self) -> tuple[np.ndarray, int]:
        m = self.match_count()
        out = np.empty(m, dtype=np.uint64)
        bits = C.c_uint32()
        _check(_lib.acg().acg_scanner_packed_records(self._h, out.ctypes.data_as(C.c_void_p), m, C.byref(bits)))
        return out, bits.value

    def format(self, fmt: str = "tsv", first: int = 0, count: int | None = None) -> bytes:
        """The match list (records [first, first+count)) as the reference's
        `acmatch match` output, formatted on the GPU (acg_scanner_format)."""
        f = {"tsv": FORMAT_TSV, "json": FORMAT_JSON}[fmt]
        if count is None:
            count = self.match_count() - first
        nb = C.c_uint64()
        _check(_lib.acg().acg_scanner_format(self._h, f, first, count, None, 0, C.byref(nb)))
        buf = np.empty(max(nb.value, 1), np.uint8)
        _check(_lib.acg().acg_scanner_format(self._h, f, first, count, buf.ctypes.data_as(C.c_void_p), buf.size,
                                             C.byref(nb)))
        return buf[:nb.value].tobytes()

    def write_matches(self, path: str, fmt: str = "tsv") -> int:
        """The whole match list to a file (acg_scanner_write_matches); bytes written."""
        f = {"tsv": FORMAT_TSV, "json": FORMAT_JSON}[fmt]
        nb = C.c_uint64()
        fd = os.open(path, os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
        try:
            _check(_lib.acg().acg_scanner_write_matches(self._h, f, fd, C.byref(nb)))
        finally:
            os.close(fd)
        return nb.value

    def copy_records(self, first: int, count: int) -> np.ndarray:
        """Packed records [first, first+count) of the list (acg_scanner_copy_records)."""
        out = np.empty(count, dtype=np.uint64)
        _check(_lib.acg().acg_scanner_copy_records(self._h, first, count, out.ctypes.data_as(C.c_void_p)))
        return out

    def pattern_counts(self) -> np.ndarray:
        out = np.empty(self.automaton.pattern_count(), dtype=np.uint64)
        _check(_lib.acg().acg_scanner_pattern_counts(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def device_pattern_counts_ptr(self) -> int:
        return _lib.acg().acg_scanner_device_pattern_counts(self._h) or 0

    def device_records_ptr(self) -> tuple[int, int]:
        bits = C.c_uint32()
        p = _lib.acg().acg_scanner_device_records(self._h, C.byref(bits))
        return (p or 0), bits.value

    def failure_follows(self) -> int:
        return _lib.acg().acg_scanner_failure_follows(self._h)

    def digest(self) -> tuple[int, int, int]:
        s, x, u = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(_lib.acg().acg_scanner_digest(self._h, C.byref(s), C.byref(x), C.byref(u)))
        return s.value, x.value, u.value

    def kernel_ms(self) -> list[float]:
        """[K1 walk, K1f fix-up, K2 prefix, K3 write, K4 counts] in ms (SCAN_PROFILE)."""
        out = (C.c_float * 5)()
        _check(_lib.acg().acg_scanner_kernel_ms(self._h, out))
        return list(out)

    def set_mode(self, mode: int) -> None:
        _check(_lib.acg().acg_scanner_set_mode(self._h, mode))

    def set_profiling(self, on: bool) -> None:
        """Per-stage event timing for the next runs (kernel_ms)."""
        _check(_lib.acg().acg_scanner_set_profiling(self._h, 1 if on else 0))

    def last_mode(self) -> tuple[str, float]:
        rate = C.c_double()
        m = _lib.acg().acg_scanner_last_mode(self._h, C.byref(rate))
        return {MODE_SPARSE: "sparse", MODE_EXACT: "exact", MODE_FILTER: "filter"}.get(m, "none"), rate.value

    def last_walk(self) -> str:
        """The walk kernel of the last EXACT run: dense hot rows (KE) or the
        compressed hot automaton (KC, csrc/ctab.hpp)."""
        return {0: "dense", 1: "ctab", 2: "sparseg"}.get(_lib.acg().acg_scanner_last_walk(self._h), "none")

    def copy_pattern_counts(self, d_dst_ptr: int, stream: int = 0) -> None:
        _check(_lib.acg().acg_scanner_copy_pattern_counts(self._h, C.c_void_p(d_dst_ptr), C.c_void_p(stream or None)))

    def replays(self) -> int:
        """Runs replayed at sync after a workspace overflow (acg_scanner_replays)."""
        return int(_lib.acg().acg_scanner_replays(self._h))

    def geometry(self) -> dict:
        nc, cb, la = C.c_uint64(), C.c_uint64(), C.c_uint32()
        _check(_lib.acg().acg_scanner_last_geometry(self._h, C.byref(nc), C.byref(cb), C.byref(la)))
        return {"n_chunks": nc.value, "chunk_bytes": cb.value, "launches": la.value}


# ---- input path (reference io.hpp:25-65) and the pipelined host scan ----------

class PinnedInput:
    """acmatch::load_input (io.hpp:25-31): the file's raw bytes, here in
    page-locked host memory (acg_load_input). `.array` is a uint8 view."""

    def __init__(self, path: str):
        ptr, n = C.c_void_p(), C.c_uint64()
        _check(_lib.acg().acg_load_input(os.fsencode(path), C.byref(ptr), C.byref(n)))
        self._ptr, self.n = ptr, n.value
        self.array = (np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(self.n,)) if self.n
                      else np.zeros(0, np.uint8))

    def __del__(self):
        if getattr(self, "_ptr", None) and self._ptr.value and _lib is not None:
            _lib.acg().acg_host_free(self._ptr)
            self._ptr = C.c_void_p()


def load_input(path: str) -> PinnedInput:
    return PinnedInput(path)


class PatternFile(NamedTuple):
    """acmatch::PatternFile (io.hpp:17-22)."""
    patterns: list
    duplicates: int
    skipped_empty: int


def load_patterns(path: str) -> PatternFile:
    """acmatch::load_patterns (io.hpp:37-65) through acg_load_patterns."""
    cp, op, cnt = C.c_void_p(), C.c_void_p(), C.c_uint32()
    dups, empty = C.c_uint64(), C.c_uint64()
    _check(_lib.acg().acg_load_patterns(os.fsencode(path), C.byref(cp), C.byref(op), C.byref(cnt), C.byref(dups),
                                        C.byref(empty)))
    try:
        P = cnt.value
        offs = np.ctypeslib.as_array(C.cast(op, C.POINTER(C.c_uint64)), shape=(P + 1,)).copy()
        total = int(offs[-1])
        data = C.string_at(cp, total) if total else b""
    finally:
        _lib.acg().acg_host_free(cp)
        _lib.acg().acg_host_free(op)
    pats = [Pattern(i, data[int(offs[i]):int(offs[i + 1])]) for i in range(P)]
    return PatternFile(pats, dups.value, empty.value)


def scan_pipelined(a: Automaton, text, device: int = 0, piece_bytes: int = 0, list_cap: int | None = None,
                   counts: bool = True, stats: bool = False, out: np.ndarray | None = None,
                   emit_from: int = 0, base_offset: int = 0):
    """acg_scan_pipelined: (packed records uint64[m] or None, id_bits, counts or
    None, m, failure follows). `text` is a uint8 array (page-locked for full
    speed: PinnedInput.array or a pinned torch tensor's numpy view) or a
    PinnedInput; `out` an optional (pinned) uint64 buffer for the records."""
    arr = text.array if isinstance(text, PinnedInput) else _as_u8(text)
    P = a.pattern_count()
    if out is None and list_cap is not None:
        out = np.empty(max(list_cap, 1), np.uint64)
    cnt = np.zeros(P, np.uint64) if counts else None
    m, ib, fol = C.c_uint64(), C.c_uint32(), C.c_uint64()
    cap = 0 if out is None else (out.size if list_cap is None else min(list_cap, out.size))
    _check(_lib.acg().acg_scan_pipelined(a.handle, device, arr.ctypes.data_as(C.c_void_p) if arr.size else None,
                                         arr.size, emit_from, base_offset, piece_bytes, SCAN_STATS if stats else 0,
                                         out.ctypes.data_as(C.c_void_p) if out is not None else None, cap,
                                         cnt.ctypes.data_as(C.c_void_p) if cnt is not None else None,
                                         C.byref(m), C.byref(ib), C.byref(fol)))
    recs = None if out is None else out[:min(m.value, cap)]
    return recs, ib.value, cnt, m.value, fol.value


# ---- the paper's dictionary-partitioned run (reference partition.hpp:29-170) ----

@dataclass
class PartitionedRun:
    """acmatch::PartitionedRun (partition.hpp:92-99) plus device-timed fields."""
    matches: list
    per_worker_build_s: list
    per_worker_scan_s: list
    total_wall_s: float
    worker_count: int
    workers_launched: int
    per_worker_gpu_scan_s: list = field(default_factory=list)
    h2d_gpu_s: float = 0.0
    merge_gpu_s: float = 0.0
    d2h_s: float = 0.0
    ids: np.ndarray | None = None
    ends: np.ndarray | None = None


def run_partitioned(patterns: Sequence[Pattern], input, worker_count: int, device: int = 0,
                    records: bool = True) -> PartitionedRun:
    """acg_run_partitioned: dictionary split into worker_count contiguous chunks,
    one worker per non-empty chunk, the device-side merge. `records=False`
    skips building the MatchRecord list (ids/ends arrays only)."""
    if worker_count < 1:
        raise InvalidWorkerCountError("worker count must be >= 1")
    concat, offs = _pack(patterns)
    text = _as_u8(input)
    h = C.c_void_p()
    _check(_lib.acg().acg_run_partitioned(concat.ctypes.data_as(C.c_void_p) if concat.size else None,
                                          offs.ctypes.data_as(C.c_void_p), len(patterns),
                                          text.ctypes.data_as(C.c_void_p) if text.size else None, text.size,
                                          worker_count, device, C.byref(h)))
    L = _lib.acg()
    try:
        m = L.acg_partitioned_match_count(h)
        ids = np.ctypeslib.as_array(C.cast(L.acg_partitioned_ids(h), C.POINTER(C.c_uint32)), shape=(m,)).copy() \
            if m else np.zeros(0, np.uint32)
        ends = np.ctypeslib.as_array(C.cast(L.acg_partitioned_ends(h), C.POINTER(C.c_uint64)), shape=(m,)).copy() \
            if m else np.zeros(0, np.uint64)
        wc, launched = C.c_uint32(), C.c_uint32()
        bp, sp, gp = C.c_void_p(), C.c_void_p(), C.c_void_p()
        tot, h2d, mg, d2h = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        _check(L.acg_partitioned_timings(h, C.byref(wc), C.byref(launched), C.byref(bp), C.byref(sp), C.byref(gp),
                                         C.byref(tot), C.byref(h2d), C.byref(mg), C.byref(d2h)))
        k = launched.value

        def arr(p):
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=(k,)).tolist() if k else []

        recs = [MatchRecord(int(i), int(e)) for i, e in zip(ids.tolist(), ends.tolist())] if records else []
        return PartitionedRun(recs, arr(bp), arr(sp), tot.value, wc.value, k,
                              [x * 1e-3 for x in arr(gp)], h2d.value * 1e-3, mg.value * 1e-3, d2h.value * 1e-3,
                              ids, ends)
    finally:
        L.acg_partitioned_destroy(h)


_SINK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64)


def scan_stream(a: Automaton, text, consume, fmt: str | None = None, device: int = 0, piece_bytes: int = 0,
                counts: bool = False):
    """acg_scan_stream: the match list handed window by window to `consume`
    (packed uint64 records and id_bits when fmt is None, else the TSV / JSON
    bytes of cmd_match's output); consume returns a truthy value to stop.
    Returns (m, per-pattern counts or None)."""
    arr = text.array if isinstance(text, PinnedInput) else _as_u8(text)
    f = {None: -1, "tsv": FORMAT_TSV, "json": FORMAT_JSON}[fmt]
    ib_holder = [a.pattern_count()]
    ib = 1
    while (1 << ib) < ib_holder[0]:
        ib += 1

    def sink(_user, data, count):
        try:
            if f < 0:
                view = np.ctypeslib.as_array(C.cast(data, C.POINTER(C.c_uint64)), shape=(count,)) if count else \
                    np.zeros(0, np.uint64)
                stop = consume(view, ib)
            else:
                stop = consume(C.string_at(data, count))
            return 1 if stop else 0
        except Exception:
            return 1

    cb = _SINK(sink)
    cnt = np.zeros(a.pattern_count(), np.uint64) if counts else None
    m, idb = C.c_uint64(), C.c_uint32()
    _check(_lib.acg().acg_scan_stream(a.handle, device, arr.ctypes.data_as(C.c_void_p) if arr.size else None, arr.size,
                                      piece_bytes, f, C.cast(cb, C.c_void_p), None,
                                      cnt.ctypes.data_as(C.c_void_p) if cnt is not None else None,
                                      C.byref(m), C.byref(idb)))
    return m.value, cnt
