"""ctypes declarations for lib/libacg.so (include/acg.h) and lib/libacg_synth.so.

The product path is the CUDA library; there is no CPU fallback. If the library
is missing the import of the binding fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")
LIBACG = os.environ.get("ACG_LIBRARY_OVERRIDE") or os.path.join(LIB_DIR, "libacg.so")  # experiments only
LIBSYNTH = os.path.join(LIB_DIR, "libacg_synth.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p

# name: (restype, argtypes) — exactly the symbols declared in include/acg.h
ACG_SYMBOLS = {
    "acg_last_error": (C.c_char_p, []),
    "acg_version": (C.c_char_p, []),
    "acg_build": (C.c_int, [vp, vp, C.c_uint32, C.POINTER(vp)]),
    "acg_automaton_destroy": (None, [vp]),
    "acg_state_count": (C.c_uint32, [vp]),
    "acg_pattern_count": (C.c_uint32, [vp]),
    "acg_max_pattern_length": (C.c_uint32, [vp]),
    "acg_goto_transition": (C.c_int, [vp, C.c_uint32, C.c_uint8, u32p]),
    "acg_transitions": (C.c_uint32, [vp, C.c_uint32, C.POINTER(u8p), C.POINTER(u32p)]),
    "acg_failure": (C.c_uint32, [vp, C.c_uint32]),
    "acg_outputs": (C.c_uint32, [vp, C.c_uint32, C.POINTER(u32p)]),
    "acg_depth": (C.c_uint32, [vp, C.c_uint32]),
    "acg_nfa_arrays": (C.c_int, [vp] + [vp] * 7),
    "acg_next_state": (C.c_uint32, [vp, C.c_uint32, C.c_uint8]),
    "acg_optimize_layout": (C.c_int, [vp, vp, C.c_uint64]),
    "acg_set_hot_limit": (C.c_int, [vp, C.c_uint32]),
    "acg_scan": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.POINTER(vp)]),
    "acg_result_match_count": (C.c_uint64, [vp]),
    "acg_result_ids": (u32p, [vp]),
    "acg_result_ends": (u64p, [vp]),
    "acg_result_pattern_counts": (u64p, [vp]),
    "acg_result_failure_follows": (C.c_uint64, [vp]),
    "acg_result_destroy": (None, [vp]),
    "acg_scanner_create": (C.c_int, [vp, C.c_int, C.c_uint32, C.POINTER(vp)]),
    "acg_scanner_destroy": (None, [vp]),
    "acg_scanner_run": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp]),
    "acg_scanner_run_host": (C.c_int, [vp, vp, C.c_uint64, vp]),
    "acg_scanner_sync": (C.c_int, [vp]),
    "acg_scanner_match_count": (C.c_uint64, [vp]),
    "acg_scanner_records": (C.c_int, [vp, vp, vp, C.c_uint64]),
    "acg_scanner_packed_records": (C.c_int, [vp, vp, C.c_uint64, u32p]),
    "acg_scanner_pattern_counts": (C.c_int, [vp, vp]),
    "acg_scanner_copy_records": (C.c_int, [vp, C.c_uint64, C.c_uint64, vp]),
    "acg_scanner_device_pattern_counts": (vp, [vp]),
    "acg_scanner_device_records": (vp, [vp, u32p]),
    "acg_scanner_failure_follows": (C.c_uint64, [vp]),
    "acg_scanner_digest": (C.c_int, [vp, u64p, u64p, u64p]),
    "acg_scanner_last_geometry": (C.c_int, [vp, u64p, u64p, u32p]),
    "acg_scanner_replays": (C.c_uint64, [vp]),
    "acg_scanner_kernel_ms": (C.c_int, [vp, C.POINTER(C.c_float)]),
    "acg_scanner_copy_pattern_counts": (C.c_int, [vp, vp, vp]),
    "acg_scanner_set_mode": (C.c_int, [vp, C.c_int]),
    "acg_scanner_set_profiling": (C.c_int, [vp, C.c_int]),
    "acg_scanner_last_mode": (C.c_int, [vp, C.POINTER(C.c_double)]),
    "acg_scanner_last_walk": (C.c_int, [vp]),
    "acg_automaton_layout": (C.c_int, [vp, u32p, u32p, u32p, u32p, C.POINTER(C.c_int)]),
    "acg_automaton_filter_info": (C.c_int, [vp, u32p, C.POINTER(C.c_double)]),
    "acg_automaton_ctab_check": (C.c_int, [vp, vp, C.c_uint64, u32p, u64p, u64p]),
    "acg_scanner_set_geometry": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint64]),
    "acg_run_partitioned": (C.c_int, [vp, vp, C.c_uint32, vp, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(vp)]),
    "acg_partitioned_match_count": (C.c_uint64, [vp]),
    "acg_partitioned_ids": (vp, [vp]),
    "acg_partitioned_ends": (vp, [vp]),
    "acg_partitioned_timings": (C.c_int, [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(vp),
                                          C.POINTER(vp), C.POINTER(vp), C.POINTER(C.c_double),
                                          C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "acg_partitioned_destroy": (None, [vp]),
    "acg_scanner_format": (C.c_int, [vp, C.c_int, C.c_uint64, C.c_uint64, vp, C.c_uint64, C.POINTER(C.c_uint64)]),
    "acg_scanner_write_matches": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_uint64)]),
    "acg_scan_stream": (C.c_int, [vp, C.c_int, vp, C.c_uint64, C.c_uint64, C.c_int, vp, vp, vp,
                                  C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]),
    "acg_load_input": (C.c_int, [C.c_char_p, C.POINTER(vp), C.POINTER(C.c_uint64)]),
    "acg_load_patterns": (C.c_int, [C.c_char_p, C.POINTER(vp), C.POINTER(vp), C.POINTER(C.c_uint32),
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "acg_host_free": (None, [vp]),
    "acg_scan_pipelined": (C.c_int, [vp, C.c_int, vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                     vp, C.c_uint64, vp,
                                     C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)]),
}

SYNTH_SYMBOLS = {
    "acg_synth_text": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, vp, C.c_int]),
    "acg_synth_patterns": (C.c_longlong, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                          vp, C.c_uint64, vp]),
}

_acg = None
_synth = None


def _bind(path: str, table: dict) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is not built; run `python -m paper_1403_7294_b200.native` (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in table.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def acg() -> C.CDLL:
    global _acg
    if _acg is None:
        _acg = _bind(LIBACG, ACG_SYMBOLS)
    return _acg


def synth() -> C.CDLL:
    global _synth
    if _synth is None:
        _synth = _bind(LIBSYNTH, SYNTH_SYMBOLS)
    return _synth
