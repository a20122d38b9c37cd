"""B200-native Aho-Corasick text scan behind the reference `acmatch` API.

The product is lib/libacg.so (C ABI: include/acg.h; C++ drop-in headers:
include/acmatch/*.hpp). This package is its Python binding plus the
workload generator and the shard runner used by the benchmark.
"""
from .acmatch import (  # noqa: F401
    SCAN_COUNTS,
    SCAN_LIST,
    SCAN_STATS,
    Automaton,
    DeviceError,
    EmptyDictionaryError,
    EmptyPatternError,
    Error,
    InvalidWorkerCountError,
    MatchRecord,
    Pattern,
    Scanner,
    ScanResult,
    ScanStats,
    build,
    kRoot,
    make_patterns,
    match_before,
    match_count,
    next_state,
    scan,
    scan_arrays,
)

__all__ = [name for name in dir() if not name.startswith("_")]
