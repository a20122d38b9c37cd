"""GPU parity of the GPU-native dictionary-partitioned run (acg_run_partitioned:
one device copy of the input, concurrent per-chunk builds and scans, the
workers' lists merged ON THE DEVICE) against the REFERENCE's own
run_partitioned (oracle/_ref: proj/include/acmatch/partition.hpp:108-170) —
merged lists, workers launched, timing fields sized to the launched workers —
including more workers than patterns (empty chunks), one worker, dense
output with many duplicate ends across chunks, and the errors."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import oracle
from paper_1403_7294_b200 import acmatch as am
from paper_1403_7294_b200 import synth

pytestmark = pytest.mark.gpu


def ref_partitioned(concat, offs, text, workers):
    cap = 1 << 22
    ids = np.zeros(cap, np.uint32)
    ends = np.zeros(cap, np.uint64)
    m, wall, launched = C.c_uint64(), C.c_double(), C.c_uint32()
    rc = oracle.ref().ref_run_partitioned(oracle._ptr(concat), oracle._ptr(offs), len(offs) - 1, oracle._ptr(text),
                                          text.size, workers, oracle._ptr(ids), oracle._ptr(ends), cap, C.byref(m),
                                          C.byref(wall), C.byref(launched))
    assert rc == 0 and m.value <= cap
    return ids[:m.value], ends[:m.value], launched.value


@pytest.mark.parametrize("cfg,mib,patterns", [(0, 2, 1000), (3, 1, 800), (4, 1, 600)])
@pytest.mark.parametrize("workers", [1, 2, 3, 7, 16])
def test_partitioned_matches_reference(cfg, mib, patterns, workers):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref is not built")
    w = synth.CONFIGS[cfg].scaled(mib << 20, patterns)
    text = synth.text(w)
    concat, offs = synth.patterns(w)
    pats = am.make_patterns(synth.pattern_list(concat, offs))
    run = am.run_partitioned(pats, text, workers, records=False)
    rids, rends, launched = ref_partitioned(concat, offs, text, workers)
    assert np.array_equal(run.ends, rends) and np.array_equal(run.ids, rids)
    assert run.workers_launched == launched == min(workers, len(pats))
    assert len(run.per_worker_build_s) == len(run.per_worker_scan_s) == len(run.per_worker_gpu_scan_s) == launched
    assert all(g > 0 for g in run.per_worker_gpu_scan_s) and run.total_wall_s > 0


def test_more_workers_than_patterns_and_worked_example():
    pats = am.make_patterns([b"AB", b"BC"])
    run = am.run_partitioned(pats, b"ABCABC", 16)
    assert run.matches == [am.MatchRecord(0, 1), am.MatchRecord(1, 2), am.MatchRecord(0, 4), am.MatchRecord(1, 5)]
    assert run.workers_launched == 2 and run.worker_count == 16


def test_errors():
    with pytest.raises(am.InvalidWorkerCountError):
        am.run_partitioned(am.make_patterns([b"A"]), b"AAA", 0)
    with pytest.raises(am.EmptyDictionaryError):
        am.run_partitioned([], b"AAA", 2)
    with pytest.raises(am.EmptyPatternError):
        am.run_partitioned(am.make_patterns([b"A", b"", b"C"]), b"AAA", 2)
