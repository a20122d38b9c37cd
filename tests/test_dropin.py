"""The reference's OWN C++ unit tests and acceptance runner, compiled
unmodified against the drop-in headers (include/acmatch/*.hpp) and linked to
libacg.so (oracle/Makefile: reftests). Passing them is the drop-in claim: a
reference user recompiles against these headers and their tests still pass,
with every scan running on the GPU.

The binaries are built in this container (they need the reference sources)
and travel prebuilt to the GPU box under oracle/_ref/; without them these
tests skip.

CPU tests run the host-only cases (automaton construction, next_state,
dictionary split, merge, and the reference's corpus/io helpers); every case
that scans needs a device and runs under -m gpu.
"""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = os.path.join(ROOT, "oracle", "_ref", "ref_unit_dropin")
ACCEPT = os.path.join(ROOT, "oracle", "_ref", "ref_acceptance_dropin")

# Cases that call scan() (directly or through run_partitioned / run_benchmark).
SCANNING = "Scan.*:RunPartitioned.*:RunBenchmark.*:SweepFileSizes.*:WriteCsv.*:GenerateCorpus.FullPlantGuaranteesCoverage"
HOST_ONLY = "-" + SCANNING


def _need(path: str) -> None:
    if not os.path.exists(path):
        pytest.skip(f"{os.path.relpath(path, ROOT)} not built (needs /root/reference at build time)")


def _run(cmd: list[str], timeout: int) -> subprocess.CompletedProcess:
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def _summary(p: subprocess.CompletedProcess) -> str:
    return (p.stdout[-4000:] + "\n" + p.stderr[-4000:]).strip()


def test_reference_unit_tests_host_only():
    _need(UNIT)
    listed = _run([UNIT, "--list", f"--gtest_filter={HOST_ONLY}"], 60).stdout.split()
    assert len(listed) >= 45, listed  # Build, NextState, Automaton, SplitPatterns, MergeMatches, corpus/io
    p = _run([UNIT, f"--gtest_filter={HOST_ONLY}"], 600)
    assert p.returncode == 0, _summary(p)
    assert f"{len(listed)} tests ran, {len(listed)} passed, 0 failed" in p.stdout


def test_reference_acceptance_host_only_criterion():
    _need(ACCEPT)
    p = _run([ACCEPT, "--criterion", "2"], 120)  # failure-transition trace: build + next_state only
    assert p.returncode == 0, _summary(p)
    assert "PASS" in p.stdout


@pytest.mark.gpu
def test_reference_unit_tests_all_on_gpu():
    _need(UNIT)
    p = _run([UNIT], 1800)
    assert p.returncode == 0, _summary(p)
    assert "0 failed" in p.stdout
    assert "Scan.MatchesNaiveOracle" in p.stdout and "RunPartitioned.PartitionInvarianceAtCorpusScale" in p.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("criterion", [1, 3, 4, 5, 6, 7, 8])
def test_reference_acceptance_criterion_on_gpu(criterion):
    _need(ACCEPT)
    p = _run([ACCEPT, "--criterion", str(criterion)], 1800)
    # 77 = the criterion skipped itself (criterion 7 below 4 hardware threads)
    assert p.returncode in (0, 77), _summary(p)
    assert ("PASS" in p.stdout) or ("SKIP" in p.stdout), _summary(p)


EXT = os.path.join(ROOT, "oracle", "_ref", "dropin_ext_tests")


@pytest.mark.gpu
def test_dropin_extensions_on_gpu():
    """This repo's C++ tests of the drop-in's extensions (tests/cpp/test_dropin_ext.cpp):
    device-timed run_partitioned fields, GPU benchmark rows and CSV, pinned-input scan."""
    _need(EXT)
    p = _run([EXT], 600)
    assert p.returncode == 0, _summary(p)
    assert "0 failed" in p.stdout
