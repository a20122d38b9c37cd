#!/bin/bash
# event pipeline: GPU tests of the exact mode + timing probes
cd "$(dirname "$0")/.."
O=gpurun_out/probe; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "events or exact or golden or gpu_scan" > $O/pytest2.log 2>&1; echo "rc=$?" >> $O/pytest2.log
P="timeout 300 python tools/exact_probe.py"
{
$P 1 0 exact both
$P 3 512 exact both
$P 3 512 exact counts
$P 3 512 exact both profile
$P 4 256 exact both
$P 4 256 exact counts
$P 4 256 exact both profile
$P 2 1024 exact both
ACG_EXACT_EVENTS=0 $P 3 512 exact both
ACG_EXACT_EVENTS=0 $P 4 256 exact both
} > $O/probe2.log 2>&1
