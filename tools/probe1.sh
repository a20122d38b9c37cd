#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/probe; mkdir -p $O
P="timeout 300 python tools/exact_probe.py"
{
$P 1 0 exact both
$P 1 0 exact counts
$P 3 512 exact both
$P 3 512 exact counts
$P 3 512 exact list
$P 3 512 exact both profile
$P 3 512 exact counts profile
$P 4 256 exact both
$P 4 256 exact counts
$P 4 256 exact both profile
$P 4 256 exact counts profile
$P 2 1024 exact both
} > $O/probe1.log 2>&1
