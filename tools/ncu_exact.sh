#!/bin/bash
# ncu --set full (source-level) of the exact walk on cfg3 / cfg4 samples
cd "$(dirname "$0")/.."
O=gpurun_out/ncu; mkdir -p $O
C3="python tools/exact_probe.py 3 256 exact both"
C4="python tools/exact_probe.py 4 64 exact both"
timeout 300 $C3 > $O/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exact_scan_kernel -s 8 -c 1 -o $O/exact_cfg3 $C3 > $O/ncu3.log 2>&1
timeout 300 $C4 > $O/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"exact_scan_kernel|scratch_copy" -s 8 -c 2 -o $O/exact_cfg4 $C4 > $O/ncu4.log 2>&1
echo done
