#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD3="python bench.py --config 3 --text-mib 256 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD3 > gpurun_out/plain3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"exact_scan_kernel<\(int\)2, \(int\)1, \(int\)2" -c 1 -o gpurun_out/prof_cfg3s $CMD3 > gpurun_out/ncu_full3.log 2>&1
echo done
