#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for o in "" "--no-counts"; do
timeout 900 python bench.py --config 3 --text-mib 512 $o --no-cpu-baseline --steps 5 --e2e-steps 1 >> gpurun_out/cfg3_exp.log 2>&1
done
timeout 900 python bench.py --config 3 --text-mib 512 --streams-per-thread 8 --no-cpu-baseline --steps 5 --e2e-steps 1 >> gpurun_out/cfg3_exp.log 2>&1
timeout 900 python bench.py --config 3 --text-mib 512 --streams-per-thread 2 --no-cpu-baseline --steps 5 --e2e-steps 1 >> gpurun_out/cfg3_exp.log 2>&1
CMD="python bench.py --config 3 --text-mib 256 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"exact_scan" -s 4 -c 1 -o gpurun_out/prof_cfg3b $CMD > gpurun_out/ncu_full3.log 2>&1
echo done
