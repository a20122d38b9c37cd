#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/counts_exp.log
for o in "" "--no-counts"; do
  timeout 600 python bench.py --config 3 $o --no-cpu-baseline --steps 5 --e2e-steps 1 >> gpurun_out/counts_exp.log 2>&1
  timeout 600 python bench.py --config 4 --text-mib 256 $o --no-cpu-baseline --steps 3 --e2e-steps 1 >> gpurun_out/counts_exp.log 2>&1
done
echo done
