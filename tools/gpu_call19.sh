#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_filter.py -m gpu -x -q > gpurun_out/pytest_filter.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_filter.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --config 2 --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
CMD3="python bench.py --config 3 --text-mib 256 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD3 > gpurun_out/plain3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"exact_scan_kernel<2, 1, 2" -c 1 -o gpurun_out/prof_cfg3s $CMD3 > gpurun_out/ncu_full3.log 2>&1
echo done
