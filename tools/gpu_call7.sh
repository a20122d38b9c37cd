#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_filter.py -m gpu -x -q > gpurun_out/pytest_scan.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_scan.log
timeout 900 python -m pytest tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/pytest_golden.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_golden.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --config 2 --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --config 2 --mode sparse --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg2s.json 2> gpurun_out/bench_cfg2s.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"qconfirm_region" -s 3 -c 1 -o gpurun_out/prof_v1 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
