#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_golden.py tests/test_dropin.py -m gpu -x -q > gpurun_out/pytest_scan.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_scan.log
rm -f gpurun_out/counts_exp.log
timeout 600 python bench.py --config 3 --no-cpu-baseline --steps 5 --e2e-steps 1 >> gpurun_out/counts_exp.log 2>&1
timeout 600 python bench.py --config 4 --text-mib 256 --no-cpu-baseline --steps 3 --e2e-steps 1 >> gpurun_out/counts_exp.log 2>&1
timeout 600 python bench.py --config 0 --no-cpu-baseline --steps 10 --e2e-steps 1 >> gpurun_out/counts_exp.log 2>&1
echo done
