#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_filter.py -m gpu -x -q > gpurun_out/pytest_scan.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_scan.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --config 4 --text-mib 256 --no-cpu-baseline --steps 3 --e2e-steps 1 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 900 python bench.py --config 2 --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --config 0 --no-cpu-baseline --steps 10 --e2e-steps 1 > gpurun_out/bench_cfg0.json 2> gpurun_out/bench_cfg0.err
echo done
