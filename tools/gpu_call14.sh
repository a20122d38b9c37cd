#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/pytest_scan.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_scan.log
timeout 900 python bench.py --config 3 --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --config 3 --streams-per-thread 4 --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg3u4.json 2> gpurun_out/bench_cfg3u4.err
timeout 900 python bench.py --config 3 --streams-per-thread 1 --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg3u1.json 2> gpurun_out/bench_cfg3u1.err
timeout 900 python bench.py --config 4 --text-mib 256 --streams-per-thread 2 --no-cpu-baseline --steps 3 --e2e-steps 1 > gpurun_out/bench_cfg4u2.json 2> gpurun_out/bench_cfg4u2.err
timeout 900 python bench.py --config 4 --text-mib 256 --no-cpu-baseline --steps 3 --e2e-steps 1 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
echo done
