#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_filter.py tests/test_gpu_scan.py -m gpu -x -q > gpurun_out/pytest_filter.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_filter.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --config 2 --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --config 4 --text-mib 256 --no-cpu-baseline --steps 3 --e2e-steps 1 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"qfilter_ldg|qconfirm_region|qorder_region" -s 9 -c 3 -o gpurun_out/prof_r9 $CMD > gpurun_out/ncu_full.log 2>&1
CMD2="python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD2 > gpurun_out/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"qfilter_ldg" -s 3 -c 1 -o gpurun_out/prof_cfg2 $CMD2 > gpurun_out/ncu_full_cfg2.log 2>&1
echo done
