#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
(timeout 300 tools/partition_timing; timeout 300 tools/partition_timing 8) > gpurun_out/partition_timing.log 2>&1
timeout 600 python -m pytest tests/test_dropin.py -m gpu -x -q > gpurun_out/pytest_dropin.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dropin.log
timeout 600 python -m pytest tests/test_gpu_filter.py -m gpu -x -q > gpurun_out/pytest_filter.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_filter.log
ACG_QKERNEL=24x2 timeout 600 python -m pytest tests/test_gpu_filter.py -m gpu -x -q > gpurun_out/pytest_filter24.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_filter24.log
for v in ring 16x2 16x3 24x2 8x4; do
  echo "== $v" >> gpurun_out/variants.log
  ACG_QKERNEL=$v timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 >> gpurun_out/variants.log 2>&1
done
for qw in 36864 57344; do
  echo "== 16x2 qwords $qw" >> gpurun_out/variants.log
  ACG_QWORDS=$qw ACG_QKERNEL=16x2 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 >> gpurun_out/variants.log 2>&1
done
timeout 300 python tools/time_runs.py > gpurun_out/time_runs.log 2>&1
echo done
