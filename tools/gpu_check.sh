#!/bin/bash
# One gpurun call: GPU tests (optionally a -k filter), smoke, bench lines.
# usage: tools/gpu_check.sh [pytest -k expr] ; BENCH="args;args" env for extra bench lines
cd "$(dirname "$0")/.."
O=gpurun_out/check
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/nvidia-smi.txt 2>&1
K=${1:-}
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
else
  timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
i=0
BENCH=${BENCH:-$(cat tools/bench_runs.txt 2>/dev/null)}
IFS=';' read -ra RUNS <<< "${BENCH:-}"
for r in "${RUNS[@]}"; do
  i=$((i+1))
  echo "== $r" >> $O/bench.log
  timeout 900 python bench.py $r >> $O/bench.log 2>> $O/bench.err
done
echo done
