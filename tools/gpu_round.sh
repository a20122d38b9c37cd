#!/bin/bash
# One gpurun call: GPU tests, bench (ours + reference arm), ncu launch list and
# one full capture of the dominant kernel. usage: tools/gpu_round.sh [kernel-regex]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-qfilter_kernel}
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_full.log 2>&1
echo "done"
