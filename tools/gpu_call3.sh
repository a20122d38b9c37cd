#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in 0 2 3 4; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:qfilter_ldg -s 3 -c 1 -o gpurun_out/prof_qfilter_ldg $CMD > gpurun_out/ncu_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:qconfirm -s 3 -c 1 -o gpurun_out/prof_qconfirm $CMD > gpurun_out/ncu_full2.log 2>&1
echo done
