#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (ours + reference arm), every
# config's bench line, ncu launch list and full captures of the dominant kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/round
O=gpurun_out/round
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for c in 0 2 3; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --e2e-steps 1 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 900 python bench.py --config 4 --text-mib 256 --no-cpu-baseline --steps 3 --e2e-steps 1 > $O/bench_cfg4_256MiB.json 2> $O/bench_cfg4.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg1.csv $CMD > $O/ncu_launches.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"qfilter_ldg|qconfirm_region|qorder_region" -s 9 -c 3 -o $O/prof_cfg1 $CMD > $O/ncu_full.log 2>&1
CMD3="python bench.py --config 3 --text-mib 256 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD3 > $O/plain3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"exact_scan_kernel<\(int\)2, \(int\)1, \(int\)2" -c 1 -o $O/prof_cfg3 $CMD3 > $O/ncu_full3.log 2>&1
echo done
