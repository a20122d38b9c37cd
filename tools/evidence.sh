#!/bin/bash
# One gpurun call of round evidence: GPU tests, smoke, bench lines, the ncu
# launch list of the default bench command and one --set full capture of the
# EXACT walk (KE) on cfg3 (CSV exports; the .ncu-rep stays on the box).
cd "$(dirname "$0")/.."
O=gpurun_out/evidence; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
BENCH=${BENCH:-"--steps 20;--config 0 --steps 20;--config 2 --steps 10 --no-cpu-baseline;--config 3 --steps 5 --no-cpu-baseline --profile-layout;--config 3 --steps 5 --no-cpu-baseline;--config 4 --text-mib 256 --steps 3 --no-cpu-baseline;--mode exact --steps 10 --no-cpu-baseline;--mode sparse --steps 10 --no-cpu-baseline"}
IFS=';' read -ra RUNS <<< "$BENCH"
for r in "${RUNS[@]}"; do
  echo "== $r" >> $O/bench.log
  timeout 900 python bench.py $r >> $O/bench.log 2>> $O/bench.err
done
timeout 600 python bench.py --steps 20 --impl reference > $O/bench_reference.json 2>> $O/bench.err
if [ -z "$NO_NCU" ]; then
  timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg1.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_launch.log 2>&1
  # --set full of the cfg1 step's kernels (KQ, V1, ORDER) at the bench's size
  C1="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qfilter_ldg|qconfirm_region|qorder_region" \
      -s 9 -c 3 -o /tmp/kq1 -f $C1 > $O/ncu_kq1.log 2>&1
  ncu -i /tmp/kq1.ncu-rep --page raw --csv > $O/ncu_cfg1_raw.csv 2>/dev/null
  ncu -i /tmp/kq1.ncu-rep --page details --csv > $O/ncu_cfg1_details.csv 2>/dev/null
  # --set full of the EXACT walk over the compressed hot automaton (KC) + E2 on cfg3 at the bench's full size
  C3="python tools/exact_probe.py 3 2048 exact both profile 0"
  timeout 300 $C3 > $O/plain_kc3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ctab_event_kernel|exact_event_kernel|event_count|event_expand" \
      -s 8 -c 2 -o /tmp/kc3 -f $C3 > $O/ncu_kc3.log 2>&1
  ncu -i /tmp/kc3.ncu-rep --page raw --csv > $O/ncu_kc_cfg3_raw.csv 2>/dev/null
  ncu -i /tmp/kc3.ncu-rep --page details --csv > $O/ncu_kc_cfg3_details.csv 2>/dev/null
  # --set full of KQ with the two-level filter (cfg2) at the bench's full size
  C2="python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qfilter_ldg" -s 4 -c 1 -o /tmp/kq2 -f $C2 > $O/ncu_kq2.log 2>&1
  ncu -i /tmp/kq2.ncu-rep --page raw --csv > $O/ncu_cfg2_raw.csv 2>/dev/null
  ncu -i /tmp/kq2.ncu-rep --page details --csv > $O/ncu_cfg2_details.csv 2>/dev/null
fi
echo done
