#!/bin/bash
# KQ: geometry variants at full size (goldens checked)
cd "$(dirname "$0")/.."
O=gpurun_out/kq2; mkdir -p $O; rm -f $O/bench.*
timeout 600 python -m pytest tests/test_gpu_filter.py -x -q > $O/pytest_filter.log 2>&1; echo "rc=$?" >> $O/pytest_filter.log
for v in "ACG_QKERNEL=16x2" "ACG_QKERNEL=20x2" "ACG_QTLD=0"; do
  echo "== cfg1 $v" >> $O/bench.log
  env $v timeout 600 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 1 >> $O/bench.log 2>> $O/bench.err
done
for v in "ACG_QKERNEL=16x2" "ACG_QKERNEL=20x2"; do
  echo "== cfg2 $v" >> $O/bench.log
  env $v timeout 600 python bench.py --config 2 --steps 10 --no-cpu-baseline --e2e-steps 1 >> $O/bench.log 2>> $O/bench.err
done
echo done
