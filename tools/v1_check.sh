#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/v1; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests -m gpu -x -q -k "filter or golden or long" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in 0 1 2 0 1 2; do
  echo "== ACG_V1_FORM=$v" >> $O/bench.log
  ACG_V1_FORM=$v timeout 600 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 1 >> $O/bench.log 2>> $O/bench.err
done
for v in 0 1; do
  echo "== cfg2 ACG_V1_FORM=$v" >> $O/bench.log
  ACG_V1_FORM=$v timeout 600 python bench.py --config 2 --steps 10 --no-cpu-baseline --e2e-steps 1 >> $O/bench.log 2>> $O/bench.err
done
echo done
