#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/unroll_exp.log
for v in default unroll4 unroll8; do
  if [ "$v" = default ]; then unset ACG_LIBRARY_OVERRIDE; else export ACG_LIBRARY_OVERRIDE=paper_1403_7294_b200/lib/variants/$v/libacg.so; fi
  echo "== $v" >> gpurun_out/unroll_exp.log
  timeout 600 python bench.py --config 3 --no-cpu-baseline --steps 5 --e2e-steps 1 >> gpurun_out/unroll_exp.log 2>&1
  timeout 600 python bench.py --config 4 --text-mib 256 --no-cpu-baseline --steps 3 --e2e-steps 1 >> gpurun_out/unroll_exp.log 2>&1
  timeout 600 python bench.py --config 0 --mode exact --no-cpu-baseline --steps 10 --e2e-steps 1 >> gpurun_out/unroll_exp.log 2>&1
done
echo done
