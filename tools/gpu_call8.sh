#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_filter.py -m gpu -x -q > gpurun_out/pytest_filter.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_filter.log
timeout 900 python -m pytest tests/test_gpu_golden.py -m gpu -x -q -k "full" > gpurun_out/pytest_golden.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_golden.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --config 2 --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --config 3 --profile-layout --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/bench_cfg3p.json 2> gpurun_out/bench_cfg3p.err
for m in sparse exact; do
timeout 600 python bench.py --config 0 --mode $m --no-cpu-baseline --steps 10 --e2e-steps 1 > gpurun_out/bench_cfg0$m.json 2> gpurun_out/bench_cfg0$m.err
timeout 600 python bench.py --config 4 --text-mib 256 --mode $m --no-cpu-baseline --steps 3 --e2e-steps 1 > gpurun_out/bench_cfg4$m.json 2> gpurun_out/bench_cfg4$m.err
done
echo done
