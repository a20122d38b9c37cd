#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/ctab3; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests/test_gpu_ctab.py tests/test_gpu_events.py tests/test_gpu_scan.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/exact_probe.py 3 2048 exact both profile 0 >> $O/probe.log 2>&1
timeout 300 python tools/exact_probe.py 4 256 exact both bfs 0 >> $O/probe.log 2>&1
timeout 600 python bench.py --config 3 --steps 5 --no-cpu-baseline --profile-layout >> $O/bench.log 2>> $O/bench.err
timeout 600 python bench.py --config 4 --text-mib 256 --steps 3 --no-cpu-baseline >> $O/bench.log 2>> $O/bench.err
echo done
