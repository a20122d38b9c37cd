#!/bin/bash
# One gpurun call: KC (compressed hot automaton) parity tests and cfg3 timings
# against KE (ACG_CTAB=0), per stream interleave.
cd "$(dirname "$0")/.."
O=gpurun_out/ctab; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests/test_gpu_ctab.py tests/test_gpu_events.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for u in 1 2 4; do
  timeout 300 python tools/exact_probe.py 3 256 exact both profile $u >> $O/probe.log 2>&1
done
timeout 300 python tools/exact_probe.py 3 256 exact both bfs 0 >> $O/probe.log 2>&1
timeout 300 python tools/exact_probe.py 3 2048 exact both profile 1 >> $O/probe.log 2>&1
timeout 300 python tools/exact_probe.py 3 2048 exact both profile 2 >> $O/probe.log 2>&1
ACG_CTAB=0 timeout 300 python tools/exact_probe.py 3 256 exact both profile 2 >> $O/probe.log 2>&1
timeout 600 python bench.py --config 3 --steps 5 --no-cpu-baseline --profile-layout >> $O/bench.log 2>> $O/bench.err
echo done
