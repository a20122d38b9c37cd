#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/e2; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests -m gpu -x -q -k "ctab or exact or golden or event or scan" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/exact_probe.py 4 256 exact both bfs 0 > $O/probe_cfg4.log 2>&1
timeout 300 python tools/exact_probe.py 3 2048 exact both profile 0 > $O/probe_cfg3.log 2>&1
echo done
