#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/kc; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests -m gpu -x -q -k "ctab or exact or golden or event" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/exact_probe.py 3 2048 exact both profile 0 > $O/probe_profile.log 2>&1
timeout 300 python tools/exact_probe.py 3 2048 exact both bfs 0 > $O/probe_bfs.log 2>&1
echo done
