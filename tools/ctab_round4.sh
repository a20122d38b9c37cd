#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/ctab4; mkdir -p $O; rm -f $O/*
for b in 2 4 6 8; do
  echo "== ACG_E2_VIS_BLOCKS=$b" >> $O/probe.log
  ACG_E2_VIS_BLOCKS=$b timeout 300 python tools/exact_probe.py 3 2048 exact both profile 0 >> $O/probe.log 2>&1
done
echo done
