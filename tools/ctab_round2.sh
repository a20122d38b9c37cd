#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/ctab2; mkdir -p $O; rm -f $O/*
for al in 256 1024; do
for c in 512 1024 2048 4096; do
  echo "== ACG_KC_CHUNK=$c ACG_KC_ALIGN=$al" >> $O/probe.log
  ACG_KC_ALIGN=$al ACG_KC_CHUNK=$c timeout 300 python tools/exact_probe.py 3 2048 exact both profile 0 >> $O/probe.log 2>&1
done; done
bash tools/gpu_ab.sh "kq_pin" "--steps 20;--config 2 --steps 10" $O/ab_kq.log
echo done
