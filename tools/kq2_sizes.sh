#!/bin/bash
# separates the dictionary effect from the text-size effect on KQ
cd "$(dirname "$0")/.."
O=gpurun_out/kq2s; mkdir -p $O; rm -f $O/*
for r in "--config 1 --text-mib 8192 --steps 10" "--config 1 --text-mib 4096 --steps 10" "--config 2 --text-mib 1024 --steps 10" "--config 2 --text-mib 2048 --steps 10" "--config 2 --text-mib 4096 --steps 10"; do
  echo "== $r" >> $O/bench.log
  timeout 600 python bench.py $r --no-cpu-baseline --e2e-steps 1 >> $O/bench.log 2>> $O/bench.err
done
echo done
