#!/bin/bash
# A/B experiment on one GPU box: bench lines for the default library and for
# lib/variants/<name>/libacg.so builds (native.build_variant), per config.
# usage: tools/gpu_ab.sh "<variant> ..." "<bench args>;<bench args>;..." [log]
# e.g.   tools/gpu_ab.sh "text_cs text_128" "--config 3 --steps 5;--config 4 --text-mib 256 --steps 3"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LOG=${3:-gpurun_out/ab.log}
rm -f "$LOG"
IFS=';' read -ra RUNS <<< "$2"
for v in default $1; do
  if [ "$v" = default ]; then unset ACG_LIBRARY_OVERRIDE; else export ACG_LIBRARY_OVERRIDE=paper_1403_7294_b200/lib/variants/$v/libacg.so; fi
  echo "== $v" >> "$LOG"
  for r in "${RUNS[@]}"; do
    timeout 600 python bench.py $r --no-cpu-baseline --e2e-steps 1 >> "$LOG" 2>&1
  done
done
