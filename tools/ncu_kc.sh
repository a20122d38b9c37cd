#!/bin/bash
# ncu --set full (source-level) of the compressed-automaton walk (KC) + E1/E2 on a cfg3 sample;
# exports raw/details/source CSVs (the .ncu-rep stays on the box).
cd "$(dirname "$0")/.."
O=gpurun_out/ncu; mkdir -p $O
R=/tmp/ncu_rep; mkdir -p $R
tag=${1:-kc3}; shift
CMD=${@:-python tools/exact_probe.py 3 256 exact both profile 2}
timeout 300 $CMD > $O/plain_$tag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ctab_event_kernel|exact_event_kernel|event_count|event_expand" \
    -s 12 -c 3 -o $R/$tag -f $CMD > $O/ncu_$tag.log 2>&1
ncu -i $R/$tag.ncu-rep --page raw --csv > $O/${tag}_raw.csv 2>/dev/null
ncu -i $R/$tag.ncu-rep --page details --csv > $O/${tag}_details.csv 2>/dev/null
ncu -i $R/$tag.ncu-rep --page source --csv -k regex:"ctab_event_kernel|exact_event_kernel" > $O/${tag}_source.csv 2>/dev/null
gzip -f $O/${tag}_source.csv
ls -la $O
echo done
