#!/bin/bash
# ncu --set full (source-level) of the EXACT event walk (KE) + E1/E2 on cfg3 / cfg4 samples;
# exports raw/details/source CSVs on the box (the .ncu-rep files stay there: too big to bring back)
cd "$(dirname "$0")/.."
O=gpurun_out/ncu; mkdir -p $O
R=/tmp/ncu_rep; mkdir -p $R
run() {  # tag cmd...
    local tag=$1; shift
    timeout 300 "$@" > $O/plain_$tag.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"exact_event_kernel|event_count|event_expand" \
        -s 12 -c 3 -o $R/$tag -f "$@" > $O/ncu_$tag.log 2>&1
    ncu -i $R/$tag.ncu-rep --page raw --csv > $O/${tag}_raw.csv 2>/dev/null
    ncu -i $R/$tag.ncu-rep --page details --csv > $O/${tag}_details.csv 2>/dev/null
    ncu -i $R/$tag.ncu-rep --page source --csv -k regex:exact_event_kernel > $O/${tag}_source.csv 2>/dev/null
    gzip -f $O/${tag}_source.csv
}
run cfg3 python tools/exact_probe.py 3 256 exact both
run cfg4 python tools/exact_probe.py 4 64 exact both
ls -la $O
echo done
