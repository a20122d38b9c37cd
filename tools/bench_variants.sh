#!/bin/bash
# Bench the default library and every lib/variants/* build (experiments only).
# usage: tools/bench_variants.sh [bench.py args...]
cd "$(dirname "$0")/.."
for v in default $(ls paper_1403_7294_b200/lib/variants 2>/dev/null); do
  if [ "$v" = default ]; then unset ACG_LIBRARY_OVERRIDE; else export ACG_LIBRARY_OVERRIDE=paper_1403_7294_b200/lib/variants/$v/libacg.so; fi
  echo "== $v"
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['stage_ms'], d['config']['scan_mode'], d['config']['excursion_event_rate'], d['check']['golden'])"
done
unset ACG_LIBRARY_OVERRIDE
