#!/bin/bash
# Row-cache budget A/B (DISC_ROW_CACHE_KB) on the row-heavy workloads.
out=gpurun_out/ab_rc.txt; : > $out
for w in bert softmax ln_gelu; do
  for kb in ${KBS:-32 48}; do
    v=$(DISC_ROW_CACHE_KB=$kb timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")
    echo "$w kb=$kb $v" >> $out
  done
done
