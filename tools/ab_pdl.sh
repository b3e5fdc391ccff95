#!/bin/bash
# A/B of the PDL modes on every workload: tools/ab_pdl.sh <tag>
tag=$1
for w in ln_gelu softmax colreduce bert; do
  for m in 0 1 2; do
    echo "$w pdl=$m $(python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --pdl $m 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["value"], d["ms_per_step"])')"
  done
done > gpurun_out/ab_$tag.txt 2>&1
