#!/bin/bash
# A/B an environment knob on every workload: tools/ab_env.sh <tag> VAR v1 v2 ...
tag=$1; var=$2; shift 2
for w in ln_gelu softmax colreduce bert; do
  for v in "$@"; do
    echo "$w $var=$v $(env $var=$v python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["value"], d["ms_per_step"], d["large_shape_GBps"])')"
  done
done > gpurun_out/ab_$tag.txt 2>&1
