#!/bin/bash
# A/B of the grouped flush phase count (DISC_GROUP_PHASES) per workload; 2 runs each.
out=gpurun_out/ab_phases.txt; : > $out
for w in stream ln_gelu bert softmax; do
  for p in 2 3 4 6; do
    for rep in 1 2; do
      v=$(DISC_GROUP_PHASES=$p timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")
      echo "$w phases=$p $v" >> $out
    done
  done
done
