#!/bin/bash
# A/B of an environment knob on one workload: tools/ab_knob.sh <VAR> "<values>" <workload> [reps]
var=$1; vals=$2; wl=$3; reps=${4:-1}
for r in $(seq $reps); do for v in $vals; do
  env $var=$v timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read())
print('$var=$v', '$wl', j['value'], {k: v['GB/s'] for k, v in j['kernel_breakdown'].items()})"
done; done
