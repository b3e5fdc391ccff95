#!/bin/bash
# A/B of in-tree library variants on one box: tools/ab.sh "<variants>" "<workloads>" [reps]
# (variant "base" = libdisc_b200.so; others = libdisc_b200_<v>.so, see build.py)
vars=$1; wls=$2; reps=${3:-2}
for r in $(seq $reps); do for wl in $wls; do for v in $vars; do
  if [ "$v" = base ]; then unset DISC_LIB_VARIANT; else export DISC_LIB_VARIANT=$v; fi
  timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read())
print('$v', '$wl', j['value'], {k: v['GB/s'] for k, v in j['kernel_breakdown'].items()})"
done; done; done
