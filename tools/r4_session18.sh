#!/bin/bash
mkdir -p gpurun_out
t=s20
bash tools/r4_ab.sh $t "pf" "softmax bert ln_gelu" 0
for v in pf main pf; do
  if [ $v = main ]; then unset DISC_LIB_VARIANT; else export DISC_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --verify off > gpurun_out/${t}_sweep_$v.json 2>> gpurun_out/${t}_err.log
  python -c "import json; j=json.load(open('gpurun_out/${t}_sweep_$v.json')); print('sweep $v', j['value'], j['large_shape_frac_of_peak'], {k: v['GB/s'] for k, v in j['per_pattern'].items()})"
done
