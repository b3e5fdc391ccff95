#!/bin/bash
# tanh's exp on the FMA pipe (variant xp) vs MUFU ex2
mkdir -p gpurun_out
t=s14
bash tools/r4_ab.sh $t "main xp" "colreduce ln_gelu bert" 0
DISC_LIB_VARIANT=xp timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "transcendental or special or random_graphs_oracle" > gpurun_out/${t}_tests_xp.log 2>&1; tail -1 gpurun_out/${t}_tests_xp.log
for v in main xp; do
  if [ $v = main ]; then unset DISC_LIB_VARIANT; else export DISC_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --verify off > gpurun_out/${t}_sweep_$v.json 2>> gpurun_out/${t}_err.log
  python -c "import json; j=json.load(open('gpurun_out/${t}_sweep_$v.json')); print('sweep $v', j['value'], j['large_shape_frac_of_peak'])"
done
