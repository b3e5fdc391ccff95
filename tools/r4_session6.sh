#!/bin/bash
# GPU session: compensated-f32 column sums (variant comp), grouped-call size on the sweep.
mkdir -p gpurun_out
t=s7
bash tools/r4_ab.sh $t "main comp" "colreduce" 0
for cfg in "32 64" "64 100" "128 120"; do
  set -- $cfg
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --chunk-gb $1 --reserve-gb $2 > gpurun_out/${t}_sweep_c$1.json 2>> gpurun_out/${t}_err.log
  python -c "import json; j=json.load(open('gpurun_out/${t}_sweep_c$1.json')); print('sweep chunk $1', j['value'], j['ms_per_step'], j['large_shape_frac_of_peak'], j['roofline']['frac'], j.get('host_bound_frac'))"
done
