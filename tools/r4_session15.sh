#!/bin/bash
mkdir -p gpurun_out
t=s16
for cfg in "128 120 16" "160 125 16" "128 120 24"; do
  set -- $cfg
  DISC_GROUP_WAVES=$3 timeout 600 python bench.py --no-cpu-baseline --no-e2e --verify off --chunk-gb $1 --reserve-gb $2 > gpurun_out/${t}_sweep_$1_$3.json 2>> gpurun_out/${t}_err.log
  python -c "import json; j=json.load(open('gpurun_out/${t}_sweep_$1_$3.json')); print('sweep chunk $1 waves $3', j['value'], j['large_shape_frac_of_peak'], j.get('host_bound_frac'))"
done
