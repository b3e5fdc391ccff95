#!/bin/bash
# GPU session: grouped-launch knobs at 128 GB grouped calls, tests.
mkdir -p gpurun_out
t=s8
for kv in "DISC_GROUP_WAVES=16" "DISC_GROUP_WAVES=32" "DISC_GROUP_WAVES=8" "DISC_GROUP_PHASES=1" "DISC_GROUP_PHASES=3"; do
  env $kv timeout 600 python bench.py --no-cpu-baseline --no-e2e --verify off > gpurun_out/${t}_sweep_$kv.json 2>> gpurun_out/${t}_err.log
  python -c "import json; j=json.load(open('gpurun_out/${t}_sweep_$kv.json')); print('sweep $kv', j['value'], j['ms_per_step'], j['large_shape_frac_of_peak'], j['roofline']['frac'], j.get('host_bound_frac'))"
done
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/${t}_tests.log 2>&1
tail -2 gpurun_out/${t}_tests.log
