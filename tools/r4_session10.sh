#!/bin/bash
# register-cap policy for fused sum rows on the 128 GB-call sweep
mkdir -p gpurun_out
t=s11
for kv in "DISC_SUM_ROW_MB=0" "DISC_SUM_ROW_MB=3" "DISC_SUM_ROW_MB=1" "DISC_SUM_ROW_MB=3 DISC_REGCAP_KEY=1"; do
  n=$(echo $kv | tr ' =' '__')
  env $kv timeout 600 python bench.py --no-cpu-baseline --no-e2e --verify off > gpurun_out/${t}_sweep_$n.json 2>> gpurun_out/${t}_err.log
  python -c "import json; j=json.load(open('gpurun_out/${t}_sweep_$n.json')); print('sweep $kv', j['value'], j['ms_per_step'], j['large_shape_frac_of_peak'], {k: v['GB/s'] for k, v in j['per_pattern'].items()})"
done
