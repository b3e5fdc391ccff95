#!/bin/bash
# odd-width row schedule knobs on softmax: per-shape scans + the softmax workload
mkdir -p gpurun_out
t=s12
S="S1=9,13,17,31,33,65,255,1025"
for kv in "X=0" "DISC_UNALIGNED_MIN=8" "DISC_UNALIGNED_MIN=64" "DISC_SHORT_MAX=16" "DISC_SHORT_MAX=32" "DISC_UNALIGNED_ROWS=0"; do
  n=$(echo $kv | tr ' =' '__')
  env $kv timeout 300 python tools/shape_scan.py softmax "$S" --copies-gb 2 > gpurun_out/${t}_scan_$n.txt 2>&1
  env $kv timeout 300 python bench.py --workload softmax --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --verify off > gpurun_out/${t}_sm_$n.json 2>> gpurun_out/${t}_err.log
  python -c "import json; j=json.load(open('gpurun_out/${t}_sm_$n.json')); print('softmax $kv', j['value'], j['large_shape_frac_of_peak'])"
  awk '{print \$2, \$(NF-2), \$(NF-1)}' gpurun_out/${t}_scan_$n.txt | tr '\n' ' '; echo
done
