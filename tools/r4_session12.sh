#!/bin/bash
# block-staged short rows with batched copies (variant cb4) vs the default schedule
mkdir -p gpurun_out
t=s13
S="S1=2,3,7,9,13,17,24,31"
timeout 300 python tools/shape_scan.py softmax "$S" --copies-gb 2 > gpurun_out/${t}_scan_main.txt 2>&1
for sm in 9 2; do
  DISC_LIB_VARIANT=cb4 DISC_STAGE_MIN=$sm timeout 300 python tools/shape_scan.py softmax "$S" --copies-gb 2 > gpurun_out/${t}_scan_cb4_$sm.txt 2>&1
done
DISC_LIB_VARIANT=cb4 DISC_STAGE_MIN=9 timeout 600 python bench.py --no-cpu-baseline --no-e2e --verify off > gpurun_out/${t}_sweep_cb4.json 2>> gpurun_out/${t}_err.log
python -c "import json; j=json.load(open('gpurun_out/${t}_sweep_cb4.json')); print('sweep cb4 stage9', j['value'], j['large_shape_frac_of_peak'])"
for f in gpurun_out/${t}_scan_*.txt; do echo "== $f"; cut -c1-20,60-200 $f; done
