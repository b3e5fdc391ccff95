#!/bin/bash
# GPU session: rows-per-thread short rows (S=2..7), argument-only epilogue register cap
# (DISC_SUM_ROW_MB=3) on softmax and the headline sweep, tests.
mkdir -p gpurun_out
t=s4
timeout 300 python tools/shape_scan.py softmax "S1=2,3,5,7,64,1024,4096" --copies-gb 2 > gpurun_out/${t}_scan_sm.txt 2>&1
DISC_SUM_ROW_MB=3 timeout 300 python tools/shape_scan.py softmax "S1=33,64,100,255,1024,4096" --copies-gb 2 > gpurun_out/${t}_scan_sm_mb3.txt 2>&1
DISC_SUM_ROW_MB=3 timeout 300 python tools/shape_scan.py bert "S=8,32,128,512" --copies-gb 2 > gpurun_out/${t}_scan_bert_mb3.txt 2>&1
bash tools/r4_ab.sh $t "main" "softmax" 0
DISC_SUM_ROW_MB=3 bash tools/r4_ab.sh ${t}mb3 "main" "softmax bert" 0
for m in 0 3; do
  DISC_SUM_ROW_MB=$m timeout 500 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${t}_sweep_mb$m.json 2>> gpurun_out/${t}_err.log
  python -c "import json; j=json.load(open('gpurun_out/${t}_sweep_mb$m.json')); print('sweep mb$m', j['value'], j['large_shape_frac_of_peak'], j['roofline']['frac'])"
done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${t}_tests.log 2>&1
tail -2 gpurun_out/${t}_tests.log
