#!/bin/bash
# GPU session: warp-staged short rows (A/B vs DISC_WARP_STAGE_MAX=2), column-pass register
# budget variants, tests, headline bench.
mkdir -p gpurun_out
t=s3
S="S1=2,3,5,7,9,13,16,17,24,31"
timeout 300 python tools/shape_scan.py softmax "$S" --copies-gb 2 > gpurun_out/${t}_scan_sm_ws.txt 2>&1
DISC_WARP_STAGE_MAX=2 timeout 300 python tools/shape_scan.py softmax "$S" --copies-gb 2 > gpurun_out/${t}_scan_sm_nows.txt 2>&1
timeout 200 python tools/shape_scan.py bert "S=8,16,24,32" --copies-gb 2 > gpurun_out/${t}_scan_bert_ws.txt 2>&1
DISC_WARP_STAGE_MAX=2 timeout 200 python tools/shape_scan.py bert "S=8,16,24,32" --copies-gb 2 > gpurun_out/${t}_scan_bert_nows.txt 2>&1
bash tools/r4_ab.sh $t "main col3" "colreduce" 0
bash tools/r4_ab.sh $t "main" "softmax" 0
DISC_WARP_STAGE_MAX=2 bash tools/r4_ab.sh ${t}nows "main" "softmax" 0
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${t}_tests.log 2>&1
tail -2 gpurun_out/${t}_tests.log
timeout 500 python bench.py > gpurun_out/${t}_bench.json 2> gpurun_out/${t}_bench.err
python -c "import json; j=json.load(open('gpurun_out/${t}_bench.json')); print(j['value'], j['large_shape_frac_of_peak'], j['roofline']['frac'], j['e2e']['value'])"
