#!/bin/bash
# unaligned thread-per-row head/tail as scalar tiles: parity + odd-width rates + sweep
mkdir -p gpurun_out
t=s17
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grouped.py tests/test_gpu_fullsize.py -q -x > gpurun_out/${t}_tests.log 2>&1; tail -1 gpurun_out/${t}_tests.log
timeout 300 python tools/shape_scan.py softmax "S1=17,31,33,65,100,255,1025" --copies-gb 2 > gpurun_out/${t}_scan.txt 2>&1
cut -c1-16,60-200 gpurun_out/${t}_scan.txt
bash tools/r4_ab.sh $t "main" "softmax bert" 0
timeout 600 python bench.py --no-cpu-baseline --no-e2e --verify off > gpurun_out/${t}_sweep.json 2>> gpurun_out/${t}_err.log
python -c "import json; j=json.load(open('gpurun_out/${t}_sweep.json')); print('sweep', j['value'], j['large_shape_frac_of_peak'])"
