#!/bin/bash
# integer-pipe f32->f64 in the column pass: parity (special values, folded, generated) + rates
mkdir -p gpurun_out
t=s10
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "special or folded or generated or random_graphs or edge" > gpurun_out/${t}_tests.log 2>&1
tail -2 gpurun_out/${t}_tests.log
bash tools/r4_ab.sh $t "main" "colreduce" 0
timeout 300 python tools/shape_scan.py colreduce "C=1,3,4,8,33,128,1024,4096" --copies-gb 2 > gpurun_out/${t}_scan_col.txt 2>&1
cat gpurun_out/${t}_scan_col.txt
