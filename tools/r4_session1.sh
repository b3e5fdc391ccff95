#!/bin/bash
# GPU session: tests on the main build, colreduce A/B of the column-pass changes, per-shape scans.
mkdir -p gpurun_out
bash tools/r4_ab.sh s2 "main nopipe off" "colreduce" 1
timeout 300 python tools/shape_scan.py colreduce "C=1,3,4,8,33,128,1024,4096" --copies-gb 2 > gpurun_out/s2_scan_col_main.txt 2>&1
DISC_LIB_VARIANT=off timeout 300 python tools/shape_scan.py colreduce "C=1,3,4,8,33,128,1024,4096" --copies-gb 2 > gpurun_out/s2_scan_col_off.txt 2>&1
timeout 400 python tools/shape_scan.py softmax "S1=2,3,5,7,9,13,16,17,24,31,33,64,100,255,1024,4096" --copies-gb 2 > gpurun_out/s2_scan_sm_main.txt 2>&1
for v in 8 16; do DISC_ROW_CPT=$v timeout 300 python tools/shape_scan.py softmax "S1=64,255,1024,4096" --copies-gb 2 > gpurun_out/s2_scan_sm_cpt$v.txt 2>&1; done
DISC_SUM_ROW_MB=1 timeout 300 python tools/shape_scan.py softmax "S1=64,255,1024,4096" --copies-gb 2 > gpurun_out/s2_scan_sm_smb.txt 2>&1
timeout 500 python bench.py > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err
python -c "import json; j=json.load(open('gpurun_out/s2_bench.json')); print(j['value'], j['large_shape_frac_of_peak'], j['roofline']['frac'], j['e2e']['value'])"
