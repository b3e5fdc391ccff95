#!/bin/bash
# ncu --set full of one shape's grouped kernels (tools/shape_scan.py, a few copies):
#   tools/prof_shape2.sh <tag> <kind> <VAR=value> [copies_gb]
tag=$1; kind=$2; val=$3; gb=${4:-1}
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_(row|col|loop)" -c 6 \
  -o /tmp/ps_${tag} python tools/shape_scan.py $kind "$val" --copies-gb $gb --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ps_${tag}.ncu-rep dram__bytes_read.sum dram__bytes_write.sum smsp__inst_executed.sum \
  > gpurun_out/ps_${tag}.txt 2>&1
ncu -i /tmp/ps_${tag}.ncu-rep --page details --csv --section WarpStateStats --section SchedulerStats \
  > gpurun_out/ps_${tag}_stalls.csv 2>/dev/null
