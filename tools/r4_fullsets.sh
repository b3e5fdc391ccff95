#!/bin/bash
# ncu --set full of the grouped kernels of each workload (tools/profile_round.sh's second half)
mkdir -p gpurun_out
tag=r4g
for w in ln_gelu softmax colreduce bert; do
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_(loop|row|col|col_finalize|row_short)_g" -c 8 \
    -o /tmp/full_${tag}_$w python tools/profile_grouped.py --workload $w --reps 1 > gpurun_out/full_${tag}_$w.log 2>&1
  python tools/ncu_summary.py /tmp/full_${tag}_$w.ncu-rep dram__bytes_read.sum dram__bytes_write.sum \
    smsp__inst_executed.sum sm__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/full_${tag}_$w.txt 2>&1
  python tools/ncu_pipes.py /tmp/full_${tag}_$w.ncu-rep > gpurun_out/pipes_${tag}_$w.txt 2>&1
done
ls -la gpurun_out | grep ${tag}_
