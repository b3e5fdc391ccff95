#!/bin/bash
# ncu evidence for profiles/: the per-launch list of the bench command (duration + DRAM
# bytes; a run under ncu is never a bench value) and --set full captures of the grouped
# kernels of one pass of each workload's sweep, summarised on the box (the reports stay
# there; only the ln_gelu report comes back).  Usage: tools/profile_round.sh <tag>
tag=$1
mkdir -p gpurun_out
# (one flush phase, as in the bench's per-kernel timing pass: traffic per launch matches roofline.bytes_per_launch)
DISC_GROUP_PHASES=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_bench_$tag.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_bench_$tag.log 2>&1
for w in ln_gelu softmax colreduce bert; do
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_(loop|row|col|col_finalize)_g" -c 8 \
    -o /tmp/full_${tag}_$w python tools/profile_grouped.py --workload $w --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/full_${tag}_$w.ncu-rep dram__bytes_read.sum dram__bytes_write.sum \
    smsp__inst_executed.sum sm__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/full_${tag}_$w.txt 2>&1
done
cp /tmp/full_${tag}_ln_gelu.ncu-rep gpurun_out/
ls -la gpurun_out | grep $tag
