#!/bin/bash
# Round-2 ncu evidence (run on the GPU box; outputs under gpurun_out/<tag>_*):
#   <tag>_launches.csv     launch list of the bench command (gpu__time_duration + DRAM bytes;
#                          cold, serialised: shares comparable with the bench, absolutes not)
#   <tag>_kt.csv/.json     per-key DRAM traffic of one bench step's timing-mode passes
#                          (tools/profile_kernels.py merge -> profiles/ncu_traffic.json)
#   <tag>_full_<p>.txt     --set full summaries of pattern p's grouped kernels
tag=$1
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
if [ -z "$SKIP_LAUNCHES" ]; then
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --verify off > gpurun_out/${tag}_launches.log 2>&1
echo "launch list rc=$?"
fi
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_kt.csv \
  python tools/profile_kernels.py run --records gpurun_out/${tag}_kt.json > gpurun_out/${tag}_kt.log 2>&1
echo "kernel traffic rc=$?"
python tools/profile_kernels.py merge --records gpurun_out/${tag}_kt.json --csv gpurun_out/${tag}_kt.csv \
  --out gpurun_out/${tag}_ncu_traffic.json > /dev/null 2>&1
for p in $2; do
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -c 10 -k "regex:k_(loop|row|col)" \
    -o /tmp/full_${tag}_$p python tools/profile_kernels.py run --patterns $p --records /tmp/rec_$p.json > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/full_${tag}_$p.ncu-rep dram__bytes_read.sum dram__bytes_write.sum \
    smsp__inst_executed.sum sm__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/${tag}_full_$p.txt 2>&1
  # (reports stay on the box: gpurun copies back at most 64 MiB)
done
ls -la gpurun_out | grep $tag
