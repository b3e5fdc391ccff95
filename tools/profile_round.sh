#!/bin/bash
# ncu evidence for profiles/: the per-launch list of the bench command (duration + DRAM
# bytes; a run under ncu is never a bench value) and --set full captures of each
# workload's top kernels at a large sweep shape.  Usage: tools/profile_round.sh <tag>
tag=$1
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_bench_$tag.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_bench_$tag.log 2>&1
for spec in "ln_gelu T=6444,H=4096 k_loop|k_row 3" "softmax S0=65536,S1=1024 k_row 2" \
            "colreduce N=262144,C=1024 k_col 2" "bert R=98304,S=256,T=8192,H=768,F=3072 k_row|k_loop 6"; do
  set -- $spec
  timeout 400 ncu --set full --import-source on --clock-control none -k "regex:$3" -c $4 \
    -o gpurun_out/full_${tag}_$1 python tools/profile_one.py --workload $1 --shape $2 --reps 1 > /dev/null 2>&1
done
ls -la gpurun_out | grep $tag
