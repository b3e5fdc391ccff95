#!/bin/bash
# One GPU round: gpu tests, bench lines for all workloads, per-launch ncu lists and an
# ncu --set full capture.  Usage: tools/gpu_round.sh <tag> [ncu_workload ncu_shape ncu_regex]
tag=$1
ncu_w=$2; ncu_shape=$3; ncu_re=$4; ncu_n=${5:-2}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x --timeout 500 > gpurun_out/tests_$tag.log 2>&1; tail -3 gpurun_out/tests_$tag.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
for w in softmax colreduce bert; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${tag}_$w.json 2>>gpurun_out/bench_$tag.err
done
for spec in "ln_gelu T=16384,H=4096" "softmax S0=16384,S1=4096" "colreduce N=65536,C=4096" "bert R=49152,S=128,T=4096,H=768,F=3072"; do
  set -- $spec
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${tag}_$1.csv python tools/profile_one.py --workload $1 --shape $2 --reps 2 > /dev/null 2>&1
done
if [ -n "$ncu_re" ]; then
  timeout 400 ncu --set full --import-source on --clock-control none -k "regex:$ncu_re" -c $ncu_n -o gpurun_out/prof_$tag \
    python tools/profile_one.py --workload $ncu_w --shape $ncu_shape --reps 1 > /dev/null 2>&1
fi
tail -2 gpurun_out/bench_$tag.err
