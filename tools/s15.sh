timeout 600 python bench.py > gpurun_out/s15_bench.json 2> gpurun_out/s15_bench.err; cat gpurun_out/s15_bench.json
for w in softmax colreduce bert stream; do timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/s15_$w.json 2>/dev/null; cat gpurun_out/s15_$w.json; done
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/s15_ref.json 2>/dev/null; cat gpurun_out/s15_ref.json
timeout 300 python tools/sweep_shapes.py --workload ln_gelu --reps 2 > gpurun_out/s15_sweep_ln.txt 2>&1; tail -3 gpurun_out/s15_sweep_ln.txt
