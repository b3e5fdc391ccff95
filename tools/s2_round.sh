set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/s2_tests.log 2>&1; tail -3 gpurun_out/s2_tests.log
timeout 600 python bench.py > gpurun_out/s2_bench_default.json 2> gpurun_out/s2_bench_default.err; cat gpurun_out/s2_bench_default.json
timeout 300 python bench.py --streams 1 --no-cpu-baseline --no-e2e > gpurun_out/s2_bench_s1.json 2>/dev/null; cat gpurun_out/s2_bench_s1.json
for w in softmax colreduce bert stream; do timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s2_bench_$w.json 2>>gpurun_out/s2_w.err; cat gpurun_out/s2_bench_$w.json; done
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/s2_ref.json 2>gpurun_out/s2_ref.err; cat gpurun_out/s2_ref.json
python -c "import __graft_entry__ as g; g.smoke()"
