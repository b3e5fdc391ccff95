set -x
timeout 600 python -m pytest tests/test_gpu_grouped.py -q -x --timeout 500 > gpurun_out/s3_tests.log 2>&1; tail -30 gpurun_out/s3_tests.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; cat gpurun_out/s3_bench.json; tail -5 gpurun_out/s3_bench.err
for w in softmax colreduce bert stream; do timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3_bench_$w.json 2>>gpurun_out/s3_w.err; cat gpurun_out/s3_bench_$w.json; done
tail -5 gpurun_out/s3_w.err
