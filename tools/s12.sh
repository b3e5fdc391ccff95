timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/s12_bench.json 2> gpurun_out/s12_bench.err; cat gpurun_out/s12_bench.json
bash tools/profile_round.sh r1b
