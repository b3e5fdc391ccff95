timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
DISC_HOST_PROFILE=1 timeout 300 python bench.py --workload stream --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/s14_stream.json 2> gpurun_out/s14_stream.err; grep "disc host" gpurun_out/s14_stream.err | tail -2; python -c "import json; j=json.load(open('gpurun_out/s14_stream.json')); print(j['value'], j['host_bound_frac'], j['device_ms_per_step'], j['ms_per_step'])"
DISC_HOST_PROFILE=1 timeout 300 python bench.py --no-cpu-baseline 2>&1 | grep "disc host" | tail -2
