timeout 600 python -m pytest tests/test_gpu_grouped.py -q -x 2>&1 | tail -2
for t in 1 4 8 16; do DISC_HOST_PROFILE=1 timeout 300 python bench.py --workload stream --host-threads $t --no-cpu-baseline --no-e2e > gpurun_out/s18_$t.json 2> gpurun_out/s18_$t.err; echo "threads $t: $(grep 'disc host' gpurun_out/s18_$t.err | tail -1)"; python -c "import json; j=json.load(open('gpurun_out/s18_$t.json')); print(j['value'], j['host_bound_frac'], j['device_ms_per_step'], j['ms_per_step'])"; done
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C2', j['value'], j['config']['host_threads'])"
nproc
