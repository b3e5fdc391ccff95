#!/bin/bash
# one tanh vote per tile (un_tile) vs per float4: rates + parity subset
mkdir -p gpurun_out
t=s15
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_grouped.py -q -x > gpurun_out/${t}_tests.log 2>&1; tail -1 gpurun_out/${t}_tests.log
bash tools/r4_ab.sh $t "main" "colreduce ln_gelu bert" 0
timeout 600 python bench.py --no-cpu-baseline --no-e2e --verify off > gpurun_out/${t}_sweep.json 2>> gpurun_out/${t}_err.log
python -c "import json; j=json.load(open('gpurun_out/${t}_sweep.json')); print('sweep', j['value'], j['large_shape_frac_of_peak'])"
