#!/bin/bash
# GPU session: warp-vote tanh on every workload, the headline sweep (full default bench
# line), tests.
mkdir -p gpurun_out
t=s6
bash tools/r4_ab.sh $t "main" "colreduce ln_gelu bert softmax" 0
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${t}_tests.log 2>&1
tail -2 gpurun_out/${t}_tests.log
timeout 600 python bench.py > gpurun_out/${t}_bench.json 2> gpurun_out/${t}_bench.err
python -c "import json; j=json.load(open('gpurun_out/${t}_bench.json')); print('sweep', j['value'], j['large_shape_frac_of_peak'], j['roofline']['frac'], j['e2e']['value'])"
