#!/bin/bash
mkdir -p gpurun_out
t=r4b
timeout 900 python bench.py > gpurun_out/${t}_bench.json 2> gpurun_out/${t}_bench.err
python -c "import json; j=json.load(open('gpurun_out/${t}_bench.json')); print('bench', j['value'], j['ms_per_step'], j['large_shape_frac_of_peak'], j['roofline'], j['e2e'], j['cpu_baseline']['value'], j['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${t}_ref.json 2>> gpurun_out/${t}_bench.err
python -c "import json; j=json.load(open('gpurun_out/${t}_ref.json')); print('ref', j['value'])"
