#!/bin/bash
# Round-end validation of the committed tree: GPU tests, smoke, the driver's bench command.
mkdir -p gpurun_out
t=r4v
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${t}_tests.log 2>&1; tail -2 gpurun_out/${t}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${t}_smoke.log 2>&1; tail -1 gpurun_out/${t}_smoke.log
timeout 900 python bench.py > gpurun_out/${t}_bench.json 2> gpurun_out/${t}_bench.err
python -c "import json; j=json.load(open('gpurun_out/${t}_bench.json')); print('bench', j['value'], j['large_shape_frac_of_peak'], j['roofline']['frac'], j['e2e']['value'], j['gpu_launches'], j['verify']['pass'] if isinstance(j['verify'], dict) else j['verify'])"
