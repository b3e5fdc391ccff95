#!/bin/bash
# Final evidence of the round: the driver's bench command and reference arm, smoke, the
# per-key ncu traffic (profiles/ncu_traffic.json) and the ncu launch list / full sets.
mkdir -p gpurun_out
t=r4g
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${t}_tests.log 2>&1; tail -2 gpurun_out/${t}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${t}_smoke.log 2>&1; tail -1 gpurun_out/${t}_smoke.log
timeout 900 python bench.py > gpurun_out/${t}_bench.json 2> gpurun_out/${t}_bench.err
python -c "import json; j=json.load(open('gpurun_out/${t}_bench.json')); print('bench', j['value'], j['ms_per_step'], j['large_shape_frac_of_peak'], j['roofline'], j['e2e']['value'], j['cpu_baseline']['value'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${t}_ref.json 2>> gpurun_out/${t}_bench.err
python -c "import json; j=json.load(open('gpurun_out/${t}_ref.json')); print('ref', j['value'], j.get('cpu_baseline'))"
timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/${t}_kt.csv python tools/profile_kernels.py run --records gpurun_out/${t}_kt.json > gpurun_out/${t}_kt.log 2>&1
python tools/profile_kernels.py merge --records gpurun_out/${t}_kt.json --csv gpurun_out/${t}_kt.csv --out gpurun_out/${t}_ncu_traffic.json >> gpurun_out/${t}_kt.log 2>&1
tail -3 gpurun_out/${t}_kt.log
bash tools/profile_round.sh $t > /dev/null 2>&1
ls gpurun_out | grep -c $t
