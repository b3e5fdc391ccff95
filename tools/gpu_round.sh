#!/bin/bash
# One GPU round: gpu tests + smoke, bench lines for every workload (default = the driver's
# headline command), the reference arm, and the ncu evidence (tools/profile_round.sh).
# Usage: tools/gpu_round.sh <tag>      (outputs under gpurun_out/<tag>_*)
tag=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${tag}_tests.log 2>&1; tail -2 gpurun_out/${tag}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
for w in softmax colreduce bert stream; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench_$w.json 2>>gpurun_out/${tag}_bench.err
done
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${tag}_ref.json 2>>gpurun_out/${tag}_bench.err
for f in gpurun_out/${tag}_bench*.json gpurun_out/${tag}_ref.json; do
  python -c "import json,sys; j=json.load(open('$f')); print('$f', j.get('value'), (j.get('e2e') or {}).get('value'), (j.get('roofline') or {}).get('frac'))"
done
bash tools/profile_round.sh $tag > /dev/null 2>&1
ls gpurun_out | grep -c $tag
