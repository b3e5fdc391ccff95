timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3
tools/ab.sh "base ch4" "softmax bert" 2
for r in 0 1; do DISC_RCP_REDVAL=$r timeout 300 python bench.py --workload softmax --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('rcp=$r', j['value'], {k: v['GB/s'] for k, v in j['kernel_breakdown'].items()})"; done
