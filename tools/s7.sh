timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3
for r in 1 2; do for wl in softmax bert ln_gelu; do for a in 0 1; do
DISC_ARG_CACHE=$a timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read())
print('arg=$a', '$wl', j['value'], {k: v['GB/s'] for k, v in j['kernel_breakdown'].items()})"
done; done; done
