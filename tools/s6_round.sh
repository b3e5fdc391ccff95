timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3
for wl in ln_gelu softmax colreduce bert; do echo "$wl"; timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['roofline']['achieved'], j['kernel_breakdown'])"; done
