timeout 600 python -m pytest tests/test_gpu_grouped.py -q -x 2>&1 | tail -2
for c in 256 1024 4096; do for p in 2 3 4; do echo "chunk $c pipes $p"; timeout 300 python bench.py --steps 3 --no-cpu-baseline --e2e-chunk-mb $c --e2e-pipes $p 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['e2e'])"; done; done
