timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
tools/ab.sh "base s1" "softmax" 2
timeout 600 python tools/sweep_shapes.py --workload softmax --reps 2 2>&1 | tail -23
