#!/bin/bash
# Round-2 late A/B session: tests on the main build, per-variant workload rates and grouped
# per-shape scans.  Usage: tools/r4_ab.sh <tag> "<variants>" "<workloads>" [tests]
#   variants: "main" = libdisc_b200.so, any other name = libdisc_b200_<name>.so
tag=$1; variants=$2; workloads=$3; tests=${4:-1}
mkdir -p gpurun_out
if [ "$tests" = 1 ]; then
  timeout 1100 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${tag}_tests.log 2>&1
  tail -2 gpurun_out/${tag}_tests.log
fi
for w in $workloads; do
  for v in $variants; do
    if [ "$v" = main ]; then unset DISC_LIB_VARIANT; else export DISC_LIB_VARIANT=$v; fi
    timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/${tag}_${w}_${v}.json 2>>gpurun_out/${tag}_err.log
    python - "$w" "$v" "gpurun_out/${tag}_${w}_${v}.json" <<'EOF'
import json, sys
try:
    j = json.load(open(sys.argv[3]))
    print(sys.argv[1], sys.argv[2], j["value"], j.get("large_shape_frac_of_peak"),
          {k: v["GB/s"] for k, v in list(j["kernel_breakdown"].items())[:6]})
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
EOF
  done
done
unset DISC_LIB_VARIANT
