#!/bin/bash
tag=$1
for f in gpurun_out/launches_${tag}_*.csv; do echo "== $f"; python tools/launches.py $f | grep -v fill_uniform; done
python - $tag <<'PY'
import json, sys, glob
tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/bench_{tag}*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "ERR", e); continue
    print(f.split("/")[-1], d["value"], "large", d["large_shape_GBps"], {k: v["GB/s"] for k, v in d["kernel_breakdown"].items()})
PY
