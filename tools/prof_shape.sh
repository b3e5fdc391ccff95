#!/bin/bash
# ncu source-level hot spots of one workload shape's kernels (single request):
#   tools/prof_shape.sh <workload> <shape> <kernel regex> <out>
w=$1; shape=$2; re=$3; out=$4
timeout 600 ncu --section SpeedOfLight --section Occupancy --section LaunchStats --section WarpStateStats --section SourceCounters --import-source on --clock-control none -f -k "regex:$re" -c 2 -o /tmp/ps python tools/profile_one.py --workload $w --shape $shape --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ps.ncu-rep > gpurun_out/${out}_summary.txt 2>&1
python - <<PY > gpurun_out/${out}_hot.txt 2>&1
import csv, subprocess, io
rep = "/tmp/ps.ncu-rep"
for kid in ("0", "1"):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", kid, "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    his = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    if not his: continue
    hi = his[-1]; hh = rows[hi]; data = rows[hi + 1:]
    ie = hh.index("Instructions Executed"); sc = hh.index("Source"); sm = hh.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[ie] or 0) for r in data); ts = sum(int(r[sm] or 0) for r in data)
    print("kernel", kid, rows[0][:1], "warp inst", tot, "samples", ts)
    for r in sorted(data, key=lambda r: -int(r[sm] or 0))[:14]:
        print("  ", r[ie], r[sm], r[sc][:80])
PY
