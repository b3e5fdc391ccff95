timeout 600 ncu --section SpeedOfLight --section Occupancy --section LaunchStats --section WarpStateStats --section SourceCounters --import-source on --clock-control none -k "regex:k_row_g" -c 6 -o /tmp/bert_rows python tools/profile_grouped.py --workload bert --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/bert_rows.ncu-rep > gpurun_out/s22_bert_rows.txt 2>&1
ncu -i /tmp/bert_rows.ncu-rep --page source --csv --print-source sass --kernel-name regex:Pre_row_fff --launch-count 1 > /dev/null 2>&1
python - <<'PY' > gpurun_out/s22_hot.txt 2>&1
import csv, subprocess, io
rep = "/tmp/bert_rows.ncu-rep"
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = {n: i for i, n in enumerate(rows[0])}
dur = {}
for r in rows[1:]:
    if r[h["Metric Name"]] == "Duration":
        dur[r[h["ID"]]] = (float(r[h["Metric Value"]].replace(",", "")), r[h["Metric Unit"]], r[h["Kernel Name"]][:90])
print(dur)
# longest kernel id
kid = max(dur, key=lambda k: dur[k][0] * (1000 if dur[k][1] == "ms" else 1))
print("longest", kid, dur[kid])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", kid, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][-1]
hh = rows[hi]; data = rows[hi + 1:]
ie = hh.index("Instructions Executed"); sc = hh.index("Source"); sm = hh.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ie] or 0) for r in data); ts = sum(int(r[sm] or 0) for r in data)
print("warp inst", tot, "samples", ts)
for r in sorted(data, key=lambda r: -int(r[sm] or 0))[:25]:
    print(r[ie], r[sm], r[sc][:90])
PY
cat gpurun_out/s22_hot.txt | head -40
