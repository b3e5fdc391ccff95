"""Pipe utilisation and warp-stall breakdown of every kernel in an ncu --set full report:
python tools/ncu_pipes.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for r in rows[2:]:
        print("==", r[hdr.index("Kernel Name")][:90] if "Kernel Name" in hdr else "")
        for m, v in zip(hdr, r):
            if (("pipe" in m and "pct_of_peak_sustained_active" in m and "inst_executed" in m) or
                    ("warp_latency_issue_stalled" in m and m.endswith(".ratio")) or
                    m in ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
                          "smsp__issue_active.avg.pct_of_peak_sustained_active", "gpu__time_duration.sum",
                          "launch__registers_per_thread", "smsp__inst_executed.sum")):
                try:
                    if float(v.replace(",", "")) < 0.05:
                        continue
                except ValueError:
                    pass
                print(f"   {m:90s} {v}")


if __name__ == "__main__":
    main(sys.argv[1])
