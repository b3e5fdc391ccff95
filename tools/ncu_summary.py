"""Key metrics of each kernel in an ncu report: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block", "Block Limit Registers",
        "Block Limit Shared Mem", "Active Warps Per Scheduler")


def main(path, raw_metrics=()):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = {n: i for i, n in enumerate(rows[0])}
    cur = None
    for r in rows[1:]:
        k = (r[h["ID"]], r[h["Kernel Name"]][:70])
        if k != cur:
            cur = k
            print(f"== {k[0]} {k[1]}")
        if r[h["Metric Name"]] in KEEP:
            print(f"   {r[h['Metric Name']][:40]:40s} {r[h['Metric Value']]:>14s} {r[h['Metric Unit']]}")
    if raw_metrics:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr = rows[0]
        for r in rows[2:]:
            print({m: r[hdr.index(m)] for m in raw_metrics if m in hdr})


if __name__ == "__main__":
    main(sys.argv[1], tuple(sys.argv[2:]))
