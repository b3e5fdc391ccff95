"""Summarise a round's ncu evidence into profiles/ (committed):

  profiles/<tag>_launches_bench.csv.gz   raw per-launch list of `python bench.py` under ncu
                                        (gpu__time_duration + dram bytes; cold, serialised)
  profiles/<tag>_launches_summary.txt    per kernel: launches, mean us, share of kernel
                                        time, mean DRAM bytes/launch, DRAM GB/s
  profiles/<tag>_full_<workload>.txt     key --set full metrics of each captured kernel
  profiles/ncu_summary.json             traffic_per_launch per schedule (bench.py reads it
                                        for roofline.traffic) + the shares above

  python tools/make_profiles.py r1
"""
import gzip
import json
import os
import re
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import launches  # noqa: E402
import ncu_summary  # noqa: E402

OUT = os.path.join(ROOT, "profiles")
SCRATCH = os.path.join(ROOT, "gpurun_out")


def schedule_of(name):
    """bench.py schedule label of a kernel name (roofline.kernel uses these)."""
    if "k_loop_g<4" in name:
        return "group:loop_v4"
    if "k_loop_g<" in name:
        return "group:loop"
    if "k_row_g<" in name:
        return "group:row_staged" if name.rstrip(")").split(",")[-1].strip().startswith("true") else "group:row"
    if "k_col_finalize_g" in name:
        return "group:col_finalize"
    if "k_col_g<" in name:
        return "group:col"
    if name.startswith("void disc_dev::k_loop<4") or name.startswith("void k_loop<4"):
        return "loop_v4"
    if "k_loop<" in name:
        return "loop"
    if "k_row<" in name:
        return "row_staged" if name.rstrip(")").split(",")[-1].strip().startswith("true") else "row"
    if "k_col_finalize" in name:
        return "col_finalize"
    if "k_col<" in name:
        return "col"
    return None


def short(name):
    name = re.sub(r"\(disc_[a-z_]+\)$", "", name)
    name = name.replace("void disc_dev::", "").replace("disc_gen::", "")
    return name[:110]


def main(tag):
    os.makedirs(OUT, exist_ok=True)
    src = os.path.join(SCRATCH, f"launches_bench_{tag}.csv")
    with open(src, "rb") as f, gzip.open(os.path.join(OUT, f"{tag}_launches_bench.csv.gz"), "wb") as g:
        shutil.copyfileobj(f, g)
    data = launches.load(src)
    per = defaultdict(lambda: [0, 0.0, 0.0])
    for (i, name), v in data.items():
        p = per[name]
        p[0] += 1
        p[1] += v.get("gpu__time_duration.sum", 0.0)
        p[2] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
    ours = {n: p for n, p in per.items() if "disc_dev" in n or n.startswith("void k_") or "k_col_finalize" in n}
    total_ns = sum(p[1] for p in ours.values())
    lines = [f"# {tag}: ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e`",
             "# (--metrics gpu__time_duration.sum,dram__bytes_{read,write}.sum --clock-control none; cold-cache,",
             "#  serialised launches: shares are comparable with the bench, absolute times are not)",
             f"# {sum(p[0] for p in per.values())} launches, {sum(p[0] for p in ours.values())} of them disc kernels",
             f"{'launches':>8s} {'mean_us':>9s} {'share':>6s} {'dramMB/l':>9s} {'dramGB/s':>9s}  kernel"]
    traffic = defaultdict(lambda: [0.0, 0])
    for n, (cnt, ns, b) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{cnt:8d} {ns / cnt / 1e3:9.2f} {ns / total_ns:6.3f} {b / cnt / 1e6:9.2f} {b / max(ns, 1):9.1f}  {short(n)}")
        s = schedule_of(n)
        if s:
            traffic[s][0] += b
            traffic[s][1] += cnt
    others = {n: p for n, p in per.items() if n not in ours}
    lines.append("# not ours (input fill / L2 flush / spin): " + ", ".join(f"{short(n)} x{p[0]}" for n, p in others.items()))
    with open(os.path.join(OUT, f"{tag}_launches_summary.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")

    fulls = {}
    for fn in sorted(os.listdir(SCRATCH)):
        m = re.match(rf"full_{tag}_(\w+)\.(ncu-rep|txt)$", fn)
        if not m or (m.group(2) == "ncu-rep" and os.path.exists(os.path.join(SCRATCH, f"full_{tag}_{m.group(1)}.txt"))):
            continue
        if m.group(2) == "txt":  # summarised on the GPU box (tools/profile_round.sh)
            text = open(os.path.join(SCRATCH, fn)).read()
        else:
            text = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"),
                                   os.path.join(SCRATCH, fn), "dram__bytes_read.sum", "dram__bytes_write.sum",
                                   "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"],
                                  capture_output=True, text=True).stdout
        with open(os.path.join(OUT, f"{tag}_full_{m.group(1)}.txt"), "w") as f:
            f.write(f"# {tag}: ncu --set full --import-source on --clock-control none of the grouped kernels of one "
                    f"pass of the {m.group(1)} sweep (tools/profile_grouped.py, see tools/profile_round.sh)\n" + text)
        fulls[m.group(1)] = fn
    summary = {"round": tag,
               "traffic_per_launch": {s: round(b / n) for s, (b, n) in traffic.items()},
               "traffic_source": f"profiles/{tag}_launches_bench.csv.gz: mean dram__bytes_read.sum + "
                                 "dram__bytes_write.sum per launch over the bench command's launches",
               "share_of_kernel_time": {short(n): round(p[1] / total_ns, 4)
                                        for n, p in sorted(ours.items(), key=lambda kv: -kv[1][1])[:12]},
               "full_captures": fulls}
    with open(os.path.join(OUT, "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print("\n".join(lines[:20]))
    print(json.dumps(summary["traffic_per_launch"]))


if __name__ == "__main__":
    main(sys.argv[1])
