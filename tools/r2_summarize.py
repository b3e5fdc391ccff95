"""Summarise a round-2 ncu launch list (tools/r2_profiles.sh <tag>_launches.csv) into
profiles/<tag>_launches_summary.txt: per kernel instantiation, launches, mean duration,
share of our kernels' time, DRAM bytes per launch and DRAM GB/s (input fill, L2 flush and
spin kernels listed separately: not ours).  Under ncu launches are serialised and caches
cold: compare shares with the bench, not absolute times.

  python tools/r2_summarize.py gpurun_out/r2o_launches.csv profiles/r2_launches_summary.txt "<command>"
"""
import collections
import csv
import gzip
import shutil
import sys

NOT_OURS = ("k_spin", "k_flush", "k_flush_read", "k_fill_uniform")


def load(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h = {n: k for k, n in enumerate(rows[i])}
    out = {}
    for r in rows[i + 1:]:
        if len(r) < len(h):
            continue
        d = out.setdefault(int(r[h["ID"]]), {"name": r[h["Kernel Name"]]})
        v = float(r[h["Metric Value"]].replace(",", ""))
        unit = r[h["Metric Unit"]]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "byte": 1, "Kbyte": 1e3,
              "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        d[r[h["Metric Name"]]] = v
    return out


def main(src, dst, cmd):
    L = load(src)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    other = collections.Counter()
    for d in L.values():
        name = d["name"].split("(")[0].replace("void ", "").replace("disc_dev::", "").replace("disc_gen::", "")
        base = name.split("<")[0]
        if base in NOT_OURS:
            other[base] += 1
            continue
        a = agg[name]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    with open(dst, "w") as f:
        f.write(f"# ncu launch list of `{cmd}`\n# (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                f"--clock-control none; cold-cache, serialised launches: shares are comparable with the bench, absolute "
                f"times are not)\n# {len(L)} launches, {sum(a[0] for a in agg.values())} of them disc kernels\n")
        f.write("launches   mean_us  share  dramMB/l  dramGB/s  kernel\n")
        for k, (n, us, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
            f.write(f"{n:8d} {us / n:9.2f} {us / tot:6.3f} {b / n / 1e6:9.2f} {b / max(us, 1e-9) / 1e3:9.1f}  {k[:110]}\n")
        f.write("# not ours (input fill / L2 flush / spin): " + ", ".join(f"{k} x{v}" for k, v in sorted(other.items())) + "\n")
    with open(src, "rb") as fi, gzip.open(dst.replace("_summary.txt", ".csv.gz"), "wb") as fo:
        shutil.copyfileobj(fi, fo)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --verify off")
