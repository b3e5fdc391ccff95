"""ncu DRAM traffic per bench kernel key -> profiles/ncu_traffic.json (bench.py's
roofline.traffic).

For every pattern of one bench step (the first timed step, the same request list bench.py
times), the pattern's requests run as ONE grouped pass in timing mode -- exactly the
analysis pass bench.py derives its kernel breakdown from (one flush phase, records per
grouped launch) -- inside a profiler range, so ncu sees only those launches.  ncu's
per-launch rows are matched to the executor's records in issue order (a column two-pass
record owns its finalize kernel), giving DRAM bytes and duration per key
"<pattern>:k<artifact>:<schedule>" next to the algorithmic bytes.

  # on the GPU box:
  ncu --profile-from-start off --clock-control none --metrics \\
      gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \\
      --log-file gpurun_out/kt.csv python tools/profile_kernels.py run --records gpurun_out/kt.json
  python tools/profile_kernels.py merge --records gpurun_out/kt.json --csv gpurun_out/kt.csv \\
      --out profiles/ncu_traffic.json
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KERNEL_PREFIXES = ("k_loop", "k_row", "k_col", "k_copy2d", "k_pad", "k_concat", "k_reduce_generic", "k_gemm")


def run(args):
    import bench
    import paper_2103_05288_b200 as D
    D.lib()
    a = types.SimpleNamespace(schedule="auto", host_threads=min(16, os.cpu_count() or 1), cache_gb=32.0,
                              arena_gb=48.0, chunk_gb=128.0, reserve_gb=120.0)
    wl = bench.make_workload(args.workload, 0, args.requests)
    B = bench.Bench(D, a, 0, wl)
    reqs = wl.requests(args.step)
    B.plans_for(reqs)
    costs = B.costs(reqs)
    pats = {}  # per graph (bench.py's kernel_breakdown keys)
    for i, (k, _) in enumerate(reqs):
        pats.setdefault(k, []).append(i)
    out = []
    only = set(args.patterns.split(",")) if args.patterns else None
    for p, idx in sorted(pats.items()):
        if only and p not in only and bench.pattern_of(p) not in only:
            continue
        batch = B.batch([reqs[i] for i in idx], [costs[i] for i in idx])
        B.record_pass(batch)  # warm (recipes, arena)
        B.L.disc_cuda_stream_synchronize(B.stream)
        B.L.disc_cuda_profiler(1)
        recs = B.record_pass(batch)
        B.L.disc_cuda_stream_synchronize(B.stream)
        B.L.disc_cuda_profiler(0)
        out.append({"pattern": p, "records": [{"key": f"{p}:k{r['kernel']}:{r['schedule']}", "bytes": r["bytes"],
                                                "ms": r["ms"], "schedule": r["schedule"]} for r in recs]})
    json.dump({"workload": wl.name, "step": args.step, "passes": out}, open(args.records, "w"))
    B.close()


def ncu_rows(path):
    text = open(path).read()
    i = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[i:])))
    h = {n: k for k, n in enumerate(rows[0])}
    launches = {}
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        lid = int(r[h["ID"]])
        ent = launches.setdefault(lid, {"name": r[h["Kernel Name"]], "m": {}})
        v = r[h["Metric Value"]].replace(",", "")
        unit = r[h["Metric Unit"]]
        x = float(v)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
                 "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(unit, 1)
        ent["m"][r[h["Metric Name"]]] = x * scale
    return [launches[k] for k in sorted(launches)]


def base(name):
    """k_loop_g from 'void disc_dev::k_loop_g<4, ...>(...)'."""
    n = name.split("(")[0].split("<")[0].strip()
    return n.split()[-1].split("::")[-1] if n else n


def merge(args):
    rec = json.load(open(args.records))
    rows = [r for r in ncu_rows(args.csv) if base(r["name"]).startswith(KERNEL_PREFIXES)
            and not base(r["name"]).startswith("k_col_finalize") or base(r["name"]).startswith("k_col_finalize")]
    def kinds(sched):
        """ncu kernel base names a record's grouped launch can have."""
        s = sched.replace("group:", "")
        if s == "mixed" or "fold" in s:  # a folded column launch issues its tile loop first
            return ("k_row_g", "k_row_g_mb", "k_row_g_smb", "k_row_short_g", "k_col_g", "k_loop_g")
        if s.startswith("col"):
            return ("k_col_g",)
        if s.startswith("row1_loop") or s.startswith("loop"):
            return ("k_loop_g",)
        if s.startswith("row"):
            return ("k_row_g", "k_row_g_mb", "k_row_g_smb", "k_row_short_g")
        if s.startswith("copy"):
            return ("k_copy2d_g",)
        return ()
    k = 0
    agg = {}
    unmatched = 0
    for ps in rec["passes"]:
        for r in ps["records"]:
            if k >= len(rows) or base(rows[k]["name"]) not in kinds(r["schedule"]):
                unmatched += 1  # no kernel for this record (all members empty) or unknown kind
                continue
            m = rows[k]["m"]
            dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
            us = m.get("gpu__time_duration.sum", 0)
            k += 1
            while k < len(rows) and base(rows[k]["name"]).startswith("k_col_finalize"):
                m = rows[k]["m"]
                dram += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
                us += m.get("gpu__time_duration.sum", 0)
                k += 1
            a = agg.setdefault(r["key"], {"launches": 0, "dram": 0.0, "alg": 0, "us": 0.0})
            a["launches"] += 1
            a["dram"] += dram
            a["alg"] += r["bytes"]
            a["us"] += us
    if k != len(rows):
        raise SystemExit(f"{len(rows) - k} ncu rows left unmatched")
    print(f"{unmatched} records without a kernel", file=sys.stderr)
    out = json.load(open(args.out)) if os.path.exists(args.out) else {}
    w = {}
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        n = a["launches"]
        w[k] = {"launches": n, "dram_bytes_per_launch": int(a["dram"] / n), "alg_bytes_per_launch": int(a["alg"] / n),
                "dram_over_alg": round(a["dram"] / max(1, a["alg"]), 4), "ncu_us_per_launch": round(a["us"] / n, 2),
                "ncu_GBps": round(a["alg"] / max(a["us"], 1e-9) / 1e3, 1)}
    out[rec["workload"]] = w
    out["_source"] = ("tools/profile_kernels.py: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                      "dram__bytes_write.sum --clock-control none over the timing-mode grouped pass of every "
                      "pattern of bench step %d" % rec["step"])
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps(w, indent=1)[:3000])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["run", "merge"])
    ap.add_argument("--workload", default="sweep")
    ap.add_argument("--requests", type=int, default=10000)
    ap.add_argument("--step", type=int, default=3)
    ap.add_argument("--records", required=True)
    ap.add_argument("--csv")
    ap.add_argument("--patterns", default="", help="run: only these patterns (comma-separated)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_traffic.json"))
    args = ap.parse_args()
    run(args) if args.mode == "run" else merge(args)


if __name__ == "__main__":
    main()
