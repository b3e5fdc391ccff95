"""Per-shape kernel rates of one pattern (each request alone, L2 flushed before it, inputs
in the bench's device arena, per-kernel device time from the executor's timing records).

  python tools/shape_scan.py softmax "S1=2,3,7,17,31,64,4096" [--bytes 256e6] [--reps 3]
  python tools/shape_scan.py colreduce "C=1,3,4,8,33,128,4096"

The other symbols are sized so each request moves ~--bytes of algorithmic bytes."""
import argparse
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def shapes(kind, var, vals, nbytes):
    out = []
    for v in vals:
        if kind == "softmax":
            out.append({"S0": max(1, int(nbytes / 12 / v)), "S1": v})
        elif kind == "colreduce":
            out.append({"C": v, "N": max(1, int(nbytes / 4 / v))})
        elif kind == "ln_gelu":
            out.append({"H": v, "T": max(1, int(nbytes / 28 / v))})
        elif kind == "bert":
            b = max(1, int(nbytes / (4 * (24 * v * v + 8 * 768 * v + 2 * 3072 * v))))
            out.append({"R": 12 * b * v, "S": v, "T": b * v, "H": 768, "F": 3072})
        else:
            raise SystemExit(kind)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind")
    ap.add_argument("values", help="VAR=v1,v2,...")
    ap.add_argument("--bytes", type=float, default=256e6)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--schedule", default="auto")
    ap.add_argument("--copies-gb", type=float, default=0.0,
                    help="run each shape as a grouped batch of copies totalling this many GB (grouped rates)")
    a = ap.parse_args()
    import paper_2103_05288_b200 as D
    D.lib()
    var, vals = a.values.split("=")
    vals = [int(x) for x in vals.split(",")]
    args = types.SimpleNamespace(schedule=a.schedule, host_threads=8, cache_gb=32.0, arena_gb=16.0, chunk_gb=32.0,
                                 reserve_gb=0, async_flush=0)
    wl = bench.make_workload("sweep", 0, 10)
    B = bench.Bench(D, args, 0, wl)
    for syms in shapes(a.kind, var, vals, a.bytes):
        reqs = [(a.kind, syms)]
        if a.copies_gb:
            one = B.costs(B.plans_for(reqs) and reqs)[0]
            reqs = reqs * max(1, int(a.copies_gb * 1e9 / max(one, 1)))
        batch = B.batch(reqs)
        B.record_pass(batch)
        best = None
        for _ in range(a.reps):
            recs = B.record_pass(batch)
            tot = sum(r["ms"] for r in recs)
            if best is None or tot < best[0]:
                best = (tot, recs)
        tot, recs = best
        ks = " ".join(f"k{r['kernel']}:{r['schedule'].replace('group:', '')}={r['bytes'] / r['ms'] / 1e6:.0f}"
                      for r in recs if r["ms"] > 0)
        print(f"{a.kind} {var}={syms.get(var)} x{len(reqs)} {syms}: {batch.bytes / 1e6:.0f} MB {tot * 1e3:.1f} us "
              f"{batch.bytes / tot / 1e6:.0f} GB/s  [{ks}]", flush=True)
    B.close()


if __name__ == "__main__":
    main()
