"""Runs one large request of a workload a few times (for ncu captures of single kernels).

  python tools/profile_one.py --workload ln_gelu --shape T=16384,H=4096 --reps 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="ln_gelu")
    ap.add_argument("--shape", default="T=16384,H=4096")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--schedule", default="auto")
    a = ap.parse_args()
    import types
    import paper_2103_05288_b200 as D
    D.lib()
    syms = {k: int(v) for k, v in (kv.split("=") for kv in a.shape.split(","))}
    args = types.SimpleNamespace(schedule=a.schedule, host_threads=8, cache_gb=32.0, arena_gb=16.0, chunk_gb=32.0,
                                 reserve_gb=0, async_flush=0)
    B = bench.Bench(D, args, 0, bench.make_workload("sweep", 0, 10))
    batch = B.batch([(a.workload, syms)])
    for _ in range(a.reps):
        recs = B.record_pass(batch)
    print("records", recs)
    B.close()


if __name__ == "__main__":
    main()
