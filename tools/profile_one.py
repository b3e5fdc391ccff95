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
    import paper_2103_05288_b200 as D
    _, graph, _ = bench.workload_single(a.workload)
    syms = {k: int(v) for k, v in (kv.split("=") for kv in a.shape.split(","))}
    plan = D.compile_graph(graph)
    reqs = bench.Requests(D, {"g": graph}, {"g": plan}, [("g", syms)])
    ex = D.Executor()
    ex.set_schedule(a.schedule)
    for _ in range(a.reps):
        reqs.run(ex)
    ex.synchronize()
    print("records", ex.launch_records())


if __name__ == "__main__":
    main()
