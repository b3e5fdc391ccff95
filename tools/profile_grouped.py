"""Runs a workload's sweep as grouped launches (bench --mode grouped) a few times, for
ncu captures of the grouped kernels:

  ncu --set full -k regex:_g --launch-skip 3 -c 3 python tools/profile_grouped.py --workload ln_gelu
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
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import paper_2103_05288_b200 as D
    _, graphs, reqs = bench.workload(a.workload)
    plans = {k: D.compile_graph(g) for k, g in graphs.items()}
    rq = bench.Requests(D, graphs, plans, reqs)
    ex = D.Executor()
    for _ in range(a.reps):
        rq.run_grouped(ex)
    ex.synchronize()


if __name__ == "__main__":
    main()
