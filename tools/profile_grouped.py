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
    import types
    import paper_2103_05288_b200 as D
    D.lib()
    args = types.SimpleNamespace(schedule="auto", host_threads=8, cache_gb=32.0, arena_gb=16.0, chunk_gb=128.0,
                                 reserve_gb=0, async_flush=0)
    wl = bench.make_workload(a.workload, 0, 10000)
    B = bench.Bench(D, args, 0, wl)
    batch = B.batch(wl.requests(0))
    for _ in range(a.reps):
        batch.run(B.ex)
    B.close()


if __name__ == "__main__":
    main()
