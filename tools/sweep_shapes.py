"""Per-shape breakdown of a bench sweep: each request run alone (L2 flushed before it),
device time per kernel from the executor's launch records.

  python tools/sweep_shapes.py --workload ln_gelu [--reps 3] [--json out.json]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="ln_gelu")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--schedule", default="auto")
    ap.add_argument("--json", default=None)
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--request", action="store_true",
                    help="time whole requests (events around the run, PDL overlap intact) instead of per kernel")
    a = ap.parse_args()
    import paper_2103_05288_b200 as D
    L = D.lib()
    _, graph, shapes = bench.workload_single(a.workload)
    D.set_pdl(a.pdl)
    plan = D.compile_graph(graph)
    evs = [C.c_void_p(), C.c_void_p()]
    for e in evs:
        D.api._cuda(L.disc_cuda_event_create(C.byref(e)))
    stream = C.c_void_p()
    D.api._cuda(L.disc_cuda_stream_create(C.byref(stream)))
    ex = D.Executor(0, stream.value)
    ex.set_schedule(a.schedule)
    flush_bytes = 1 << 30
    flush = C.c_void_p()
    D.api._cuda(L.disc_cuda_malloc(flush_bytes, stream, C.byref(flush)))
    rows = []
    tot_b = tot_ms = 0.0
    for syms in shapes:
        reqs = bench.Requests(D, {"g": graph}, {"g": plan}, [("g", syms)])
        reqs.run(ex)  # warm
        ex.synchronize()
        if a.request:
            tot = 0.0
            for _ in range(a.reps):
                L.disc_cuda_flush_l2(flush, flush_bytes, stream)
                L.disc_cuda_spin(2000, stream)
                L.disc_cuda_event_record(evs[0], stream)
                reqs.run(ex)
                L.disc_cuda_event_record(evs[1], stream)
                ex.synchronize()
                ms = C.c_float()
                L.disc_cuda_event_elapsed_ms(evs[0], evs[1], C.byref(ms))
                tot += ms.value / a.reps
            b = ex.algorithmic_bytes()
            tot_b += b
            tot_ms += tot
            rows.append({"shape": {k: v for k, v in syms.items() if not k.startswith("_")}, "bytes": int(b),
                         "us": round(tot * 1e3, 2), "GBps": round(b / tot / 1e6, 1)})
            print(f"{str(rows[-1]['shape']):34s} {b / 1e6:9.2f}MB {tot * 1e3:9.2f}us {rows[-1]['GBps']:8.1f} GB/s", flush=True)
            del reqs
            continue
        ex.set_timing(True)
        per = {}
        for _ in range(a.reps):
            L.disc_cuda_flush_l2(flush, flush_bytes, stream)
            L.disc_cuda_spin(2000, stream)  # queue the request: events time the device only
            reqs.run(ex)
            ex.synchronize()
            for r in ex.launch_records():
                k = f"k{r['kernel']}:{r['schedule']}"
                p = per.setdefault(k, [0, 0.0])
                p[0] += r["bytes"] / a.reps
                p[1] += r["ms"] / a.reps
        ex.set_timing(False)
        b = sum(v[0] for v in per.values())
        ms = sum(v[1] for v in per.values())
        tot_b += b
        tot_ms += ms
        rows.append({"shape": {k: v for k, v in syms.items() if not k.startswith("_")}, "bytes": int(b),
                     "us": round(ms * 1e3, 2), "GBps": round(b / ms / 1e6, 1) if ms else None,
                     "kernels": {k: [round(v[1] * 1e3, 2), round(v[0] / v[1] / 1e6, 1) if v[1] else None]
                                 for k, v in per.items()}})
        print(f"{str(rows[-1]['shape']):34s} {b / 1e6:9.2f}MB {ms * 1e3:9.2f}us {rows[-1]['GBps']:8.1f} GB/s  "
              + " ".join(f"{k}={v[0]}us/{v[1]}" for k, v in rows[-1]["kernels"].items()), flush=True)
        del reqs
    print(f"aggregate {tot_b / tot_ms / 1e6:.1f} GB/s over {len(rows)} shapes (kernel time only)")
    if a.json:
        json.dump(rows, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
