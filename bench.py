#!/usr/bin/env python
"""disc-b200 benchmark: fused-kernel HBM GB/s across a dynamic-shape sweep, 0 recompiles.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload ln_gelu|softmax|colreduce|bert|stream]
  python bench.py --impl reference ...     # the reference's own CPU executor, same metric

Workload (BASELINE.json configs[1]): one plan of the LN-like + bias +
tanh-GELU graph compiled ONCE and run over 192 distinct runtime shapes [T, H] (T
log-uniform 1..16384, 64 samples x H in {768, 1024, 4096}).  A step = one pass over the
sweep.  Bytes are the algorithmic boundary bytes of every fused launch (SURVEY §8d:
4 x (external inputs read + external outputs written), broadcast sources at source size).
``--workload stream`` is C5: >= 10k distinct (graph, shape) requests over C1-C4 and the
reference fixtures, one plan per graph, 0 recompiles.

  value    = bytes / device time of the K timed steps (CUDA events on the executor's
             stream, inputs resident in HBM, L2 flushed before each step)
  e2e      = same bytes / wall time through the public C ABI with host inputs: H2D of
             every request's inputs from pinned memory and D2H of its outputs inside
             the timed region
  roofline = the dominant kernel (largest share of device time): its bytes / its mean
             CUDA-event launch duration (measured in an untimed pass queued behind a spin
             kernel, so events see device execution), against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline = the reference executor (oracle/_ref, built from /root/reference) on a
             bounded sample of the same sweep, 1 host thread

Multi-GPU (torchrun, one process per GPU): the workload is N distinct sweeps (N x the
requests; C2 draws each replica with its own seed), sharded across ranks by the
dispatcher's deterministic LPT partition on algorithmic bytes (paper_2103_05288_b200/
dispatch.py) -- per-GPU work stays ~fixed (weak scaling) and no collective touches the
data path; the timed region is bracketed by barriers, the max over ranks is reported and
value = all ranks' bytes / that time.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused-kernel HBM GB/s (% of peak) across dynamic-shape sweep; 0 recompiles"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# Workloads: (description, {kind: graph}, [(kind, syms)])

def load_fixtures():
    """Reference fixture graphs for the C5 stream (GEMM fixtures excluded: library calls)."""
    fx = json.load(open(os.path.join(ROOT, "tests", "golden", "fixtures.json")))
    return {k: (json.loads(v["graph"]), v["bindings"]) for k, v in sorted(fx.items())
            if k not in ("matmul", "transformer")}


def workload(name, replica=0):
    from paper_2103_05288_b200 import workloads as W
    if name == "ln_gelu":
        g = W.ln_gelu_graph()
        return ("C2 LN-like+bias+tanh-GELU [T,H], T log-uniform 1..16384 x H {768,1024,4096}", {name: g},
                [(name, s) for s in W.ln_shapes(seed=20261017 + replica)])
    if name == "softmax":
        return ("C1 softmax [B,S], S 1..4096, B = 2^26/S", {name: W.softmax_graph_for(0)},
                [(name, {"S0": s["S0"], "S1": s["_S"]}) for s in W.softmax_shapes()])
    if name == "colreduce":
        return "C3 column reduce with prologue [N,C]", {name: W.colreduce_graph()}, \
            [(name, s) for s in W.colreduce_shapes()]
    if name == "bert":
        return "C4 BERT-base non-GEMM subgraphs, S 8..512, B {1,8,32}", {name: W.bert_graph()}, \
            [(name, s) for s in W.bert_shapes()]
    if name == "stream":
        graphs, reqs = W.mixed_stream(10000, seed=20261017 + replica, fixtures=load_fixtures())
        return ("C5 stream: 10000 distinct (graph, shape) requests over C1-C4 + fixtures "
                "(chain, diamond, empty, reshape, softmax, split), <= 4 MB input each", graphs, reqs)
    raise SystemExit(f"unknown workload {name}")


def workload_single(name):
    """(description, graph, [syms]) of a one-graph workload (tools/)."""
    wname, graphs, reqs = workload(name)
    (g,) = graphs.values()
    return wname, g, [s for _, s in reqs]


def const_value(name, syms):
    from paper_2103_05288_b200 import workloads as W
    if name == "inv_h":
        return 1.0 / syms.get("H", 1)
    return W.CONST_INPUTS.get(name)


def input_shape(inp, syms):
    return tuple(syms[d] if isinstance(d, str) else d for d in inp["shape"])


class Requests:
    """Device-resident inputs for every request, bound once; run = one stream pass."""

    def __init__(self, D, graphs, plans, reqs, seed=0):
        self.D = D
        self.bufs = []
        self.input_bytes = 0
        names, data, dims, offs, hplans = [], [], [], [0], []
        self._keep = []
        for r, (kind, syms) in enumerate(reqs):
            g = graphs[kind]
            for j, i in enumerate(g["inputs"]):
                shape = input_shape(i, syms)
                cv = const_value(i["id"], syms)
                if cv is not None:
                    b = D.DeviceBuffer.from_numpy(np.full(shape, cv, np.float32))
                else:
                    b = D.DeviceBuffer(shape)
                    b.fill_uniform(seed * 1000003 + r * 97 + j)
                self.bufs.append(b)
                d = np.array(shape, dtype=np.int64)
                self._keep.append(d)
                names.append(i["id"].encode())
                data.append(b.ptr.value)
                dims.append(d)
                self.input_bytes += b.nbytes
            offs.append(len(names))
            hplans.append(plans[kind]._h)
        self.n = len(reqs)
        t = max(len(names), 1)
        self.c_names = (C.c_char_p * t)(*names)
        self.c_data = (C.c_void_p * t)(*data)
        self.c_dims = (C.c_void_p * t)(*[d.ctypes.data for d in dims])
        self.c_ranks = (C.c_int * t)(*[d.size for d in dims])
        self.c_offs = (C.c_int * (self.n + 1))(*offs)
        self.c_plans = (C.c_void_p * max(self.n, 1))(*hplans)

    def run(self, ex):
        if self.n == 0:
            return
        rc = self.D.lib().disc_executor_run_stream(ex._h, self.n, self.c_plans, self.c_offs, self.c_names,
                                                    self.c_data, self.c_dims, self.c_ranks, 0)
        self.D.api._check(rc)

    def run_grouped(self, ex):
        """One grouped call: every request's runtime flow on the host, then the same plan
        kernel of all requests as one grouped launch (disc_executor_run_grouped)."""
        if self.n == 0:
            return
        rc = self.D.lib().disc_executor_run_grouped(ex._h, self.n, self.c_plans, self.c_offs, self.c_names,
                                                     self.c_data, self.c_dims, self.c_ranks, 0)
        self.D.api._check(rc)

    def run_streams(self, exs, which):
        """Requests interleaved over executors (own stream each): request r on which[r]."""
        if self.n == 0:
            return
        c_exs = (C.c_void_p * len(exs))(*[e._h for e in exs])
        c_which = (C.c_int * self.n)(*which)
        rc = self.D.lib().disc_executors_run_interleaved(c_exs, len(exs), self.n, c_which, self.c_plans, self.c_offs,
                                                          self.c_names, self.c_data, self.c_dims, self.c_ranks, 0)
        self.D.api._check(rc)


# ---------------------------------------------------------------------------
# Clocks during the timed region (B200_PROFILING.md clocks line)

class ClockSampler:
    def __init__(self, device):
        self.samples = []
        self.proc = None
        self.device = device

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------

def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(schedule):
    """dram bytes per launch for the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        t = json.load(open(p)).get("traffic_per_launch", {})
    except Exception:
        return None
    while schedule:  # "group:row_fused_cached" -> "group:row_fused" -> "group:row"
        if schedule in t:
            return t[schedule]
        schedule = schedule.rsplit("_", 1)[0] if "_" in schedule else ""
    return None


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "reference":
            dist.init_process_group("gloo")
        else:
            # BENCH_DEVICES_OVERRIDE=1: ranks share the visible GPUs round-robin over gloo
            # (exercises the multi-rank path on a 1-GPU box; not a scaling measurement)
            if os.environ.get("BENCH_DEVICES_OVERRIDE"):
                local = local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
            dist.init_process_group("gloo" if os.environ.get("BENCH_DEVICES_OVERRIDE") else "nccl")
    return world, rank, local, dist


def _dev(dist, local):
    return "cpu" if dist is not None and dist.get_backend() == "gloo" else f"cuda:{local}"


def barrier(dist, local):
    if dist is not None:
        import torch
        t = torch.zeros(1, device=_dev(dist, local))
        dist.all_reduce(t)
        torch.cuda.synchronize()


def allreduce(dist, local, v, op="max"):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=_dev(dist, local))
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def make_inputs(graph, syms, rng):
    inputs = {}
    for i in graph["inputs"]:
        shape = input_shape(i, syms)
        cv = const_value(i["id"], syms)
        inputs[i["id"]] = np.full(shape, cv, np.float32) if cv is not None else \
            rng.uniform(0.25, 2.0, size=shape).astype(np.float32)
    return inputs


def cpu_order(costs):
    """Request indices from the median of the byte distribution outward (bounded samples
    that stay representative of mid-size requests)."""
    order = sorted(range(len(costs)), key=lambda i: costs[i])
    mid = len(order) // 2
    out = []
    for d in range(len(order)):
        for j in ((mid + d, mid - d - 1) if d else (mid,)):
            if 0 <= j < len(order) and order[j] not in out:
                out.append(order[j])
    return out


def cpu_baseline(graphs, reqs, costs, budget_s=15.0):
    """Reference executor (oracle/_ref) on a bounded sample of the sweep, 1 thread:
    requests from the median outward until ~budget_s of CPU time."""
    from oracle import ref
    if not ref.available():
        return None
    rps = {k: ref.RefPlan(ref.compile(json.dumps(g))) for k, g in graphs.items()}
    rng = np.random.default_rng(0)
    total_bytes, total_s, used = 0, 0.0, []
    t_start = time.perf_counter()
    for i in cpu_order(costs):
        kind, syms = reqs[i]
        inputs = make_inputs(graphs[kind], syms, rng)
        rps[kind].run(inputs)  # warm the reference allocator cache
        total_s += rps[kind].time(inputs, 1)
        total_bytes += costs[i]
        used.append({k: v for k, v in syms.items() if not k.startswith("_")})
        if total_s > budget_s or time.perf_counter() - t_start > 3 * budget_s:
            break
    return {"value": total_bytes / total_s / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference",
            "sample": f"{len(used)} requests of the same sweep from the median size outward "
                      f"(e.g. {used[0]}), reference Executor::run, 1 thread, {total_s:.1f}s timed"}


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU executor, all host threads, same metric."""
    if world > 1 and rank != 0:
        return
    from oracle import ref
    import paper_2103_05288_b200 as D
    wname, graphs, reqs = workload(args.workload)
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    from concurrent.futures import ThreadPoolExecutor
    nthreads = os.cpu_count() or 1
    plans = {k: D.compile_graph(g) for k, g in graphs.items()}  # byte accounting only (host shape program)
    costs = [plans[k].algorithmic_bytes({i["id"]: input_shape(i, s) for i in graphs[k]["inputs"]}) for k, s in reqs]
    # per step: requests from the median outward, ~1 s of single-thread reference work per
    # host thread (estimated at the reference's ~0.2 GB/s/thread), all threads busy
    order = cpu_order(costs)
    budget = 0.2e9 * 1.0 * nthreads
    pick, acc = [], 0
    for i in order:
        pick.append(i)
        acc += costs[i]
        if acc >= budget or len(pick) >= 4096:
            break
    sample, scost = [reqs[i] for i in pick], [costs[i] for i in pick]
    rng = np.random.default_rng(0)
    inputs = [make_inputs(graphs[k], s, rng) for k, s in sample]
    ref_json = {k: ref.compile(json.dumps(g)) for k, g in graphs.items()}
    rps = [{k: ref.RefPlan(j) for k, j in ref_json.items()} for _ in range(nthreads)]
    nbytes = sum(scost)

    def step():
        def work(t):
            for i in range(t, len(sample), nthreads):
                rps[t][sample[i][0]].time(inputs[i], 1)
        with ThreadPoolExecutor(nthreads) as pool:
            list(pool.map(work, range(nthreads)))

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    v = nbytes * args.steps / dt / 1e9
    sample_desc = f"{len(sample)} requests of the sweep per step, reference Executor::run, {nthreads} threads"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wname, "sample": sample_desc},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": nthreads, "kind": "reference", "sample": sample_desc},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="disc", choices=["disc", "reference"])
    ap.add_argument("--workload", default="ln_gelu")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--schedule", default="auto")
    ap.add_argument("--e2e-pipes", type=int, default=3, help="executors/streams the e2e pass alternates over")
    ap.add_argument("--e2e-chunk-mb", type=int, default=256,
                    help="grouped e2e: boundary bytes per disc_executor_run_grouped call")
    ap.add_argument("--mode", default="grouped", choices=["grouped", "streams"],
                    help="grouped: one disc_executor_run_grouped call per step (the same plan kernel of all "
                         "requests fused into one grouped launch); streams: per-request launches interleaved "
                         "over --streams executors")
    ap.add_argument("--host-threads", type=int, default=min(16, os.cpu_count() or 1),
                    help="grouped mode: host threads running the requests' runtime flows")
    ap.add_argument("--streams", type=int, default=2,
                    help="executors/streams per GPU the requests are interleaved over (independent requests overlap)")
    ap.add_argument("--stream-policy", default="lpt", choices=["size", "lpt"],
                    help="size: requests >= --big-bytes on stream 0, the rest LPT over the others; lpt: LPT over all")
    ap.add_argument("--big-bytes", type=float, default=256e6)
    ap.add_argument("--pdl", type=int, default=1, choices=[0, 1, 2],
                    help="programmatic dependent launch: 0 off, 1 overlap launch, 2 + early CTA launch")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world, rank, local, dist = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        if dist is not None:
            dist.destroy_process_group()
        return

    import paper_2103_05288_b200 as D
    from paper_2103_05288_b200.dispatch import shard
    D.lib()
    D.set_pdl(args.pdl)
    wname, graphs, reqs = workload(args.workload)
    for r in range(1, world):  # N distinct sweeps, sharded below
        _, g2, rq2 = workload(args.workload, replica=r)
        graphs.update(g2)
        reqs = reqs + rq2
    D.api._cuda(D.lib().disc_cuda_set_device(local))
    streams, exs = [], []
    for _ in range(max(1, args.streams) if args.mode == "streams" else 1):
        st = C.c_void_p()
        D.api._cuda(D.lib().disc_cuda_stream_create(C.byref(st)))
        streams.append(st)
        exs.append(D.Executor(local, st.value))
        exs[-1].set_schedule(args.schedule)
        if args.mode == "grouped":
            exs[-1].set_host_threads(args.host_threads)
    stream, ex = streams[0], exs[0]
    compiler = D.Compiler()
    plans = {}
    for k, s in reqs:  # every request asks the cache: 1 compile per distinct graph
        plans[k] = compiler.compile(graphs[k])
    costs = [plans[k].algorithmic_bytes({i["id"]: input_shape(i, s) for i in graphs[k]["inputs"]}) for k, s in reqs]
    mine = shard(costs, world)[rank]
    my_reqs = [reqs[i] for i in mine]
    my_bytes = sum(costs[i] for i in mine)
    which = [0] * len(mine)  # request -> local stream
    mc = [costs[i] for i in mine]
    if args.stream_policy == "size" and len(exs) > 1:
        # large requests serialise on stream 0 (one-wave kernels that fill the GPU);
        # small/mid ones (latency-bound per kernel) spread over the other streams
        small = [j for j, c in enumerate(mc) if c < args.big_bytes]
        for k, part in enumerate(shard([mc[j] for j in small], len(exs) - 1)):
            for j in part:
                which[small[j]] = k + 1
    else:
        for k, part in enumerate(shard(mc, len(exs))):  # balanced by bytes (LPT)
            for j in part:
                which[j] = k
    rq = Requests(D, graphs, plans, my_reqs, seed=rank)
    D.api._cuda(D.lib().disc_cuda_device_synchronize())

    sm, l2, hbm = C.c_int(), C.c_int64(), C.c_int64()
    D.lib().disc_cuda_device_info(local, C.byref(sm), C.byref(l2), C.byref(hbm))
    flush_bytes = max(4 * l2.value, 1 << 28)
    flush = C.c_void_p()
    D.api._cuda(D.lib().disc_cuda_malloc(flush_bytes, stream, C.byref(flush)))
    ev = [C.c_void_p(), C.c_void_p()]
    for e in ev:
        D.api._cuda(D.lib().disc_cuda_event_create(C.byref(e)))
    join = []
    for _ in streams:
        e = C.c_void_p()
        D.api._cuda(D.lib().disc_cuda_event_create(C.byref(e)))
        join.append(e)
    L = D.lib()

    def one_pass():
        """One pass over this rank's requests, all streams joined back into streams[0]."""
        if args.mode == "grouped":
            rq.run_grouped(ex)
            return
        if len(exs) == 1:
            rq.run(ex)
            return
        for st in streams[1:]:
            L.disc_cuda_stream_wait_event(st, ev[0])
        rq.run_streams(exs, which)
        for st, e in zip(streams[1:], join[1:]):
            L.disc_cuda_event_record(e, st)
            L.disc_cuda_stream_wait_event(stream, e)

    for _ in range(args.warmup):
        L.disc_cuda_event_record(ev[0], stream)
        one_pass()
        L.disc_cuda_stream_synchronize(stream)
    D.api._cuda(L.disc_cuda_device_synchronize())
    step_bytes = sum(e.algorithmic_bytes() for e in exs)  # executors' own count for the last pass (this rank)
    if step_bytes != my_bytes:
        log(f"warning: executor bytes {step_bytes} != planned {my_bytes}")
    total_bytes = allreduce(dist, local, step_bytes, "sum")

    # ---- timed region: K steps, device time per step (flush untimed) ----
    launches0 = D.kernel_launches()
    step_ms = []
    step_ev = []
    for _ in range(2 * args.steps):
        e = C.c_void_p()
        D.api._cuda(L.disc_cuda_event_create(C.byref(e)))
        step_ev.append(e)
    barrier(dist, local)
    wall0 = time.perf_counter()
    with ClockSampler(local) as clk:
        # K steps issued back to back (the host prepares step i+1 while the device runs
        # step i); each step's device time is its own event pair, the L2 flush before it
        # is outside the pair.
        for i in range(args.steps):
            L.disc_cuda_flush_l2(flush, flush_bytes, stream)
            L.disc_cuda_event_record(step_ev[2 * i], stream)
            if args.mode != "grouped":
                L.disc_cuda_event_record(ev[0], stream)  # the interleaved streams wait on it
            one_pass()
            L.disc_cuda_event_record(step_ev[2 * i + 1], stream)
        L.disc_cuda_stream_synchronize(stream)
        for i in range(args.steps):
            ms = C.c_float()
            L.disc_cuda_event_elapsed_ms(step_ev[2 * i], step_ev[2 * i + 1], C.byref(ms))
            step_ms.append(ms.value)
    wall = time.perf_counter() - wall0
    flushes = args.steps
    gpu_launches = D.kernel_launches() - launches0 - flushes
    barrier(dist, local)
    total_ms = allreduce(dist, local, sum(step_ms), "max")
    ms_per_step = total_ms / args.steps
    value = total_bytes / (ms_per_step / 1e3) / 1e9
    compile_count = compiler.stats()["compile_count"]

    # ---- per-kernel device time (untimed pass): the pass is queued behind a spin
    # kernel so per-launch events see device execution, not host submission gaps ----
    records = []
    ex.set_timing(True)
    for _ in range(2):
        D.lib().disc_cuda_flush_l2(flush, flush_bytes, stream)
        D.lib().disc_cuda_spin(50000, stream)
        if args.mode == "grouped":
            rq.run_grouped(ex)  # one record per grouped launch
        else:
            rq.run(ex)
        D.lib().disc_cuda_stream_synchronize(stream)
        records.extend(ex.launch_records())
    ex.set_timing(False)
    device_ms = sum(r["ms"] for r in records) / 2

    # ---- roofline: dominant kernel ----
    peak, peak_kind = peaks()
    by_kernel = {}
    for r in records:
        k = (r["kernel"], r["schedule"])
        b = by_kernel.setdefault(k, [0, 0.0, 0])
        b[0] += r["bytes"]
        b[1] += r["ms"]
        b[2] += 1
    (dk, dsched), (dbytes, dms, dn) = max(by_kernel.items(), key=lambda kv: kv[1][1])
    achieved = dbytes / (dms / 1e3) / 1e9 if dms > 0 else 0.0
    kernel_ms_total = sum(v[1] for v in by_kernel.values())
    breakdown = {f"k{k}:{s}": {"GB/s": round(b / (ms / 1e3) / 1e9, 1) if ms else None,
                              "share": round(ms / kernel_ms_total, 3) if kernel_ms_total else None,
                              "launches_per_step": n // 2}
                 for (k, s), (b, ms, n) in sorted(by_kernel.items())}
    if len(breakdown) > 12:  # stream: many artifacts; keep the 12 largest shares
        breakdown = dict(sorted(breakdown.items(), key=lambda kv: -(kv[1]["share"] or 0))[:12])
    # large-shape class (the >=70% target applies to large shapes)
    big = [r for r in records if r["bytes"] >= (64 << 20)]
    big_gbs = sum(r["bytes"] for r in big) / (sum(r["ms"] for r in big) / 1e3) / 1e9 if big else None

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(D, graphs, plans, my_reqs, [costs[i] for i in mine], local, stream, pipes=args.e2e_pipes,
                          grouped=args.mode == "grouped", chunk_bytes=args.e2e_chunk_mb << 20)
        if e2e is not None and dist is not None:
            e2e["value"] = round(allreduce(dist, local, e2e["bytes"], "sum") /
                                 allreduce(dist, local, e2e["seconds"], "max") / 1e9, 2)
    clocks = clk.summary()

    out = None
    if rank == 0:
        cpu = None if args.no_cpu_baseline or world > 1 else cpu_baseline(graphs, reqs, costs)
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (uniform [0.25, 2) f32, device-generated)",
            "config": {"workload": wname, "distinct_shapes": len(set((k, tuple(sorted(s.items()))) for k, s in reqs)),
                       "requests_per_step": len(reqs), "graphs": len(graphs), "bytes_per_step": int(total_bytes),
                       "l2": "flushed before each step (4x L2 write)",
                       "parallelism": f"request-sharded x{world} (LPT on algorithmic bytes, no collectives)",
                       "schedule": args.schedule, "pdl": args.pdl, "mode": args.mode,
                       "host_threads": args.host_threads if args.mode == "grouped" else 1,
                       "streams_per_gpu": len(exs),
                       "stream_policy": args.stream_policy if len(exs) > 1 else None},
            "frac_of_hbm_peak": round(value / world / peak, 4),
            "recompiles": compile_count - len(graphs),
            "compile_count": compile_count,
            "large_shape_GBps": round(big_gbs, 1) if big_gbs else None,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": ncu_traffic(dsched),
                         "kernel": f"artifact {dk} ({dsched})", "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs",
                         "bytes_per_launch": dbytes // max(dn, 1), "mean_launch_ms": round(dms / max(dn, 1), 5)},
            "kernel_breakdown": breakdown,
            "device_ms_per_step": round(device_ms, 4),
            "host_bound_frac": round(max(0.0, 1 - device_ms / ms_per_step), 3),
            "cpu_baseline": cpu,
            "e2e": {k: v for k, v in e2e.items() if k not in ("bytes", "seconds")} if e2e else None,
            "gpu_launches": gpu_launches,
            "clocks": clocks,
            "wall_s_timed": round(wall, 3),
        }
        print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


def measure_e2e(D, graphs, plans, reqs, costs, device, stream, max_input_bytes=8 << 30, pipes=3, grouped=True,
                chunk_bytes=1 << 30):
    """Public API, host buffers: every request's inputs go H2D from pinned memory inside
    disc_executor_run(inputs_on_host=1), its outputs D2H into pinned memory
    (disc_executor_copy_output, async); wall time of one pass.  Requests alternate over
    `pipes` executors (own stream + allocator each), so one request's D2H overlaps the
    next one's H2D and compute (PCIe is full duplex).  Requests up to max_input_bytes of
    pinned input (the whole C2 sweep fits)."""
    L = D.lib()
    exs, streams = [], []
    for _ in range(pipes):
        st = C.c_void_p()
        D.api._cuda(L.disc_cuda_stream_create(C.byref(st)))
        streams.append(st)
        exs.append(D.Executor(device, st.value))
    pinned, work = [], []
    h2d = d2h = in_bytes = nbytes = 0
    rng = np.random.default_rng(1)
    for (kind, syms), cost in zip(reqs, costs):
        g = graphs[kind]
        ptrs, dims = [], []
        size = sum(4 * int(np.prod(input_shape(i, syms))) for i in g["inputs"])
        if in_bytes + size > max_input_bytes:
            break
        in_bytes += size
        for i in g["inputs"]:
            shape = input_shape(i, syms)
            n = int(np.prod(shape))
            p = C.c_void_p()
            D.api._cuda(L.disc_cuda_host_alloc(max(4 * n, 16), C.byref(p)))
            arr = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float)), shape=(max(n, 1),))
            cv = const_value(i["id"], syms)
            arr[:n] = cv if cv is not None else rng.uniform(0.25, 2.0, size=n).astype(np.float32)
            pinned.append(p)
            ptrs.append(p.value)
            dims.append(np.array(shape, dtype=np.int64))
            h2d += 4 * n
        names = [i["id"] for i in g["inputs"]]
        work.append((plans[kind], (C.c_char_p * len(names))(*[s.encode() for s in names]),
                     (C.c_void_p * len(ptrs))(*ptrs), dims, (C.c_void_p * len(dims))(*[d.ctypes.data for d in dims]),
                     (C.c_int * len(dims))(*[d.size for d in dims])))
        nbytes += cost
    if not work:
        return None
    outs = {}

    def out_buf(key, n):
        if key not in outs:
            p = C.c_void_p()
            D.api._cuda(L.disc_cuda_host_alloc(max(4 * n, 16), C.byref(p)))
            outs[key] = p
        return outs[key]

    # grouped: consecutive requests in chunks of ~chunk_bytes of boundary traffic, one
    # disc_executor_run_grouped(inputs_on_host=1) call per chunk, chunks alternating over
    # the pipes (chunk c's H2D overlaps chunk c-1's kernels and chunk c-2's D2H)
    chunks, cur, acc = [], [], 0
    for r, cost in enumerate(costs[:len(work)]):
        cur.append(r)
        acc += cost
        if acc >= chunk_bytes:
            chunks.append(cur)
            cur, acc = [], 0
    if cur:
        chunks.append(cur)
    cargs = []
    for ch in chunks:
        names, datas, dimsp, ranks, offs, hplans = [], [], [], [], [0], []
        for r in ch:
            plan, c_names, data, dims, c_dims, c_ranks = work[r]
            n = len(dims)
            names += [c_names[i] for i in range(n)]
            datas += [data[i] for i in range(n)]
            dimsp += [c_dims[i] for i in range(n)]
            ranks += [c_ranks[i] for i in range(n)]
            offs.append(offs[-1] + n)
            hplans.append(plan._h)
        t = max(len(names), 1)
        cargs.append((len(ch), (C.c_void_p * len(ch))(*hplans), (C.c_int * (len(ch) + 1))(*offs),
                      (C.c_char_p * t)(*names), (C.c_void_p * t)(*datas), (C.c_void_p * t)(*dimsp),
                      (C.c_int * t)(*ranks)))

    def one_pass_grouped():
        nonlocal d2h
        d2h = 0
        for c, (ch, a) in enumerate(zip(chunks, cargs)):
            ex = exs[c % pipes]
            D.api._check(L.disc_executor_run_grouped(ex._h, *a, 1))
            for j, r in enumerate(ch):
                for o, (_, odims) in enumerate(ex.request_output_views(j)):
                    n = int(np.prod(odims)) if odims else 1
                    if n:
                        D.api._check(L.disc_executor_copy_request_output(ex._h, j, o, out_buf((r, o), n), 2))
                    d2h += 4 * n
        for ex in exs:
            ex.synchronize()

    def one_pass():
        nonlocal d2h
        if grouped:
            return one_pass_grouped()
        d2h = 0
        for r, (plan, c_names, data, dims, c_dims, c_ranks) in enumerate(work):
            ex = exs[r % pipes]
            D.api._check(L.disc_executor_run(ex._h, plan._h, len(dims), c_names, data, c_dims, c_ranks, 1))
            for o, (_, odims) in enumerate(ex.output_views()):
                n = int(np.prod(odims)) if odims else 1
                key = (r, o)
                if key not in outs:
                    p = C.c_void_p()
                    D.api._cuda(L.disc_cuda_host_alloc(max(4 * n, 16), C.byref(p)))
                    outs[key] = p
                if n:
                    D.api._check(L.disc_executor_copy_output(ex._h, o, outs[key], 2))
                d2h += 4 * n
        for ex in exs:
            ex.synchronize()

    one_pass()  # warm allocators + staging
    t0 = time.perf_counter()
    one_pass()
    dt = time.perf_counter() - t0
    for p in pinned + list(outs.values()):
        L.disc_cuda_host_free(p)
    del exs
    path = (f"disc_executor_run_grouped(inputs_on_host=1) per chunk of requests ({len(chunks)} chunks of "
            f"~{chunk_bytes >> 20} MB) + disc_executor_copy_request_output(pinned host, async), chunks alternating "
            f"over {pipes} executors/streams") if grouped else \
        (f"disc_executor_run(inputs_on_host=1) + disc_executor_copy_output(pinned host, async) per "
         f"request, requests alternating over {pipes} executors/streams")
    return {"value": round(nbytes / dt / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(dt * 1e3, 3), "requests": len(work),
            "path": path, "bytes": nbytes, "seconds": dt}


if __name__ == "__main__":
    main()
