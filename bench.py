#!/usr/bin/env python
"""disc-b200 benchmark: fused-kernel HBM GB/s across a dynamic-shape sweep, 0 recompiles.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload sweep|ln_gelu|softmax|colreduce|bert|stream]
                  [--verify off|sample|full]
  python bench.py --impl reference ...     # the reference's own CPU executor, same workload

Headline workload ``sweep`` (BASELINE metric; SURVEY §8(d) C5 over the FULL C1-C4
ranges): every step is 10 000 distinct (graph, shape) requests, kinds round-robin over
C1 softmax, C2 LN+bias+GELU, C3 column reduce, C4 BERT non-GEMM and the reference
fixtures, every dimension drawn log-uniformly over its whole configured range, FRESH
shapes every step (no shape repeats in the run, so the recipe cache is cold).  One plan
per graph is compiled once: 0 recompiles.  A step = the step's requests issued through
disc_executor_run_grouped in chunks of ~--chunk-gb of algorithmic bytes (host flow of
chunk c+1 overlaps the device work of chunk c).  Inputs are views into a device-resident
arena of uniform [0.25, 2) f32 (inputs already in HBM when the timed region starts,
>> L2; the L2 is also flushed before every step).

  value    = algorithmic bytes (4 x (external inputs read + outputs
             written) per fused launch, broadcast sources at source size) of the K timed
             steps / their device time (CUDA events on the executor stream, max over ranks)
  e2e      = the same metric through the public C ABI with HOST buffers: H2D of every
             request's inputs (pinned) and D2H of its outputs inside the timed region, on
             a stratified sample of a step (bounded pinned memory)
  roofline = the dominant kernel, keyed (pattern, plan kernel, schedule): its bytes / its
             mean CUDA-event duration in per-pattern passes, against MEASURED_PEAKS.json
  cpu_baseline = the reference executor (oracle/_ref) on a stratified sample of the same
             step, 1 host thread
  verify   = B200 outputs of a timed step's exact grouped pass against the reference
             executor (oracle/verify.py): sample (default) or full (every request with
             inputs <= 2^22 elements + sampled rows of every larger one)

Multi-GPU (torchrun, one process per GPU): ``sweep`` draws an independent 10k-request
stream per rank (weak scaling); the fixed sweeps are replicated and LPT-sharded on
algorithmic bytes (paper_2103_05288_b200/dispatch.py).  No collective touches the data
path; barriers bracket the timed region and the max over ranks is reported.
"""
from __future__ import annotations

import argparse
import ctypes as C
import importlib.util
import json
import math
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
LARGE = 64 << 20  # "large shape": a request moving >= 64 MiB of algorithmic bytes
MAIN_KINDS = ("softmax", "ln_gelu", "colreduce", "bert")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def W():
    """paper_2103_05288_b200/workloads.py loaded by path: pure Python graph/shape
    definitions, so the reference arm never imports (or maps) the B200 package."""
    mod = sys.modules.get("disc_workloads")
    if mod is None:
        spec = importlib.util.spec_from_file_location("disc_workloads",
                                                      os.path.join(ROOT, "paper_2103_05288_b200", "workloads.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        sys.modules["disc_workloads"] = mod
    return mod


def host_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def load_fixtures():
    """Reference fixture graphs (GEMM fixtures excluded: library calls, not fused kernels)."""
    fx = json.load(open(os.path.join(ROOT, "tests", "golden", "fixtures.json")))
    return {k: (json.loads(v["graph"]), v["bindings"]) for k, v in sorted(fx.items())
            if k not in ("matmul", "transformer")}


# ---------------------------------------------------------------------------
# Workloads

class Workload:
    """name, description, {kind: graph}; requests(step) -> [(kind, syms)].  Fresh
    workloads draw new shapes every step; fixed ones repeat one sweep."""

    def __init__(self, name, desc, graphs, fixed=None, draw=None):
        self.name, self.desc, self.graphs = name, desc, graphs
        self._fixed, self._draw, self._steps = fixed, draw, []
        self.fresh = draw is not None

    def requests(self, step):
        if self._fixed is not None:
            return self._fixed
        while len(self._steps) <= step:
            self._steps.append(self._draw(len(self._steps)))
        return self._steps[step]


def make_workload(name, replica=0, n_requests=10000):
    w = W()
    if name == "sweep":
        fx = load_fixtures()
        graphs = w.sweep_graphs(fx)
        return Workload(name, f"C5 full-range sweep: {n_requests} distinct (graph, shape) requests per step, fresh "
                              "shapes every step, over C1 softmax [B<=2^26/S, S<=4096], C2 LN+bias+GELU [T<=16384, "
                              "H in {768,1024,4096}], C3 column reduce [N<=2^22, C<=4096], C4 BERT non-GEMM "
                              "[B<=32, S 8..512] and the reference fixtures (chain, diamond, empty, reshape, "
                              "softmax, split); dims log-uniform", graphs,
                        draw=lambda step: w.full_sweep(step, n=n_requests, seed=20261017 + 1000003 * replica,
                                                       fixtures=fx)[1])
    if name == "ln_gelu":
        return Workload(name, "C2 LN-like+bias+tanh-GELU [T,H], T log-uniform 1..16384 x H {768,1024,4096}",
                        {name: w.ln_gelu_graph()}, fixed=[(name, s) for s in w.ln_shapes(seed=20261017 + replica)])
    if name == "softmax":
        return Workload(name, "C1 softmax [B,S], S 1..4096, B = 2^26/S", {name: w.softmax_graph_for(0)},
                        fixed=[(name, {"S0": s["S0"], "S1": s["_S"]}) for s in w.softmax_shapes()])
    if name == "colreduce":
        return Workload(name, "C3 column reduce with prologue [N,C]", {name: w.colreduce_graph()},
                        fixed=[(name, s) for s in w.colreduce_shapes()])
    if name == "bert":
        return Workload(name, "C4 BERT-base non-GEMM subgraphs, S 8..512, B {1,8,32}", {name: w.bert_graph()},
                        fixed=[(name, s) for s in w.bert_shapes()])
    if name == "stream":
        graphs, reqs = w.mixed_stream(10000, seed=20261017 + replica, fixtures=load_fixtures())
        return Workload(name, "C5 small-shape stream: 10000 distinct (graph, shape) requests over C1-C4 + fixtures, "
                              "<= 4 MB input each (same shapes every step)", graphs, fixed=reqs)
    raise SystemExit(f"unknown workload {name}")


def input_shape(inp, syms):
    return tuple(syms[d] if isinstance(d, str) else d for d in inp["shape"])


def const_value(name, syms):
    if name == "inv_h":
        return 1.0 / syms.get("H", 1)
    return W().CONST_INPUTS.get(name)


def stratified(items, costs, budget, seed=0):
    """Systematic sample of `items` (sorted by (kind, cost)) whose cost sums to ~budget:
    every m-th request from a seeded offset, so every pattern and size class is present
    in proportion."""
    total = sum(costs)
    if total <= budget:
        return list(range(len(items)))
    order = sorted(range(len(items)), key=lambda i: (items[i][0], costs[i]))
    m = max(1, math.ceil(total / max(budget, 1)))
    start = seed % m
    return sorted(order[start::m])


# ---------------------------------------------------------------------------
# Device side (B200 arm)

class Arena:
    """Device-resident synthetic inputs: one buffer of uniform [0.25, 2) f32; every request
    input is a 256 B-aligned view at a moving cursor (wrapping), so consecutive requests
    read distinct memory.  [1]-shaped constants (eps, GELU constants, 1/H, ...) come from
    a small constant table."""

    def __init__(self, D, nbytes, stream, seed=0):
        self.D, self.L, self.stream = D, D.lib(), stream
        self.nbytes = nbytes // 256 * 256
        self.ptr = C.c_void_p()
        D.api._cuda(self.L.disc_cuda_malloc(self.nbytes, stream, C.byref(self.ptr)), "arena")
        D.api._cuda(self.L.disc_cuda_fill_uniform(self.ptr, self.nbytes // 4, 0x5EED + seed, 0.25, 2.0, stream), "fill")
        self.cursor = 0
        self.consts, self.cvals = {}, []
        self.cptr = C.c_void_p()
        D.api._cuda(self.L.disc_cuda_malloc(4096, stream, C.byref(self.cptr)), "const table")

    def const(self, v):
        v = float(np.float32(v))
        if v not in self.consts:
            self.consts[v] = len(self.cvals)
            self.cvals.append(v)
            arr = np.array(self.cvals, np.float32)
            self.D.api._cuda(self.L.disc_cuda_memcpy(self.cptr, arr.ctypes.data, arr.nbytes, 0, self.stream), "h2d")
            self.D.api._cuda(self.L.disc_cuda_stream_synchronize(self.stream), "sync")
        return self.cptr.value + 4 * self.consts[v]

    def take(self, nbytes):
        nbytes = (max(nbytes, 4) + 255) // 256 * 256
        if nbytes > self.nbytes:
            raise RuntimeError(f"input of {nbytes} B exceeds the {self.nbytes} B arena")
        if self.cursor + nbytes > self.nbytes:
            self.cursor = 0
        p = self.ptr.value + self.cursor
        self.cursor += nbytes
        return p

    def d2h(self, ptr, shape, rows=None):
        """Host copy of a device tensor (optionally only rows `rows` of its leading dim)."""
        L, D = self.L, self.D
        shape = tuple(shape)
        if not ptr and int(np.prod(shape)):
            raise RuntimeError(f"d2h: null device pointer for a {shape} tensor")
        if rows is None:
            a = np.empty(shape, np.float32)
            if a.size:
                D.api._cuda(L.disc_cuda_memcpy(a.ctypes.data, C.c_void_p(ptr), a.nbytes, 1, self.stream), "d2h")
            return a
        row = int(np.prod(shape[1:])) if len(shape) > 1 else 1
        a = np.empty((len(rows),) + shape[1:], np.float32)
        for j, r in enumerate(rows):
            if not 0 <= int(r) < shape[0]:
                raise RuntimeError(f"d2h: row {int(r)} outside a {shape} tensor")
            if row:
                D.api._cuda(L.disc_cuda_memcpy(a.ctypes.data + 4 * row * j, C.c_void_p(ptr + 4 * row * int(r)),
                                               4 * row, 1, self.stream), f"d2h row {int(r)} of {shape} at {ptr:#x}")
        return a


call_ms_mallocs = []  # pool-malloc counter after each timed grouped call (diagnostics)


class StepBatch:
    """One step's requests as flat C-ABI arrays (names / data / dims / ranks / offsets /
    plans), bound to arena views, split into chunks of ~chunk_bytes algorithmic bytes."""

    _names = {}

    def __init__(self, D, arena, graphs, plans, reqs, costs, chunk_bytes):
        self.D, self.L = D, D.lib()
        self.reqs, self.costs, self.graphs = reqs, costs, graphs
        n_in = sum(len(graphs[k]["inputs"]) for k, _ in reqs)
        self.names = np.zeros(max(n_in, 1), np.uint64)
        self.data = np.zeros(max(n_in, 1), np.uint64)
        self.dimsp = np.zeros(max(n_in, 1), np.uint64)
        self.ranks = np.zeros(max(n_in, 1), np.int32)
        self.offs = np.zeros(len(reqs) + 1, np.int32)
        self.plans = np.array([plans[k]._h.value for k, _ in reqs] or [0], np.uint64)
        flat = []
        self.bind = []  # per request: [(input id, ptr, shape)]
        i = 0
        for r, (kind, syms) in enumerate(reqs):
            b = []
            for inp in graphs[kind]["inputs"]:
                shape = input_shape(inp, syms)
                cv = const_value(inp["id"], syms)
                p = arena.const(cv) if cv is not None else arena.take(4 * int(np.prod(shape)))
                nm = StepBatch._names.setdefault(inp["id"], C.create_string_buffer(inp["id"].encode()))
                self.names[i] = C.addressof(nm)
                self.data[i] = p
                self.ranks[i] = len(shape)
                flat.append((i, shape))
                b.append((inp["id"], p, shape))
                i += 1
            self.offs[r + 1] = i
            self.bind.append(b)
        self.dims_flat = np.array([d for _, s in flat for d in s] or [0], np.int64)
        pos = 0
        base = self.dims_flat.ctypes.data
        for k, s in flat:
            self.dimsp[k] = base + 8 * pos
            pos += len(s)
        # chunks: consecutive requests up to chunk_bytes of algorithmic bytes
        self.chunks, r0, acc = [], 0, 0
        for r, c in enumerate(costs):
            acc += c
            if acc >= chunk_bytes:
                self.chunks.append((r0, r + 1))
                r0, acc = r + 1, 0
        if r0 < len(reqs):
            self.chunks.append((r0, len(reqs)))
        self.chunk_offs = [np.ascontiguousarray(self.offs[a:b + 1] - self.offs[a]) for a, b in self.chunks]
        self.bytes = int(sum(costs))

    def _p(self, arr, k, ctype):
        return C.cast(C.c_void_p(arr.ctypes.data + arr.itemsize * int(k)), C.POINTER(ctype))

    def run(self, ex, on_chunk=None, call_ms=None):
        L = self.L
        for ci, (a, b) in enumerate(self.chunks):
            t0 = time.perf_counter()
            i0 = int(self.offs[a])
            rc = L.disc_executor_run_grouped(ex._h, b - a, self._p(self.plans, a, C.c_void_p),
                                             self.chunk_offs[ci].ctypes.data_as(C.POINTER(C.c_int)),
                                             self._p(self.names, i0, C.c_char_p), self._p(self.data, i0, C.c_void_p),
                                             self._p(self.dimsp, i0, C.c_void_p), self._p(self.ranks, i0, C.c_int), 0)
            self.D.api._check(rc)
            if call_ms is not None:
                call_ms.append((time.perf_counter() - t0) * 1e3)
                call_ms_mallocs.append(alloc_stats(self.D)[0])
            if on_chunk is not None:
                ex.wait_issued()
                on_chunk(ci, a, b)
        ex.wait_issued()  # the caller records events / launches on the stream next


class Bench:
    """Device state of the B200 arm: executor, arena, plans, events, L2 flush buffer."""

    def __init__(self, D, args, local, workload):
        self.D, self.L, self.args, self.wl, self.local = D, D.lib(), args, workload, local
        L = self.L
        D.api._cuda(L.disc_cuda_set_device(local))
        st = C.c_void_p()
        D.api._cuda(L.disc_cuda_stream_create(C.byref(st)))
        self.stream = st
        self.ex = D.Executor(local, st.value)
        self.ex.set_schedule(args.schedule)
        self.ex.set_host_threads(args.host_threads)
        self.ex.set_cache_budget(int(args.cache_gb * (1 << 30)))
        self.ex.set_async_flush(bool(getattr(args, "async_flush", 1)))
        if getattr(args, "reserve_gb", 0):
            self.ex.reserve(int(args.reserve_gb * (1 << 30)))
        self.compiler = D.Compiler()
        self.plans = {}
        sm, l2, hbm = C.c_int(), C.c_int64(), C.c_int64()
        L.disc_cuda_device_info(local, C.byref(sm), C.byref(l2), C.byref(hbm))
        self.hbm = hbm.value
        self.flush_bytes = max(4 * l2.value, 1 << 28)
        self.flush = C.c_void_p()
        D.api._cuda(L.disc_cuda_malloc(self.flush_bytes, st, C.byref(self.flush)))
        arena_bytes = int(min(args.arena_gb * (1 << 30), 0.3 * self.hbm)) if self.hbm else int(args.arena_gb * (1 << 30))
        self.arena = Arena(D, arena_bytes, st, seed=local)
        D.api._cuda(L.disc_cuda_stream_synchronize(st))

    def release(self):
        """Releases the executor (its reserved buffer arena) and the device input arena once
        the device-input passes are done, so the e2e pass's executors have the HBM."""
        L = self.L
        L.disc_cuda_stream_synchronize(self.stream)
        if self.ex is not None:
            self.ex.close()
            self.ex = None
        if self.arena is not None:
            for p in (self.arena.ptr, self.arena.cptr):
                L.disc_cuda_free(p, self.stream)
            self.arena = None
        L.disc_cuda_stream_synchronize(self.stream)

    def close(self):
        """Releases the executor, arena, flush buffer and stream (tests create several)."""
        L = self.L
        self.release()
        L.disc_cuda_free(self.flush, self.stream)
        L.disc_cuda_stream_synchronize(self.stream)
        L.disc_cuda_stream_destroy(self.stream)

    def plans_for(self, reqs):
        for k in {k for k, _ in reqs}:  # one compile per distinct graph (Compiler cache); the handle is kept
            if k not in self.plans:      # alive for every batch that points at it
                self.plans[k] = self.compiler.compile(self.wl.graphs[k])
        return self.plans

    def costs(self, reqs):
        g = self.wl.graphs
        return [self.plans[k].algorithmic_bytes({i["id"]: input_shape(i, s) for i in g[k]["inputs"]}) for k, s in reqs]

    def batch(self, reqs, costs=None):
        self.plans_for(reqs)
        costs = costs if costs is not None else self.costs(reqs)
        return StepBatch(self.D, self.arena, self.wl.graphs, self.plans, reqs, costs, self.args.chunk_gb * (1 << 30))

    def event(self):
        e = C.c_void_p()
        self.D.api._cuda(self.L.disc_cuda_event_create(C.byref(e)))
        return e

    def timed_pass(self, batch, flush=True):
        """Device ms of one pass over `batch` (events on the executor stream)."""
        L = self.L
        a, b = self.event(), self.event()
        if flush:
            L.disc_cuda_flush_l2(self.flush, self.flush_bytes, self.stream)
        L.disc_cuda_event_record(a, self.stream)
        batch.run(self.ex)
        L.disc_cuda_event_record(b, self.stream)
        L.disc_cuda_stream_synchronize(self.stream)
        ms = C.c_float()
        L.disc_cuda_event_elapsed_ms(a, b, C.byref(ms))
        L.disc_cuda_event_destroy(a)
        L.disc_cuda_event_destroy(b)
        return ms.value

    def device_bound_pass(self, batch, spin_us=600000):
        """Device ms of one pass issued exactly as timed (same chunks, phases, threads) while
        the stream is held behind a spin kernel, so the host's issue time is hidden: the
        step's device-bound time (host_bound_frac compares the timed step with it)."""
        L = self.L
        a, b = self.event(), self.event()
        L.disc_cuda_flush_l2(self.flush, self.flush_bytes, self.stream)
        L.disc_cuda_spin(spin_us, self.stream)
        L.disc_cuda_event_record(a, self.stream)
        t0 = time.perf_counter()
        batch.run(self.ex)
        host_ms = (time.perf_counter() - t0) * 1e3
        L.disc_cuda_event_record(b, self.stream)
        L.disc_cuda_stream_synchronize(self.stream)
        ms = C.c_float()
        L.disc_cuda_event_elapsed_ms(a, b, C.byref(ms))
        L.disc_cuda_event_destroy(a)
        L.disc_cuda_event_destroy(b)
        if host_ms > spin_us / 1e3:
            log(f"[bench] device_bound_pass: host issue {host_ms:.1f} ms exceeded the {spin_us / 1e3:.0f} ms spin")
        return ms.value, host_ms

    def record_pass(self, batch):
        """Per grouped launch records (timing mode: device ms per launch) of one pass."""
        recs = []
        self.ex.set_timing(True)
        self.L.disc_cuda_flush_l2(self.flush, self.flush_bytes, self.stream)
        self.L.disc_cuda_spin(20000, self.stream)  # queue behind a spin: events see device time
        batch.run(self.ex, on_chunk=lambda ci, a, b: recs.extend(self.ex.launch_records()))
        self.ex.set_timing(False)
        self.L.disc_cuda_stream_synchronize(self.stream)
        return recs


# ---------------------------------------------------------------------------
# Clocks during the timed region (B200_PROFILING.md clocks line)

class ClockSampler:
    def __init__(self, device):
        self.samples, self.proc, self.device = [], None, device

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


def alloc_stats(D):
    m, f, o = C.c_int64(), C.c_int64(), C.c_int64()
    D.lib().disc_cuda_alloc_stats(C.byref(m), C.byref(f), C.byref(o))
    return m.value, f.value, o.value


def cpu_times():
    try:
        with open("/proc/stat") as fh:
            return [int(x) for x in fh.readline().split()[1:]]
    except OSError:
        return None


def cpu_steal(a, b):
    """Fraction of CPU time stolen by the hypervisor between two /proc/stat samples."""
    if not a or not b or len(a) < 8:
        return None
    d = [y - x for x, y in zip(a, b)]
    return round(d[7] / max(1, sum(d[:8])), 4)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured MEASURED_PEAKS.json hbm_gbs"
    return 6650.0, "fallback B200_PROFILING.md"


def ncu_traffic(workload, key):
    """DRAM bytes per launch of kernel `key` ("pattern:k<artifact>:<schedule>") from the
    committed same-workload ncu capture (tools/profile_kernels.py -> profiles/ncu_traffic.json),
    with the algorithmic bytes of the profiled launches for comparison."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        t = json.load(open(p)).get(workload, {}).get(key)
    except Exception:
        return None, None
    if not t:
        return None, None
    return t.get("dram_bytes_per_launch"), t


# ---------------------------------------------------------------------------
# Distributed plumbing

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
        if torch.cuda.is_available():
            torch.cuda.synchronize()


def allreduce(dist, local, v, op="max"):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=_dev(dist, local))
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


# ---------------------------------------------------------------------------
# Reference (CPU) side: cpu_baseline and --impl reference.  Inputs are views into a host
# pool of uniform [0.25, 2) f32 (the reference executor copies its inputs anyway).

class HostPool:
    def __init__(self, numel=1 << 27, seed=0):
        self.a = np.random.default_rng(seed).uniform(0.25, 2.0, size=numel).astype(np.float32)
        self.cursor = 0

    def inputs(self, graph, syms):
        out = {}
        for i in graph["inputs"]:
            shape = input_shape(i, syms)
            cv = const_value(i["id"], syms)
            if cv is not None:
                out[i["id"]] = np.full(shape, cv, np.float32)
                continue
            n = int(np.prod(shape))
            if self.cursor + n > self.a.size:
                self.cursor = 0
            out[i["id"]] = self.a[self.cursor:self.cursor + n].reshape(shape)
            self.cursor += (n + 63) // 64 * 64
        return out


def ref_costs(ref_plans_bytes, graphs, reqs):
    return [ref_plans_bytes[k]({i["id"]: input_shape(i, s) for i in graphs[k]["inputs"]}) for k, s in reqs]


def cpu_baseline(workload, reqs, budget_s=15.0):
    """Reference executor (oracle/_ref) on a stratified sample of one step, 1 thread."""
    from oracle import plan_bytes, ref
    if not ref.available():
        return None
    rj = {k: ref.compile(json.dumps(g)) for k, g in workload.graphs.items()}
    pb = {k: plan_bytes.PlanBytes(j) for k, j in rj.items()}
    costs = ref_costs(pb, workload.graphs, reqs)
    pick = stratified(reqs, costs, 0.16e9 * budget_s)  # ~0.16 GB/s per reference thread
    rps = {k: ref.RefPlan(j) for k, j in rj.items()}
    pool = HostPool()
    tot_b, tot_s = 0, 0.0
    for i in pick:
        kind, syms = reqs[i]
        x = pool.inputs(workload.graphs[kind], syms)
        tot_s += rps[kind].time(x, 1)
        tot_b += costs[i]
    return {"value": tot_b / max(tot_s, 1e-9) / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference",
            "sample": f"{len(pick)} of {len(reqs)} requests of the same step (stratified by pattern and size, "
                      f"{tot_b / 1e9:.2f} GB), reference Executor::run (oracle/_ref), 1 thread, {tot_s:.1f} s",
            "host": host_info()}


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU executor (oracle/_ref, built unmodified
    from /root/reference) on every host thread, over the SAME per-step request lists as the
    B200 arm (same workload, seeds and steps), each step a stratified bounded sample.
    Byte accounting comes from the reference's own plan JSON (oracle/plan_bytes.py); the
    B200 package is never imported."""
    if world > 1 and rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor
    from oracle import plan_bytes, ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    wl = make_workload(args.workload, 0, args.requests)
    nthreads = os.cpu_count() or 1
    rj = {k: ref.compile(json.dumps(g)) for k, g in wl.graphs.items()}
    pb = {k: plan_bytes.PlanBytes(j) for k, j in rj.items()}
    rps = [{k: ref.RefPlan(j) for k, j in rj.items()} for _ in range(nthreads)]
    pool = HostPool()
    step_budget = args.ref_step_s * 1.3e9 * nthreads / 16  # ~1.3 GB/s on 16 reference threads

    def step(i, budget):
        reqs = wl.requests(i)
        costs = ref_costs(pb, wl.graphs, reqs)
        pick = stratified(reqs, costs, budget, seed=i)
        inputs = [pool.inputs(wl.graphs[reqs[j][0]], reqs[j][1]) for j in pick]
        order = sorted(range(len(pick)), key=lambda j: -costs[pick[j]])  # LPT over the threads
        lanes = [[] for _ in range(nthreads)]
        load = [0] * nthreads
        for j in order:
            t = load.index(min(load))
            lanes[t].append(j)
            load[t] += costs[pick[j]]

        def work(t):
            for j in lanes[t]:
                rps[t][reqs[pick[j]][0]].time(inputs[j], 1)
        t0 = time.perf_counter()
        with ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(work, range(nthreads)))
        return time.perf_counter() - t0, sum(costs[j] for j in pick), len(pick), len(reqs)

    for i in range(args.warmup):
        step(i, step_budget / 8)
    secs = nbytes = npick = nreq = 0
    for i in range(args.warmup, args.warmup + args.steps):
        s, b, p, n = step(i, step_budget)
        secs += s
        nbytes += b
        npick += p
        nreq += n
    v = nbytes / secs / 1e9
    sample = (f"{npick} of {nreq} requests over {args.steps} steps (the B200 arm's steps {args.warmup}.."
              f"{args.warmup + args.steps - 1}; stratified by pattern and size), reference Executor::run "
              f"(oracle/_ref), {nthreads} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (uniform [0.25, 2) f32)",
        "config": {"workload": wl.desc, "requests_per_step": len(wl.requests(args.warmup)), "sample": sample},
        "host": host_info(),
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": nthreads, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ---------------------------------------------------------------------------
# Verification of a timed step's exact grouped pass (outside the timed region)

def verify_pass(B, wl, batch, mode, threads, seed=0):
    """Re-runs a timed step's batch exactly as timed (same arena inputs, chunks, grouped
    calls, host threads and flush phases), pulls inputs/outputs of the checked requests and
    hands them to the reference checker (oracle/verify.py)."""
    from oracle import verify as V
    rng = np.random.default_rng(seed)
    reqs, costs = batch.reqs, batch.costs
    if mode == "sample":  # every large request gets a chance, small ones a stratified share
        chosen = set(stratified(reqs, costs, 2e9, seed=seed))
        large_frac = 0.05
    else:
        chosen = set(range(len(reqs)))
        large_frac = 1.0
    checker = V.Checker(wl.graphs, threads=threads)
    A = B.arena

    def on_chunk(ci, a, b):
        B.L.disc_cuda_stream_synchronize(B.stream)
        for r in range(a, b):
            kind, syms = reqs[r]
            shapes = {name: shape for name, _, shape in batch.bind[r]}
            small = max((int(np.prod(s)) for s in shapes.values()), default=0) <= V.SMALL_NUMEL
            if small and r not in chosen:
                continue
            if not small and rng.random() >= large_frac:
                continue
            plan = V.check_plan(kind, shapes, True, rng)
            if plan is None:
                continue
            try:
                check_one(r, a, kind, syms, plan)
            except Exception as ex:
                raise RuntimeError(f"verify: request {r} ({kind} {syms}, mode {plan.mode}, chunk [{a},{b})): "
                                   f"{type(ex).__name__}: {ex}") from ex

    def check_one(r, a, kind, syms, plan):
        views = B.ex.request_output_views(r - a)
        picks = V.expected_output_rows(kind, plan, len(views))
        inputs, got = {}, []
        if plan.mode == "rows":
            ins, _ = V.ROW_SPEC[kind]
            for name, p, shape in batch.bind[r]:
                inputs[name] = A.d2h(p, shape, plan.pick[ins[name]]) if name in ins else A.d2h(p, shape)
            for (p, dims), rows in zip(views, picks):
                got.append(A.d2h(p, dims, rows))
        elif plan.mode == "cols":
            cols = plan.pick["c"]
            for name, p, shape in batch.bind[r]:
                full = A.d2h(p, shape)
                ax = V.COL_SPEC[kind][0].get(name)
                inputs[name] = np.ascontiguousarray(np.take(full, cols, axis=ax)) if ax is not None else full
            for (p, dims), _ in zip(views, picks):
                got.append(A.d2h(p, dims)[cols])
        else:
            for name, p, shape in batch.bind[r]:
                inputs[name] = A.d2h(p, shape)
            for p, dims in views:
                got.append(A.d2h(p, dims))
        B.L.disc_cuda_stream_synchronize(B.stream)
        checker.submit(f"{kind} {syms}", kind, plan.mode, inputs, got)

    batch.run(B.ex, on_chunk=on_chunk)
    out = checker.finish()
    out["mode"] = mode
    out["step_requests"] = len(reqs)
    return out


# ---------------------------------------------------------------------------
# e2e: public C ABI with host buffers

def measure_e2e(B, wl, reqs, costs, budget_bytes, pipes=3, chunk_bytes=256 << 20):
    """disc_executor_run_grouped(inputs_on_host=1) over a stratified sample of the step
    (pinned host inputs, ~budget_bytes of input), outputs D2H into pinned host memory with
    disc_executor_copy_request_output; chunks alternate over `pipes` executors/streams so
    one chunk's H2D overlaps another's kernels and D2H.  Wall time of one pass."""
    D, L = B.D, B.L
    g = wl.graphs
    in_bytes = [sum(4 * int(np.prod(input_shape(i, s))) for i in g[k]["inputs"]) for k, s in reqs]
    pick = stratified(reqs, in_bytes, budget_bytes, seed=1)
    sub = [reqs[i] for i in pick]
    scost = [costs[i] for i in pick]
    B.plans_for(sub)
    exs, streams = [], []
    for _ in range(pipes):
        st = C.c_void_p()
        D.api._cuda(L.disc_cuda_stream_create(C.byref(st)))
        streams.append(st)
        e = D.Executor(B.local, st.value)
        e.set_host_threads(max(1, B.args.host_threads // 2))
        exs.append(e)
    pinned, work = [], []
    rng = np.random.default_rng(1)
    h2d = 0
    for kind, syms in sub:
        ptrs, dims = [], []
        for i in g[kind]["inputs"]:
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
        work.append((B.plans[kind], [i["id"] for i in g[kind]["inputs"]], ptrs, dims))
    chunks, cur, acc = [], [], 0
    for r, c in enumerate(scost):
        cur.append(r)
        acc += c
        if acc >= chunk_bytes:
            chunks.append(cur)
            cur, acc = [], 0
    if cur:
        chunks.append(cur)
    cargs, keep = [], []
    for ch in chunks:
        names, datas, dimsp, ranks, offs, hplans = [], [], [], [], [0], []
        for r in ch:
            plan, nm, ptrs, dims = work[r]
            names += [s.encode() for s in nm]
            datas += ptrs
            dimsp += [d.ctypes.data for d in dims]
            ranks += [d.size for d in dims]
            offs.append(offs[-1] + len(nm))
            hplans.append(plan._h)
        t = max(len(names), 1)
        a = (len(ch), (C.c_void_p * len(ch))(*hplans), (C.c_int * (len(ch) + 1))(*offs), (C.c_char_p * t)(*names),
             (C.c_void_p * t)(*datas), (C.c_void_p * t)(*dimsp), (C.c_int * t)(*ranks))
        cargs.append(a)
    outs = {}

    def out_buf(key, n):
        if key not in outs:
            p = C.c_void_p()
            D.api._cuda(L.disc_cuda_host_alloc(max(4 * n, 16), C.byref(p)))
            outs[key] = p
        return outs[key]

    d2h = 0

    def one_pass():
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

    one_pass()  # warm allocators, staging and recipes
    t0 = time.perf_counter()
    one_pass()
    dt = time.perf_counter() - t0
    for p in pinned + list(outs.values()):
        L.disc_cuda_host_free(p)
    del exs
    nbytes = sum(scost)
    return {"value": round(nbytes / dt / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(dt * 1e3, 3), "requests": len(sub),
            "sample": f"{len(sub)} of {len(reqs)} requests of a timed step (stratified by pattern and size)",
            "path": f"disc_executor_run_grouped(inputs_on_host=1) per chunk (~{chunk_bytes >> 20} MB of algorithmic "
                    f"bytes, {len(chunks)} chunks) + disc_executor_copy_request_output(pinned host, async), chunks "
                    f"alternating over {pipes} executors/streams",
            "bytes": nbytes, "seconds": dt}


# ---------------------------------------------------------------------------

def pattern_of(kind):
    return kind if kind in MAIN_KINDS else "fixtures"


def analyse(B, wl, reqs, costs, peak):
    """Untimed analysis of one step: per-pattern device-bound GB/s (all and large requests;
    each pass issued behind a spin kernel, so it is the kernels' rate, not the host's),
    per-kernel records keyed (pattern, artifact, schedule), the dominant kernel, and the
    device-only time of the whole step."""
    pats = {}
    for i, (k, _) in enumerate(reqs):
        pats.setdefault(pattern_of(k), []).append(i)
    per_pattern, records = {}, {}
    for p, idx in sorted(pats.items()):
        sub, sc = [reqs[i] for i in idx], [costs[i] for i in idx]
        ms, _ = B.device_bound_pass(B.batch(sub, sc))
        b = sum(sc)
        ent = {"requests": len(sub), "bytes": b, "GB/s": round(b / ms / 1e6, 1) if ms > 0 else None}
        ent["frac_of_peak"] = round(ent["GB/s"] / peak, 4) if ent["GB/s"] else None
        big = [i for i in idx if costs[i] >= LARGE]
        if big:
            lb = sum(costs[i] for i in big)
            lms, _ = B.device_bound_pass(B.batch([reqs[i] for i in big], [costs[i] for i in big]))
            ent["large"] = {"requests": len(big), "bytes": lb, "GB/s": round(lb / lms / 1e6, 1) if lms > 0 else None}
            ent["large"]["frac_of_peak"] = round(ent["large"]["GB/s"] / peak, 4) if ent["large"]["GB/s"] else None
            ent["large_byte_share"] = round(lb / b, 4) if b else None
        per_pattern[p] = ent
        # per-kernel records keyed (graph, plan kernel, schedule): one timing pass per graph
        kinds = sorted({reqs[i][0] for i in idx})
        for kind in kinds:
            kidx = [i for i in idx if reqs[i][0] == kind]
            for r in B.record_pass(B.batch([reqs[i] for i in kidx], [costs[i] for i in kidx])):
                key = f"{kind}:k{r['kernel']}:{r['schedule']}"
                a = records.setdefault(key, [0, 0.0, 0])
                a[0] += r["bytes"]
                a[1] += r["ms"]
                a[2] += 1
    # the generic path: the same passes with the generated kernels off (tape interpreter)
    B.D.set_specialization(False)
    try:
        for p, idx in sorted(pats.items()):
            sub, sc = [reqs[i] for i in idx], [costs[i] for i in idx]
            ms, _ = B.device_bound_pass(B.batch(sub, sc))
            per_pattern[p]["generic_GBps"] = round(sum(sc) / ms / 1e6, 1) if ms > 0 else None
            if per_pattern[p].get("GB/s"):
                per_pattern[p]["generic_over_generated"] = round(per_pattern[p]["generic_GBps"] / per_pattern[p]["GB/s"], 3)
    finally:
        B.D.set_specialization(True)
    full = B.record_pass(B.batch(reqs, costs))
    device_bound_ms, host_issue_ms = B.device_bound_pass(B.batch(reqs, costs))
    return per_pattern, records, device_bound_ms, host_issue_ms, len(full)


def random_graph_rate(B, peak, per_graph=5, max_numel=1 << 22, seed=7):
    """Arbitrary graphs (the reference's RandomGraphGen graphs committed in
    tests/golden/random_plans.json.gz, 200 seeds) at random shapes: device-bound GB/s of one
    grouped pass and the share of fused launches that found a generated kernel (the rest
    run the tape interpreter).  Shapes: each symbol log-uniform, inputs <= max_numel; a
    binding the runtime flow would reject (host dry run) is redrawn."""
    import gzip
    import random
    D = B.D
    gr = json.load(gzip.open(os.path.join(ROOT, "tests", "golden", "random_plans.json.gz"), "rt"))
    rng = random.Random(seed)
    comp = D.Compiler()
    reqs_g, reqs = {}, []
    for key in sorted(gr, key=int):
        g = json.loads(gr[key]["graph"]) if isinstance(gr[key]["graph"], str) else gr[key]["graph"]
        plan = comp.compile(g)
        syms = sorted({d for i in g["inputs"] for d in i["shape"] if isinstance(d, str)})
        got = 0
        for _ in range(per_graph * 8):
            if got == per_graph:
                break
            v = {x: W()._logu(rng, 1, 4096) for x in syms}
            shapes = {i["id"]: input_shape(i, v) for i in g["inputs"]}
            if max((int(np.prod(sh)) for sh in shapes.values()), default=0) > max_numel:
                continue
            try:
                D.group_dry_run([(plan, shapes)])
            except D.DiscError:
                continue
            kind = f"rg{key}"
            reqs_g[kind] = g
            reqs.append((kind, v))
            B.plans[kind] = plan
            got += 1
    saved = B.wl.graphs
    B.wl.graphs = dict(saved, **reqs_g)
    try:
        batch = B.batch(reqs)
        B.device_bound_pass(batch)  # warm
        s0, f0 = D.lib().disc_cuda_specialized_launches(), D.lib().disc_cuda_fused_launches()
        ms, _ = B.device_bound_pass(batch)
        s1, f1 = D.lib().disc_cuda_specialized_launches(), D.lib().disc_cuda_fused_launches()
    finally:
        B.wl.graphs = saved
    gbs = batch.bytes / ms / 1e6 if ms > 0 else None
    return {"graphs": len(reqs_g), "requests": len(reqs), "bytes": batch.bytes, "GB/s": round(gbs, 1) if gbs else None,
            "frac_of_peak": round(gbs / peak, 4) if gbs else None,
            "generated_frac": round((s1 - s0) / max(1, f1 - f0), 4),
            "source": "tests/golden/random_plans.json.gz (reference RandomGraphGen seeds 0-199), symbols log-uniform 1..4096"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="disc", choices=["disc", "reference"])
    ap.add_argument("--workload", default="sweep")
    ap.add_argument("--requests", type=int, default=10000, help="sweep: distinct requests per step")
    ap.add_argument("--verify", default="sample", choices=["off", "sample", "full"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-analysis", action="store_true")
    ap.add_argument("--schedule", default="auto")
    # A/B s7 on B200 (sweep): 32 GB 4441, 64 GB 4675, 128 GB 4818 GB/s -- fewer grouped calls,
    # fewer level boundaries (kernel tails) per step
    ap.add_argument("--chunk-gb", type=float, default=128.0, help="algorithmic bytes per grouped call")
    ap.add_argument("--arena-gb", type=float, default=48.0)
    ap.add_argument("--cache-gb", type=float, default=32.0, help="executor idle device-memory budget (caches + arena)")
    ap.add_argument("--async-flush", type=int, default=1, choices=[0, 1],
                    help="issue grouped launches from a background thread (flows of the next chunk overlap)")
    ap.add_argument("--reserve-gb", type=float, default=120.0, help="executor buffer arena reserved up front")
    ap.add_argument("--e2e-gb", type=float, default=4.0, help="e2e: pinned host input bytes")
    ap.add_argument("--e2e-pipes", type=int, default=8, help="e2e: executors/streams the chunks alternate over")
    ap.add_argument("--e2e-chunk-mb", type=int, default=64, help="e2e: algorithmic MB per grouped call")
    ap.add_argument("--ref-step-s", type=float, default=4.0, help="reference arm: seconds of CPU work per step")
    ap.add_argument("--host-threads", type=int, default=0,
                    help="host threads per rank for the runtime flows (0: cores / ranks, max 32)")
    ap.add_argument("--pdl", type=int, default=1, choices=[0, 1, 2])
    ap.add_argument("--host-only", action="store_true",
                    help="capture mode (no device): time the host side (runtime flows + flush) of every step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world, rank, local, dist = dist_setup(args)
    if args.host_threads <= 0:
        args.host_threads = max(1, min(32, (os.cpu_count() or 1) // max(1, world)))
    if args.impl == "reference":
        run_reference(args, world, rank)
        if dist is not None:
            dist.destroy_process_group()
        return

    import paper_2103_05288_b200 as D
    D.lib()
    D.set_pdl(args.pdl)
    if args.host_only:
        D.lib().disc_cuda_set_capture(2)
    if args.workload == "sweep":
        wl = make_workload("sweep", rank, args.requests)
        shard = None
    else:
        from paper_2103_05288_b200.dispatch import shard as lpt
        wl = make_workload(args.workload, 0)
        reqs_all = list(wl.requests(0))
        for r in range(1, world):  # N replicas of the sweep, LPT-sharded below
            w2 = make_workload(args.workload, r)
            wl.graphs.update(w2.graphs)
            reqs_all += w2.requests(0)
        shard = (lpt, reqs_all)
    B = Bench(D, args, local, wl)
    if shard is not None:
        lpt, reqs_all = shard
        B.plans_for(reqs_all)
        costs_all = B.costs(reqs_all)
        mine = lpt(costs_all, world)[rank]
        fixed = [reqs_all[i] for i in mine]
        wl = Workload(wl.name, wl.desc, wl.graphs, fixed=fixed)
        B.wl = wl

    # all steps' batches are built before the timed region (the request list is the input)
    t0 = time.perf_counter()
    batches = []
    for i in range(args.warmup + args.steps):
        reqs = wl.requests(i)
        batches.append(B.batch(reqs))
        if not wl.fresh:
            batches += [batches[0]] * (args.warmup + args.steps - 1)
            break
    log(f"[bench] {len(batches)} step batches built in {time.perf_counter() - t0:.1f}s "
        f"({len(wl.requests(0))} requests/step, {batches[0].bytes / 1e9:.1f} GB/step, {len(batches[0].chunks)} chunks)")
    L = B.L
    if args.host_only:
        for i, b in enumerate(batches):
            t1 = time.perf_counter()
            b.run(B.ex)
            log(f"[bench host-only] step {i}: {len(b.reqs)} requests, {len(b.chunks)} chunks, host "
                f"{(time.perf_counter() - t1) * 1e3:.1f} ms ({(time.perf_counter() - t1) / max(1, len(b.reqs)) * 1e6:.2f} "
                f"us/request), {b.bytes / 1e9:.1f} GB")
        return
    for i in range(args.warmup):
        batches[i].run(B.ex)
        L.disc_cuda_stream_synchronize(B.stream)
    D.api._cuda(L.disc_cuda_device_synchronize())

    # ---- timed region: K steps issued back to back; per step an event pair (the L2 flush
    # before it outside the pair); host flow of step i+1 overlaps device work of step i ----
    ev = [B.event() for _ in range(2 * args.steps)]
    call_ms = []
    al0 = alloc_stats(D)
    cpu0 = cpu_times()
    spec0, fused0 = D.lib().disc_cuda_specialized_launches(), D.lib().disc_cuda_fused_launches()
    launches0 = D.kernel_launches()
    barrier(dist, local)
    wall0 = time.perf_counter()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            L.disc_cuda_flush_l2(B.flush, B.flush_bytes, B.stream)
            L.disc_cuda_event_record(ev[2 * i], B.stream)
            batches[args.warmup + i].run(B.ex, call_ms=call_ms)
            L.disc_cuda_event_record(ev[2 * i + 1], B.stream)
        L.disc_cuda_stream_synchronize(B.stream)
    wall = time.perf_counter() - wall0
    al1 = alloc_stats(D)
    cpu1 = cpu_times()
    spec1, fused1 = D.lib().disc_cuda_specialized_launches(), D.lib().disc_cuda_fused_launches()
    host_diag = {"grouped_calls": len(call_ms), "call_ms_sum": round(sum(call_ms), 2),
                 "call_ms_max": round(max(call_ms), 2) if call_ms else None,
                 "call_ms_p50": round(statistics.median(call_ms), 2) if call_ms else None,
                 "pool_mallocs": al1[0] - al0[0], "pool_frees": al1[1] - al0[1], "oom_retries": al1[2] - al0[2],
                 "cpu_steal_frac": cpu_steal(cpu0, cpu1),
                 "fused_launches": fused1 - fused0, "generated_frac": round((spec1 - spec0) / max(1, fused1 - fused0), 4)}
    mal = [b - a for a, b in zip([al0[0]] + call_ms_mallocs[:-1], call_ms_mallocs)]
    slow = sorted(range(len(call_ms)), key=lambda k: -call_ms[k])[:6]
    host_diag["slowest_calls"] = [(k, round(call_ms[k], 1), mal[k]) for k in slow]
    log(f"[bench] host: {host_diag}")
    step_ms = []
    for i in range(args.steps):
        ms = C.c_float()
        L.disc_cuda_event_elapsed_ms(ev[2 * i], ev[2 * i + 1], C.byref(ms))
        step_ms.append(ms.value)
    gpu_launches = D.kernel_launches() - launches0 - args.steps
    my_bytes = sum(batches[args.warmup + i].bytes for i in range(args.steps))
    barrier(dist, local)
    total_ms = allreduce(dist, local, sum(step_ms), "max")
    total_bytes = allreduce(dist, local, my_bytes, "sum")
    ms_per_step = total_ms / args.steps
    value = total_bytes / (total_ms / 1e3) / 1e9
    compile_count = B.compiler.stats()["compile_count"]
    distinct = len({(k, tuple(sorted(s.items()))) for i in range(args.warmup + args.steps) for k, s in wl.requests(i)})
    peak, peak_src = peaks()
    clocks = clk.summary()
    log(f"[bench] timed: {value:.1f} GB/s ({value / world / peak:.3f} of peak), {ms_per_step:.2f} ms/step, "
        f"{total_bytes / args.steps / 1e9:.1f} GB/step, {distinct} distinct shapes, clocks {clocks}")

    # ---- untimed: analysis of the first timed step ----
    reqs0 = wl.requests(args.warmup)
    costs0 = batches[args.warmup].costs
    analysis = None
    if not args.no_analysis:
        per_pattern, records, device_ms, host_issue_ms, n_group_launches = analyse(B, wl, reqs0, costs0, peak)
        (dk, (db, dms, dn)) = max(records.items(), key=lambda kv: kv[1][1])
        achieved = db / (dms / 1e3) / 1e9 if dms > 0 else 0.0
        traffic, tinfo = ncu_traffic(wl.name, dk)
        tot_ms = sum(v[1] for v in records.values())
        breakdown = {k: {"GB/s": round(b / (ms / 1e3) / 1e9, 1) if ms else None,
                         "share": round(ms / tot_ms, 3) if tot_ms else None, "launches": n}
                     for k, (b, ms, n) in sorted(records.items(), key=lambda kv: -kv[1][1])[:16]}
        analysis = {
            "per_pattern": per_pattern,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dk,
                         "peak_source": peak_src, "bytes_per_launch": db // max(dn, 1),
                         "mean_launch_ms": round(dms / max(dn, 1), 5),
                         "traffic_source": (f"profiles/ncu_traffic.json[{wl.name}][{dk}]: ncu dram bytes of the same "
                                            f"kernel, algorithmic {tinfo.get('alg_bytes_per_launch')} B/launch there")
                         if tinfo else "no committed ncu capture for this (workload, kernel)"},
            "kernel_breakdown": breakdown,
            "random_graphs": random_graph_rate(B, peak),
            "device_ms_step": round(device_ms, 3),
            "host_issue_ms_step": round(host_issue_ms, 3),
            "grouped_launches_step": n_group_launches,
        }

    out = None
    ver = None
    if args.verify != "off" and rank == 0:
        from oracle import ref as _ref
        if _ref.available():
            ver = verify_pass(B, wl, batches[args.warmup], args.verify, threads=max(1, (os.cpu_count() or 2) - 1))
    e2e = None
    if not args.no_e2e:
        B.release()  # the timed passes' reserved arena (120 GB) and device inputs: e2e stages its own
        e2e = measure_e2e(B, wl, reqs0, costs0, int(args.e2e_gb * (1 << 30)), pipes=args.e2e_pipes,
                          chunk_bytes=int(args.e2e_chunk_mb) << 20)
        if dist is not None:
            e2e["value"] = round(allreduce(dist, local, e2e["bytes"], "sum") /
                                 allreduce(dist, local, e2e["seconds"], "max") / 1e9, 2)
    if rank == 0:
        cpu = None if args.no_cpu_baseline or world > 1 else cpu_baseline(wl, reqs0)
        big = {p: e.get("large", {}).get("frac_of_peak") for p, e in (analysis or {}).get("per_pattern", {}).items()
               if p in MAIN_KINDS}
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (uniform [0.25, 2) f32 device arena; inputs resident in HBM)",
            "config": {"workload": wl.desc, "workload_name": wl.name,
                       "distinct_shapes": distinct, "requests_per_step": len(reqs0),
                       "fresh_shapes_every_step": wl.fresh, "graphs": len(wl.graphs),
                       "bytes_per_step": int(total_bytes / args.steps),
                       "l2": "flushed before each step (4x L2 write); inputs >> L2",
                       "parallelism": f"request-sharded x{world} (no collectives)",
                       "chunk_gb": args.chunk_gb, "host_threads": args.host_threads, "pdl": args.pdl,
                       "async_flush": args.async_flush,
                       "schedule": args.schedule},
            "frac_of_hbm_peak": round(value / world / peak, 4),
            "compile_count": compile_count, "recompiles": compile_count - len(wl.graphs),
            "large_shape_frac_of_peak": big,
            "roofline": (analysis or {}).get("roofline"),
            "per_pattern": (analysis or {}).get("per_pattern"),
            "generic_GBps": {p: e.get("generic_GBps") for p, e in ((analysis or {}).get("per_pattern") or {}).items()},
            "random_graphs": (analysis or {}).get("random_graphs"),
            "kernel_breakdown": (analysis or {}).get("kernel_breakdown"),
            "device_ms_per_step": (analysis or {}).get("device_ms_step"),
            "host_issue_ms_per_step": (analysis or {}).get("host_issue_ms_step"),
            "host_bound_frac": round(max(0.0, 1 - analysis["device_ms_step"] / ms_per_step), 3) if analysis else None,
            "cpu_baseline": cpu,
            "e2e": {k: v for k, v in e2e.items() if k not in ("bytes", "seconds")} if e2e else None,
            "verify": ver,
            "gpu_launches": gpu_launches,
            "host_diag": host_diag,
            "clocks": clocks,
            "host": host_info(),
            "wall_s_timed": round(wall, 3),
        }
        print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
