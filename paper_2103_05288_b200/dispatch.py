"""Multi-GPU request dispatcher: independent variable-shape requests are
sharded across the GPUs of one box with no collective on the data path -- a request
(plan + inputs) is self-contained and the path has no cross-request reduction.

* ``shard(costs, world)``: deterministic greedy LPT (largest request first, to the rank
  with the least assigned bytes, lowest rank on ties).  Every rank of a multi-process
  job computes the same assignment locally, so no exchange is needed (bench.py under
  torchrun, or any one-process-per-GPU deployment).
* ``Dispatcher``: the in-process form over the native dispatcher (csrc/capi_dispatch.cpp)
  -- one C++ worker thread per device, each with its own executor (caching allocator,
  buffer arena, host-flow threads) and stream, pinned to its own CPU slice; a batch is
  split by the same LPT rule and each worker runs its share as one grouped call.  Plans
  are shared read-only across devices (kernels take the lowered program by value, so there
  is no per-device upload); the compiler cache is shared too.

Costs are the requests' algorithmic boundary bytes (``CompiledPlan.algorithmic_bytes``,
computed on the host from the shape program, no device work).
"""
from __future__ import annotations

import ctypes as C
import heapq
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import api


def shard(costs: Sequence[int], world: int) -> List[List[int]]:
    """Request indices per rank (each rank's list in original request order)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-int(costs[i]), i))
    heap = [(0, r) for r in range(world)]
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + int(costs[i]), r))
    for lst in out:
        lst.sort()
    return out


def shard_loads(costs: Sequence[int], parts: List[List[int]]) -> List[int]:
    return [sum(int(costs[i]) for i in p) for p in parts]


def request_bytes(plan: "api.CompiledPlan", inputs: Dict[str, object]) -> int:
    import numpy as np
    shapes = {k: tuple(v.shape) if hasattr(v, "shape") else np.shape(v) for k, v in inputs.items()}
    return plan.algorithmic_bytes(shapes)


class Dispatcher:
    """In-process multi-GPU dispatcher over the native one (disc_dispatcher_*,
    csrc/capi_dispatch.cpp): one C++ worker thread per device entry, each with its own
    executor, stream and host-flow threads, pinned to its own slice of the process's CPUs.
    A batch is split by greedy LPT on algorithmic bytes (the rule of ``shard``) and each
    worker runs its share as one grouped call.

    ``map(requests)`` runs (plan, inputs) pairs (host numpy inputs) and returns an
    ExecResult-like object per request, in order; ``run_grouped`` leaves the outputs
    device-resident (``request_output`` / ``fetch``)."""

    def __init__(self, devices: Optional[Sequence[int]] = None, host_threads: int = 0):
        L = api.lib()
        if devices is None:
            n = C.c_int()
            api._cuda(L.disc_cuda_device_count(C.byref(n)), "device count")
            devices = list(range(n.value))
        if not devices:
            raise api.DiscError(4, "no CUDA device available", "runtime")
        self.devices = list(devices)
        self._h = C.c_void_p()
        api._check(L.disc_dispatcher_create(len(self.devices), (C.c_int * len(self.devices))(*self.devices),
                                            int(host_threads), C.byref(self._h)))
        self.assigned = [0] * len(self.devices)  # requests routed per worker (all batches)
        self._n = 0

    def _flat(self, requests):
        keep, names, datas, dims, ranks, offs, plans = [], [], [], [], [], [0], []
        for plan, inputs in requests:
            for k, v in inputs.items():
                a = np.ascontiguousarray(np.asarray(v, dtype=np.float32))
                d = np.array(a.shape, dtype=np.int64)
                keep += [a, d]
                names.append(k.encode())
                datas.append(a.ctypes.data if a.size else 0)
                dims.append(d.ctypes.data)
                ranks.append(d.size)
            offs.append(len(names))
            plans.append(plan._h)
        t, n = max(len(names), 1), max(len(requests), 1)
        return keep, ((C.c_void_p * n)(*plans), (C.c_int * (len(requests) + 1))(*offs), (C.c_char_p * t)(*names),
                      (C.c_void_p * t)(*datas), (C.c_void_p * t)(*dims), (C.c_int * t)(*ranks))

    def assign(self, requests) -> List[int]:
        """Worker of each request under the LPT rule (host only)."""
        keep, (plans, offs, names, _, dims, ranks) = self._flat(requests)
        out = (C.c_int * max(len(requests), 1))()
        api._check(api.lib().disc_dispatcher_assign(self._h, len(requests), plans, offs, names, dims, ranks, out))
        return list(out)[:len(requests)]

    def run_grouped(self, requests: Sequence[Tuple["api.CompiledPlan", Dict[str, object]]]) -> None:
        keep, (plans, offs, names, datas, dims, ranks) = self._flat(requests)
        L = api.lib()
        api._check(L.disc_dispatcher_run_grouped(self._h, len(requests), plans, offs, names, datas, dims, ranks, 1,
                                                 None))
        self._n = len(requests)
        for r in range(self._n):
            self.assigned[L.disc_dispatcher_request_worker(self._h, r)] += 1

    def worker_of(self, r: int) -> int:
        return api.lib().disc_dispatcher_request_worker(self._h, r)

    def fetch(self, r: int) -> List[np.ndarray]:
        """Host copies of request r's outputs (last batch)."""
        L = api.lib()
        out = []
        for i in range(L.disc_dispatcher_num_request_outputs(self._h, r)):
            p, d, k, dev = C.c_void_p(), C.POINTER(C.c_int64)(), C.c_int(), C.c_int()
            api._check(L.disc_dispatcher_request_output(self._h, r, i, C.byref(p), C.byref(d), C.byref(k),
                                                        C.byref(dev)))
            a = np.empty(tuple(d[j] for j in range(k.value)), dtype=np.float32)
            if a.size:
                api._check(L.disc_dispatcher_copy_request_output(self._h, r, i, C.c_void_p(a.ctypes.data), 1))
            out.append(a)
        return out

    def worker_stats(self) -> List[Dict[str, float]]:
        L = api.lib()
        res = []
        for w in range(len(self.devices)):
            n, b, ms = C.c_int64(), C.c_int64(), C.c_double()
            api._check(L.disc_dispatcher_worker_stats(self._h, w, C.byref(n), C.byref(b), C.byref(ms)))
            res.append({"device": self.devices[w], "requests": n.value, "bytes": b.value, "ms": ms.value})
        return res

    def map(self, requests: Sequence[Tuple["api.CompiledPlan", Dict[str, object]]]) -> list:
        self.run_grouped(requests)
        return [_Result(self.fetch(r), self.devices[self.worker_of(r)]) for r in range(len(requests))]

    def close(self) -> None:
        if self._h:
            api.lib().disc_dispatcher_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class _Result:
    def __init__(self, outputs, device):
        self.outputs, self.device = outputs, device
