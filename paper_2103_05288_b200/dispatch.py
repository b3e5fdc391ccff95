"""Multi-GPU request dispatcher: independent variable-shape requests are
sharded across the GPUs of one box with no collective on the data path -- a request
(plan + inputs) is self-contained and the path has no cross-request reduction.

* ``shard(costs, world)``: deterministic greedy LPT (largest request first, to the rank
  with the least assigned bytes, lowest rank on ties).  Every rank of a multi-process
  job computes the same assignment locally, so no exchange is needed (bench.py under
  torchrun, or any one-process-per-GPU deployment).
* ``Dispatcher``: the in-process form -- one worker thread per device, each with its own
  executor (device caching allocator) and stream; requests go to the device with the
  least outstanding algorithmic bytes (round-robin tie-break).  Plans are shared
  read-only across devices (kernels take the lowered program by value, so there is no
  per-device upload); the compiler cache is shared too.

Costs are the requests' algorithmic boundary bytes (``CompiledPlan.algorithmic_bytes``,
computed on the host from the shape program, no device work).
"""
from __future__ import annotations

import ctypes as C
import heapq
import queue
import threading
from concurrent.futures import Future
from typing import Dict, List, Optional, Sequence, Tuple

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


class _Worker(threading.Thread):
    def __init__(self, device: int):
        super().__init__(daemon=True, name=f"disc-gpu{device}")
        self.device = device
        self.q: "queue.Queue" = queue.Queue()
        self.ready = threading.Event()
        self.error: Optional[BaseException] = None
        self.start()

    def run(self):
        try:
            L = api.lib()
            api._cuda(L.disc_cuda_set_device(self.device), "set device")
            self.stream = C.c_void_p()
            api._cuda(L.disc_cuda_stream_create(C.byref(self.stream)), "stream create")
            self.ex = api.Executor(self.device, self.stream.value)
        except BaseException as e:  # surfaced by submit()
            self.error = e
            self.ready.set()
            return
        self.ready.set()
        while True:
            item = self.q.get()
            if item is None:
                break
            fn, fut, done = item
            if not fut.set_running_or_notify_cancel():
                done()
                continue
            try:
                fut.set_result(fn(self.ex))
            except BaseException as e:
                fut.set_exception(e)
            finally:
                done()
        self.ex = None
        api.lib().disc_cuda_stream_destroy(self.stream)


class Dispatcher:
    """Routes requests to per-device workers by least outstanding bytes.

    ``submit(plan, inputs)`` returns a Future of the ExecResult (host outputs);
    ``map(requests)`` runs a list of (plan, inputs) and returns the results in order.
    """

    def __init__(self, devices: Optional[Sequence[int]] = None):
        if devices is None:
            n = C.c_int()
            api._cuda(api.lib().disc_cuda_device_count(C.byref(n)), "device count")
            devices = list(range(n.value))
        if not devices:
            raise api.DiscError(4, "no CUDA device available", "runtime")
        self.devices = list(devices)
        self._workers = [_Worker(d) for d in self.devices]
        for w in self._workers:
            w.ready.wait()
            if w.error is not None:
                raise w.error
        self._lock = threading.Lock()
        self._outstanding = [0] * len(self.devices)
        self._next = 0
        self.assigned = [0] * len(self.devices)  # requests routed per device (stats)

    def _pick(self, nbytes: int) -> int:
        with self._lock:
            n = len(self._outstanding)
            best = min(self._outstanding)
            for k in range(n):  # round-robin among the least loaded
                i = (self._next + k) % n
                if self._outstanding[i] == best:
                    break
            self._next = (i + 1) % n
            self._outstanding[i] += nbytes
            self.assigned[i] += 1
            return i

    def _release(self, i: int, nbytes: int) -> None:
        with self._lock:
            self._outstanding[i] -= nbytes

    def submit(self, plan: "api.CompiledPlan", inputs: Dict[str, object], nbytes: Optional[int] = None) -> Future:
        nb = request_bytes(plan, inputs) if nbytes is None else int(nbytes)
        i = self._pick(nb)
        fut: Future = Future()
        self._workers[i].q.put((lambda ex: ex.run(plan, inputs), fut, lambda: self._release(i, nb)))
        return fut

    def map(self, requests: Sequence[Tuple["api.CompiledPlan", Dict[str, object]]]) -> list:
        futs = [self.submit(p, x) for p, x in requests]
        return [f.result() for f in futs]

    def close(self) -> None:
        for w in self._workers:
            w.q.put(None)
        for w in self._workers:
            w.join()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
