"""Python host API over libdisc_b200.so (C ABI: include/disc_b200.h, include/disc_cuda.h).

Mirrors the reference's C++ surface (proj/include/disc/*.hpp) so tests read like the
reference's own:  ``compile_graph``, ``static_specialize``, ``Compiler`` (plan cache),
``CompiledPlan`` (plan JSON round trip, check_plan), ``Executor.run`` -> ``ExecResult``
(outputs, ``ExecStats``, ``buffer_events``), ``Executor.run_kernel`` and ``guard_passes``.
Errors raise ``DiscError`` carrying the reference's error class and message.

The product path is the CUDA library only: there is no CPU fallback, and loading fails
loudly if the extension has not been built.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libdisc_b200.so")
# A/B experiments (tools/ab_*.sh): an alternative in-tree build of the same library
if os.environ.get("DISC_LIB_VARIANT"):
    LIB_PATH = os.path.join(os.path.dirname(LIB_PATH), f"libdisc_b200_{os.environ['DISC_LIB_VARIANT']}.so")
_lib: Optional[C.CDLL] = None

ERROR_CLASSES = ("usage", "parse", "validation", "compile", "runtime", "internal")
STAT_KEYS = ("launch_count", "library_calls", "host_instruction_count", "peak_bytes",
             "alloc_calls", "allocator_cache_hits", "aliased_allocs")


class DiscError(RuntimeError):
    """error[<class>]: <message>; .code is the reference CLI exit code (2/3/4)."""

    def __init__(self, code: int, message: str, error_class: str):
        super().__init__(message)
        self.code = code
        self.error_class = error_class


def _declare(L: C.CDLL) -> None:
    vp, cp, i32, i64 = C.c_void_p, C.c_char_p, C.c_int, C.c_int64
    P = C.POINTER
    sig = {
        "disc_last_error": ([], cp), "disc_last_error_class": ([], i32), "disc_free": ([vp], None),
        "disc_version": ([], cp),
        "disc_compile_graph": ([cp, i32, i32, i32, P(vp)], i32),
        "disc_static_specialize": ([cp, P(vp)], i32),
        "disc_compiler_create": ([i32, i32, i32, P(vp)], i32),
        "disc_compiler_destroy": ([vp], None),
        "disc_compiler_compile": ([vp, cp, P(vp)], i32),
        "disc_compiler_stats": ([vp, P(i64), P(i64)], None),
        "disc_cache_key": ([cp, i32, i32, i32, P(vp)], i32),
        "disc_dump_stage": ([cp, i32, i32, cp, P(vp)], i32),
        "disc_lower_dhlo_json": ([cp, P(vp)], i32),
        "disc_dhlo_roundtrip": ([cp, P(vp)], i32),
        "disc_plan_from_json": ([cp, P(vp)], i32),
        "disc_plan_to_json": ([vp, P(vp)], i32),
        "disc_plan_check": ([vp, P(vp)], i32),
        "disc_plan_retain": ([vp], None), "disc_plan_release": ([vp], None),
        "disc_plan_num_inputs": ([vp], i32), "disc_plan_input_name": ([vp, i32], cp),
        "disc_plan_input_rank": ([vp, i32], i32),
        "disc_plan_num_outputs": ([vp], i32), "disc_plan_output_name": ([vp, i32], cp),
        "disc_plan_num_kernels": ([vp], i32),
        "disc_plan_eager_op_count": ([vp], i64), "disc_plan_host_instruction_count": ([vp], i64),
        "disc_plan_eval_shapes": ([vp, i32, P(vp), P(i32), P(i64), i32, P(i32)], i32),
        "disc_executor_create": ([i32, vp, P(vp)], i32),
        "disc_executor_destroy": ([vp], None),
        "disc_executor_set_stream": ([vp, vp], i32),
        "disc_executor_run": ([vp, vp, i32, P(cp), P(vp), P(vp), P(i32), i32], i32),
        "disc_executor_run_batch": ([vp, vp, i32, i32, P(cp), P(vp), P(vp), P(i32), i32], i32),
        "disc_executor_run_stream": ([vp, i32, P(vp), P(i32), P(cp), P(vp), P(vp), P(i32), i32], i32),
        "disc_plan_algorithmic_bytes": ([vp, i32, P(cp), P(vp), P(i32), P(i64)], i32),
        "disc_executors_run_interleaved": ([P(vp), i32, i32, P(i32), P(vp), P(i32), P(cp), P(vp), P(vp), P(i32), i32],
                                           i32),
        "disc_cuda_stream_wait_event": ([vp, vp], i32),
        "disc_executor_run_grouped": ([vp, i32, P(vp), P(i32), P(cp), P(vp), P(vp), P(i32), i32], i32),
        "disc_executor_num_requests": ([vp], i32),
        "disc_executor_set_host_threads": ([vp, i32], i32),
        "disc_executor_set_graphs": ([vp, i32], i32),
        "disc_executor_graph_replays": ([vp], i64),
        "disc_executor_num_request_outputs": ([vp, i32], i32),
        "disc_executor_request_output": ([vp, i32, i32, P(vp), P(P(i64)), P(i32)], i32),
        "disc_executor_copy_request_output": ([vp, i32, i32, vp, i32], i32),
        "disc_executor_request_stats": ([vp, i32, P(i64)], i32),
        "disc_cuda_queue_active": ([], i32),
        "disc_executor_num_outputs": ([vp], i32),
        "disc_executor_output": ([vp, i32, P(vp), P(P(i64)), P(i32)], i32),
        "disc_executor_copy_output": ([vp, i32, vp, i32], i32),
        "disc_executor_synchronize": ([vp], i32),
        "disc_executor_stats": ([vp, P(i64), P(C.c_double)], i32),
        "disc_executor_num_events": ([vp], i32),
        "disc_executor_event": ([vp, i32, P(i32)], i32),
        "disc_executor_device_launches": ([vp], i64),
        "disc_executor_set_timing": ([vp, i32], i32),
        "disc_executor_num_records": ([vp], i32),
        "disc_executor_record": ([vp, i32, P(i32), P(i32), P(i64), P(C.c_double), P(i32), P(cp)], i32),
        "disc_executor_algorithmic_bytes": ([vp], i64),
        "disc_executor_set_schedule": ([vp, cp], i32),
        "disc_executor_set_cache_budget": ([vp, i64], i32),
        "disc_executor_reserve": ([vp, i64], i32),
        "disc_executor_set_async_flush": ([vp, i32], i32),
        "disc_executor_wait_issued": ([vp], i32),
        "disc_plan_identity": ([vp], vp),
        "disc_dispatcher_create": ([i32, P(i32), i32, P(vp)], i32),
        "disc_dispatcher_destroy": ([vp], None),
        "disc_dispatcher_num_workers": ([vp], i32),
        "disc_dispatcher_worker_device": ([vp, i32], i32),
        "disc_dispatcher_assign": ([vp, i32, P(vp), P(i32), P(cp), P(vp), P(i32), P(i32)], i32),
        "disc_dispatcher_run_grouped": ([vp, i32, P(vp), P(i32), P(cp), P(vp), P(vp), P(i32), i32, P(i32)], i32),
        "disc_dispatcher_request_worker": ([vp, i32], i32),
        "disc_dispatcher_num_request_outputs": ([vp, i32], i32),
        "disc_dispatcher_request_output": ([vp, i32, i32, P(vp), P(P(i64)), P(i32), P(i32)], i32),
        "disc_dispatcher_copy_request_output": ([vp, i32, i32, vp, i32], i32),
        "disc_dispatcher_worker_stats": ([vp, i32, P(i64), P(i64), P(C.c_double)], i32),
        "disc_executor_run_kernel": ([vp, vp, i32, i32, i32, P(vp), P(vp), P(i32), P(i64), i32], i32),
        "disc_guard_passes": ([vp, i32, i32, P(i64), i32], i32),
        "disc_plan_capture_programs": ([vp, i32, P(cp), P(vp), P(i32), P(vp)], i32),
        "disc_plan_host_overhead": ([vp, i32, P(cp), P(vp), P(i32), i32, P(C.c_double)], i32),
        "disc_plan_group_dry_run": ([i32, P(vp), P(i32), P(cp), P(vp), P(i32), i32, P(vp)], i32),
        "disc_cuda_set_specialization": ([i32], i32),
        "disc_cuda_specialized_launches": ([], i64),
        "disc_cuda_fused_launches": ([], i64),
        "disc_cuda_profiler": ([i32], i32),
        "disc_cuda_num_specializations": ([], i32),
        "disc_cuda_set_capture": ([i32], i32),
        "disc_cuda_capture_records": ([P(vp)], i32),
        # device layer (disc_cuda.h)
        "disc_cuda_last_error": ([], cp),
        "disc_cuda_device_count": ([P(i32)], i32),
        "disc_cuda_set_device": ([i32], i32),
        "disc_cuda_device_info": ([i32, P(i32), P(i64), P(i64)], i32),
        "disc_cuda_stream_create": ([P(vp)], i32),
        "disc_cuda_stream_destroy": ([vp], i32),
        "disc_cuda_stream_synchronize": ([vp], i32),
        "disc_cuda_device_synchronize": ([], i32),
        "disc_cuda_malloc": ([C.c_size_t, vp, P(vp)], i32),
        "disc_cuda_free": ([vp, vp], i32),
        "disc_cuda_host_alloc": ([C.c_size_t, P(vp)], i32),
        "disc_cuda_host_free": ([vp], i32),
        "disc_cuda_memcpy": ([vp, vp, C.c_size_t, i32, vp], i32),
        "disc_cuda_memset": ([vp, i32, C.c_size_t, vp], i32),
        "disc_cuda_event_create": ([P(vp)], i32),
        "disc_cuda_event_destroy": ([vp], i32),
        "disc_cuda_event_record": ([vp, vp], i32),
        "disc_cuda_event_synchronize": ([vp], i32),
        "disc_cuda_event_elapsed_ms": ([vp, vp, P(C.c_float)], i32),
        "disc_cuda_fill_uniform": ([vp, i64, C.c_uint64, C.c_float, C.c_float, vp], i32),
        "disc_cuda_flush_l2": ([vp, C.c_size_t, vp], i32),
        "disc_cuda_spin": ([C.c_uint64, vp], i32),
        "disc_cuda_set_pdl": ([i32], i32),
        "disc_cuda_pdl_mode": ([], i32),
        "disc_cuda_kernel_launches": ([], i64),
        "disc_cuda_alloc_stats": ([vp, vp, vp], i64),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"disc-b200 CUDA library not built: {LIB_PATH} "
                              "(run `python -m paper_2103_05288_b200.build`)")
        L = C.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        L = lib()
        cls = L.disc_last_error_class()
        raise DiscError(rc, L.disc_last_error().decode(),
                        ERROR_CLASSES[cls] if 0 <= cls < len(ERROR_CLASSES) else "internal")


def _cuda(rc: int, what: str = "cuda") -> None:
    if rc != 0:
        raise DiscError(4, f"{what}: {lib().disc_cuda_last_error().decode()}", "runtime")


def _take(p: C.c_void_p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    lib().disc_free(p)
    return s


def _str(fn, *args) -> str:
    out = C.c_void_p()
    _check(fn(*args, C.byref(out)))
    return _take(out)


def _graph_text(g) -> str:
    return g if isinstance(g, str) else json.dumps(g)


# ---------------------------------------------------------------------------
# Compile side.

@dataclass
class CompileOptions:
    inject_constraints: bool = True
    enable_fusion: bool = True
    static_fallback: bool = False

    def flags(self) -> Tuple[int, int, int]:
        return int(self.inject_constraints), int(self.enable_fusion), int(self.static_fallback)


class CompiledPlan:
    """Immutable compiled runtime flow (reference CompiledPlan, runtime_program.hpp:120)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def identity(self) -> int:
        """Address of the underlying plan object (shared by Compiler cache hits)."""
        return lib().disc_plan_identity(self._h) or 0

    def __del__(self):
        try:
            if self._h:
                lib().disc_plan_release(self._h)
        except Exception:
            pass

    @staticmethod
    def from_json(text: str) -> "CompiledPlan":
        h = C.c_void_p()
        _check(lib().disc_plan_from_json(text.encode(), C.byref(h)))
        return CompiledPlan(h)

    def to_json(self) -> str:
        return _str(lib().disc_plan_to_json, self._h)

    def check(self) -> List[str]:
        return json.loads(_str(lib().disc_plan_check, self._h))

    @property
    def input_names(self) -> List[str]:
        L = lib()
        return [L.disc_plan_input_name(self._h, i).decode() for i in range(L.disc_plan_num_inputs(self._h))]

    @property
    def output_names(self) -> List[str]:
        L = lib()
        return [L.disc_plan_output_name(self._h, i).decode() for i in range(L.disc_plan_num_outputs(self._h))]

    @property
    def num_kernels(self) -> int:
        return lib().disc_plan_num_kernels(self._h)

    @property
    def eager_op_count(self) -> int:
        return lib().disc_plan_eager_op_count(self._h)

    @property
    def host_instruction_count(self) -> int:
        return lib().disc_plan_host_instruction_count(self._h)

    def algorithmic_bytes(self, input_shapes: Dict[str, Sequence[int]]) -> int:
        """SURVEY §8d boundary bytes of one run at these input shapes (host only)."""
        names = list(input_shapes)
        dims = [np.array(input_shapes[n], dtype=np.int64) for n in names]
        k = len(names)
        c_names = (C.c_char_p * max(k, 1))(*[n.encode() for n in names])
        c_dims = (C.c_void_p * max(k, 1))(*[d.ctypes.data for d in dims])
        c_ranks = (C.c_int * max(k, 1))(*[d.size for d in dims])
        out = C.c_int64()
        _check(lib().disc_plan_algorithmic_bytes(self._h, k, c_names, c_dims, c_ranks, C.byref(out)))
        return out.value

    def eval_shapes(self, input_dims: Sequence[Sequence[int]]) -> List[int]:
        arrs = [np.asarray(d, dtype=np.int64) for d in input_dims]
        n = len(arrs)
        ptrs = (C.c_void_p * max(n, 1))(*[a.ctypes.data for a in arrs])
        ranks = (C.c_int * max(n, 1))(*[a.size for a in arrs])
        cap = 4096
        regs = (C.c_int64 * cap)()
        nregs = C.c_int()
        _check(lib().disc_plan_eval_shapes(self._h, n, ptrs, ranks, regs, cap, C.byref(nregs)))
        return list(regs[: nregs.value])


def compile_graph(graph, opts: Optional[CompileOptions] = None) -> CompiledPlan:
    """parse_graph + compile_graph (framework.cpp:350, codegen.cpp:688)."""
    o = opts or CompileOptions()
    h = C.c_void_p()
    _check(lib().disc_compile_graph(_graph_text(graph).encode(), *o.flags(), C.byref(h)))
    return CompiledPlan(h)


def static_specialize(graph) -> CompiledPlan:
    h = C.c_void_p()
    _check(lib().disc_static_specialize(_graph_text(graph).encode(), C.byref(h)))
    return CompiledPlan(h)


def cache_key(graph, opts: Optional[CompileOptions] = None) -> str:
    o = opts or CompileOptions()
    return _str(lib().disc_cache_key, _graph_text(graph).encode(), *o.flags())


def dump_stage(graph, stage: str, opts: Optional[CompileOptions] = None) -> str:
    o = opts or CompileOptions()
    return _str(lib().disc_dump_stage, _graph_text(graph).encode(), o.flags()[0], o.flags()[1], stage.encode())


def lower_dhlo_json(graph) -> str:
    return _str(lib().disc_lower_dhlo_json, _graph_text(graph).encode())


def dhlo_roundtrip(dhlo_json: str) -> str:
    return _str(lib().disc_dhlo_roundtrip, dhlo_json.encode())


class Compiler:
    """Shape-agnostic plan cache (reference Compiler, codegen.hpp:65-83)."""

    def __init__(self, opts: Optional[CompileOptions] = None):
        o = opts or CompileOptions()
        self._h = C.c_void_p()
        _check(lib().disc_compiler_create(*o.flags(), C.byref(self._h)))

    def __del__(self):
        try:
            lib().disc_compiler_destroy(self._h)
        except Exception:
            pass

    def compile(self, graph) -> CompiledPlan:
        h = C.c_void_p()
        _check(lib().disc_compiler_compile(self._h, _graph_text(graph).encode(), C.byref(h)))
        return CompiledPlan(h)

    def stats(self) -> Dict[str, int]:
        a, b = C.c_int64(), C.c_int64()
        lib().disc_compiler_stats(self._h, C.byref(a), C.byref(b))
        return {"compile_count": a.value, "cache_hits": b.value}


# ---------------------------------------------------------------------------
# Device memory (thin wrapper over disc_cuda.h; torch is not required).

class DeviceBuffer:
    """A device f32 tensor allocated from the stream-ordered pool."""

    def __init__(self, shape: Sequence[int], stream: Optional[int] = None):
        self.shape = tuple(int(d) for d in shape)
        self.numel = int(np.prod(self.shape)) if self.shape else 1
        self.nbytes = 4 * self.numel
        self.stream = stream
        self.ptr = C.c_void_p()
        _cuda(lib().disc_cuda_malloc(max(self.nbytes, 16), stream, C.byref(self.ptr)), "malloc")

    def free(self):
        if self.ptr:
            lib().disc_cuda_free(self.ptr, self.stream)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    @staticmethod
    def from_numpy(a: np.ndarray, stream: Optional[int] = None) -> "DeviceBuffer":
        a = np.array(a, dtype=np.float32, order="C", copy=True)
        b = DeviceBuffer(a.shape, stream)
        if b.nbytes:
            _cuda(lib().disc_cuda_memcpy(b.ptr, a.ctypes.data, b.nbytes, 0, stream), "h2d")
            _cuda(lib().disc_cuda_stream_synchronize(stream), "sync")
        return b

    def fill_uniform(self, seed: int, lo: float = 0.25, hi: float = 2.0) -> "DeviceBuffer":
        _cuda(lib().disc_cuda_fill_uniform(self.ptr, self.numel, seed, lo, hi, self.stream), "fill")
        return self

    def numpy(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=np.float32)
        if self.nbytes:
            _cuda(lib().disc_cuda_memcpy(out.ctypes.data, self.ptr, self.nbytes, 1, self.stream), "d2h")
            _cuda(lib().disc_cuda_stream_synchronize(self.stream), "sync")
        return out


def cuda_available() -> bool:
    try:
        n = C.c_int()
        return lib().disc_cuda_device_count(C.byref(n)) == 0 and n.value > 0
    except Exception:
        return False


def kernel_launches() -> int:
    return lib().disc_cuda_kernel_launches()


# ---------------------------------------------------------------------------
# Runtime flow.

@dataclass
class ExecStats:
    launch_count: int = 0
    library_calls: int = 0
    host_instruction_count: int = 0
    peak_bytes: int = 0
    alloc_calls: int = 0
    allocator_cache_hits: int = 0
    aliased_allocs: int = 0
    host_ms: float = 0.0
    kernel_ms: float = 0.0

    def as_dict(self) -> Dict[str, int]:
        return {k: getattr(self, k) for k in STAT_KEYS}


@dataclass
class ExecResult:
    outputs: List[np.ndarray]
    stats: ExecStats
    buffer_events: List[Tuple[int, int, int, int]] = field(default_factory=list)
    device_launches: int = 0


class Executor:
    """Runtime flow on one device + stream (reference Executor, executor.hpp:74-83).

    ``run(plan, inputs)`` takes numpy arrays (copied H2D inside the call) or
    DeviceBuffers (bound in place) and returns host outputs; ``run_device`` keeps the
    outputs on the device (valid until the next run)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self._h = C.c_void_p()
        self.stream = stream
        _check(lib().disc_executor_create(device, stream, C.byref(self._h)))

    def close(self) -> None:
        """Destroys the device executor now (idempotent); needed before the caller's
        stream is destroyed, since other references may keep this object alive."""
        h, self._h = self._h, C.c_void_p()
        if h:
            lib().disc_executor_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_timing(self, on: bool) -> None:
        lib().disc_executor_set_timing(self._h, int(on))

    def set_schedule(self, schedule: str) -> None:
        _check(lib().disc_executor_set_schedule(self._h, schedule.encode()))

    def set_host_threads(self, n: int) -> None:
        """Worker threads for the host flow of grouped calls (run_grouped)."""
        _check(lib().disc_executor_set_host_threads(self._h, int(n)))

    def set_graphs(self, on: bool) -> None:
        """Static plans as CUDA graphs (captured on the second identical run, then replayed)."""
        _check(lib().disc_executor_set_graphs(self._h, int(on)))

    def graph_replays(self) -> int:
        return lib().disc_executor_graph_replays(self._h)

    def set_cache_budget(self, nbytes: int) -> None:
        lib().disc_executor_set_cache_budget(self._h, int(nbytes))

    def set_async_flush(self, on: bool) -> None:
        _check(lib().disc_executor_set_async_flush(self._h, int(on)))

    def wait_issued(self) -> None:
        _check(lib().disc_executor_wait_issued(self._h))

    def reserve(self, nbytes: int) -> None:
        """Reserves device memory for the buffer arena up front (never released)."""
        _check(lib().disc_executor_reserve(self._h, int(nbytes)))

    def _bind(self, inputs: Dict[str, object]):
        names = list(inputs.keys())
        keep, datas, dims = [], [], []
        host = None
        for n in names:
            v = inputs[n]
            if isinstance(v, DeviceBuffer):
                is_host = False
                datas.append(v.ptr.value)
                d = np.array(v.shape, dtype=np.int64)
            else:
                is_host = True
                a = np.array(v, dtype=np.float32, order="C", copy=False)
                if not a.flags.c_contiguous:
                    a = np.ascontiguousarray(a)
                keep.append(a)
                datas.append(a.ctypes.data if a.size else 0)
                d = np.array(a.shape, dtype=np.int64)
            if host is None:
                host = is_host
            elif host != is_host:
                raise DiscError(2, "inputs must be all host or all device", "usage")
            keep.append(d)
            dims.append(d)
        n = len(names)
        c_names = (C.c_char_p * max(n, 1))(*[s.encode() for s in names])
        c_data = (C.c_void_p * max(n, 1))(*datas)
        c_dims = (C.c_void_p * max(n, 1))(*[d.ctypes.data for d in dims])
        c_ranks = (C.c_int * max(n, 1))(*[d.size for d in dims])
        return keep, n, c_names, c_data, c_dims, c_ranks, bool(host)

    def run_device(self, plan: CompiledPlan, inputs: Dict[str, object]) -> None:
        keep, n, names, data, dims, ranks, host = self._bind(inputs)
        _check(lib().disc_executor_run(self._h, plan._h, n, names, data, dims, ranks, int(host)))

    def run_stream(self, requests: Sequence[Tuple[CompiledPlan, Dict[str, object]]], grouped: bool = False) -> None:
        """Runs (plan, inputs) requests on this executor's stream (inputs all
        device-resident or all host).  grouped=False: back to back, outputs of the last
        request stay readable.  grouped=True: disc_executor_run_grouped -- the same plan
        kernel of all requests runs as one grouped launch; every request's outputs stay
        readable (request_outputs)."""
        keep, names, datas, dims, offs, plans = [], [], [], [], [0], []
        host = None
        for plan, inputs in requests:
            k, n, c_names, c_data, c_dims, c_ranks, h = self._bind(inputs)
            keep.append((k, c_names, c_data, c_dims, c_ranks))
            if host is None:
                host = h
            elif host != h:
                raise DiscError(2, "inputs must be all host or all device", "usage")
            names.extend(c_names[i] for i in range(n))
            datas.extend(c_data[i] for i in range(n))
            dims.extend(c_dims[i] for i in range(n))
            keep.append([c_ranks[i] for i in range(n)])
            offs.append(offs[-1] + n)
            plans.append(plan._h)
        ranks = [r for item in keep if isinstance(item, list) for r in item]
        m = len(requests)
        t = max(offs[-1], 1)
        fn = lib().disc_executor_run_grouped if grouped else lib().disc_executor_run_stream
        _check(fn(
            self._h, m, (C.c_void_p * max(m, 1))(*plans), (C.c_int * (m + 1))(*offs), (C.c_char_p * t)(*names),
            (C.c_void_p * t)(*datas), (C.c_void_p * t)(*dims), (C.c_int * t)(*ranks), int(bool(host))))

    def run_grouped(self, requests: Sequence[Tuple[CompiledPlan, Dict[str, object]]]) -> List[List[np.ndarray]]:
        """Grouped execution of independent requests; returns every request's host outputs."""
        self.run_stream(requests, grouped=True)
        outs = self.fetch_request_outputs()
        self.synchronize()
        return outs

    def request_output_views(self, r: int) -> List[Tuple[int, Tuple[int, ...]]]:
        L = lib()
        res = []
        for i in range(L.disc_executor_num_request_outputs(self._h, r)):
            p, d, k = C.c_void_p(), C.POINTER(C.c_int64)(), C.c_int()
            _check(L.disc_executor_request_output(self._h, r, i, C.byref(p), C.byref(d), C.byref(k)))
            res.append((p.value or 0, tuple(d[j] for j in range(k.value))))
        return res

    def fetch_request_outputs(self) -> List[List[np.ndarray]]:
        L = lib()
        out = []
        for r in range(L.disc_executor_num_requests(self._h)):
            row = []
            for i, (_, dims) in enumerate(self.request_output_views(r)):
                a = np.empty(dims, dtype=np.float32)
                if a.size:
                    _check(L.disc_executor_copy_request_output(self._h, r, i, a.ctypes.data, 1))
                row.append(a)
            out.append(row)
        return out

    def request_stats(self, r: int) -> ExecStats:
        s = (C.c_int64 * 7)()
        _check(lib().disc_executor_request_stats(self._h, r, s))
        return ExecStats(*list(s), 0.0, 0.0)

    def output_views(self) -> List[Tuple[int, Tuple[int, ...]]]:
        L = lib()
        res = []
        for i in range(L.disc_executor_num_outputs(self._h)):
            p, d, r = C.c_void_p(), C.POINTER(C.c_int64)(), C.c_int()
            _check(L.disc_executor_output(self._h, i, C.byref(p), C.byref(d), C.byref(r)))
            res.append((p.value or 0, tuple(d[k] for k in range(r.value))))
        return res

    def fetch_outputs(self) -> List[np.ndarray]:
        outs = []
        for i, (_, dims) in enumerate(self.output_views()):
            a = np.empty(dims, dtype=np.float32)
            if a.size:
                _check(lib().disc_executor_copy_output(self._h, i, a.ctypes.data, 1))
            outs.append(a)
        return outs

    def stats(self) -> ExecStats:
        s = (C.c_int64 * 7)()
        ms = (C.c_double * 2)()
        lib().disc_executor_stats(self._h, s, ms)
        return ExecStats(*list(s), ms[0], ms[1])

    def buffer_events(self) -> List[Tuple[int, int, int, int]]:
        L = lib()
        four = (C.c_int * 4)()
        ev = []
        for i in range(L.disc_executor_num_events(self._h)):
            L.disc_executor_event(self._h, i, four)
            ev.append(tuple(four))
        return ev

    def launch_records(self) -> List[Dict[str, object]]:
        """Per-kLaunch records of the last run (schedule, algorithmic bytes, device ms)."""
        L = lib()
        out = []
        for i in range(L.disc_executor_num_records(self._h)):
            ins, k, dk = C.c_int(), C.c_int(), C.c_int()
            b, ms, sch = C.c_int64(), C.c_double(), C.c_char_p()
            _check(L.disc_executor_record(self._h, i, C.byref(ins), C.byref(k), C.byref(b), C.byref(ms),
                                          C.byref(dk), C.byref(sch)))
            out.append({"instr": ins.value, "kernel": k.value, "bytes": b.value, "ms": ms.value,
                        "device_kernels": dk.value, "schedule": sch.value.decode()})
        return out

    def algorithmic_bytes(self) -> int:
        return lib().disc_executor_algorithmic_bytes(self._h)

    def device_launches(self) -> int:
        return lib().disc_executor_device_launches(self._h)

    def synchronize(self) -> None:
        _check(lib().disc_executor_synchronize(self._h))

    def run(self, plan: CompiledPlan, inputs: Dict[str, object]) -> ExecResult:
        self.run_device(plan, inputs)
        outs = self.fetch_outputs()
        self.synchronize()
        return ExecResult(outs, self.stats(), self.buffer_events(), self.device_launches())

    def run_kernel(self, plan: CompiledPlan, kernel: int, version: int, externals: Sequence[np.ndarray],
                   regs: Sequence[int]) -> List[np.ndarray]:
        """run_kernel (executor.cpp:137-219) on the device; returns host outputs."""
        bufs = [DeviceBuffer.from_numpy(x, self.stream) for x in externals]
        dims = [np.array(b.shape, dtype=np.int64) for b in bufs]
        n = len(bufs)
        c_ext = (C.c_void_p * max(n, 1))(*[b.ptr.value for b in bufs])
        c_dims = (C.c_void_p * max(n, 1))(*[d.ctypes.data for d in dims])
        c_ranks = (C.c_int * max(n, 1))(*[d.size for d in dims])
        r = (C.c_int64 * max(len(regs), 1))(*regs)
        _check(lib().disc_executor_run_kernel(self._h, plan._h, kernel, version, n, c_ext, c_dims, c_ranks, r,
                                              len(regs)))
        outs = self.fetch_outputs()
        self.synchronize()
        del bufs
        return outs


def capture_programs(plan: CompiledPlan, input_shapes: Dict[str, Sequence[int]]) -> list:
    """Host-only dry run: the lowered device programs of every fused launch."""
    names = list(input_shapes)
    dims = [np.array(input_shapes[n], dtype=np.int64) for n in names]
    k = len(names)
    c_names = (C.c_char_p * max(k, 1))(*[n.encode() for n in names])
    c_dims = (C.c_void_p * max(k, 1))(*[d.ctypes.data for d in dims])
    c_ranks = (C.c_int * max(k, 1))(*[d.size for d in dims])
    return json.loads(_str(lib().disc_plan_capture_programs, plan._h, k, c_names, c_dims, c_ranks))


def host_overhead_us(plan: CompiledPlan, input_shapes: Dict[str, Sequence[int]], iters: int = 2000) -> float:
    """Host cost of one run of the runtime flow (no device work), in microseconds."""
    names = list(input_shapes)
    dims = [np.array(input_shapes[n], dtype=np.int64) for n in names]
    k = len(names)
    c_names = (C.c_char_p * max(k, 1))(*[n.encode() for n in names])
    c_dims = (C.c_void_p * max(k, 1))(*[d.ctypes.data for d in dims])
    c_ranks = (C.c_int * max(k, 1))(*[d.size for d in dims])
    us = C.c_double()
    _check(lib().disc_plan_host_overhead(plan._h, k, c_names, c_dims, c_ranks, iters, C.byref(us)))
    return us.value


def new_stream() -> int:
    """A non-blocking CUDA stream (disc_cuda_stream_create), e.g. for Executor(0, stream)."""
    st = C.c_void_p()
    _cuda(lib().disc_cuda_stream_create(C.byref(st)))
    return st.value


def group_dry_run(requests: Sequence[Tuple[CompiledPlan, Dict[str, Sequence[int]]]], host_threads: int = 1) -> list:
    """Host-only flush plan of disc_executor_run_grouped for (plan, {input: shape}) requests
    (no device needed): one dict per issued action (grouped launches with their members'
    work in issue order, grouped copies, single ops)."""
    names, dims, ranks, offs, plans, keep = [], [], [], [0], [], []
    for plan, shapes in requests:
        for k, shp in shapes.items():
            d = np.array(shp, dtype=np.int64)
            keep.append(d)
            names.append(k.encode())
            dims.append(d.ctypes.data)
            ranks.append(d.size)
        offs.append(len(names))
        plans.append(plan._h)
    m, t = len(requests), max(len(names), 1)
    out = C.c_void_p()
    _check(lib().disc_plan_group_dry_run(m, (C.c_void_p * max(m, 1))(*plans), (C.c_int * (m + 1))(*offs),
                                         (C.c_char_p * t)(*names), (C.c_void_p * t)(*dims), (C.c_int * t)(*ranks),
                                         int(host_threads), C.byref(out)))
    return json.loads(_take(out))


def set_specialization(enabled: bool) -> None:
    lib().disc_cuda_set_specialization(int(enabled))


def set_pdl(mode: int) -> None:
    """Programmatic dependent launch between fused kernels: 0 off, 1 (default) launch
    overlap + dependency wait, 2 also early launch of the next kernel's CTAs."""
    lib().disc_cuda_set_pdl(int(mode))


def specialized_launches() -> int:
    return lib().disc_cuda_specialized_launches()


def guard_passes(plan: CompiledPlan, kernel: int, version: int, regs: Sequence[int]) -> bool:
    r = (C.c_int64 * max(len(regs), 1))(*regs)
    return lib().disc_guard_passes(plan._h, kernel, version, r, len(regs)) == 1
