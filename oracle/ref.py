"""TEST INFRASTRUCTURE ONLY -- ctypes binding to oracle/_ref/libdisc_ref.so.

libdisc_ref.so is the *unmodified* reference DISC artifact (/root/reference/proj/src/*.cpp)
plus oracle/ref_shim.cpp, built by oracle/Makefile.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / ``--impl reference`` legs may import this module; the
product (paper_2103_05288_b200) never does.

Every call here is a reference entry point:
  compile()        -> disc::compile_graph + plan_to_json   (codegen.cpp:688, runtime_program.cpp:182)
  RefPlan.run()    -> disc::Executor::run                  (executor.cpp:221-465)
  eval_eager()     -> disc::eval_eager(FrameworkGraph)     (interpreter.cpp:222-378)
  run_kernel()     -> disc::run_kernel                     (executor.cpp:137-219)
  random_graph() / make_binding() / random_symbols()      (tests/testutil.hpp:86-432)
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libdisc_ref.so")
_lib: Optional[C.CDLL] = None

STAT_KEYS = ("launch_count", "library_calls", "host_instruction_count", "peak_bytes",
             "alloc_calls", "allocator_cache_hits", "aliased_allocs")


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run `make -C oracle`)")
        L = C.CDLL(LIB_PATH)
        vp, cp, i64, i32 = C.c_void_p, C.c_char_p, C.c_int64, C.c_int
        pp = C.POINTER(C.c_char_p)
        L.dref_last_error.restype = cp
        L.dref_free.argtypes = [vp]
        for name in ("dref_compile",):
            getattr(L, name).argtypes = [cp, i32, i32, i32, C.POINTER(vp)]
        L.dref_static_specialize.argtypes = [cp, C.POINTER(vp)]
        L.dref_cache_key.argtypes = [cp, i32, i32, i32, C.POINTER(vp)]
        L.dref_dump_stage.argtypes = [cp, i32, i32, cp, C.POINTER(vp)]
        L.dref_lower_dhlo_json.argtypes = [cp, C.POINTER(vp)]
        L.dref_roundtrip_plan.argtypes = [cp, C.POINTER(vp)]
        L.dref_compiler_new.argtypes = [i32, i32, i32, C.POINTER(vp)]
        L.dref_compiler_free.argtypes = [vp]
        L.dref_compiler_compile.argtypes = [vp, cp, C.POINTER(vp)]
        L.dref_compiler_stats.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        L.dref_plan_load.argtypes = [cp, C.POINTER(vp)]
        L.dref_plan_free.argtypes = [vp]
        L.dref_executor_new.restype = vp
        L.dref_executor_free.argtypes = [vp]
        runargs = [vp, vp, i32, C.POINTER(cp), C.POINTER(vp), C.POINTER(vp), C.POINTER(i32)]
        L.dref_executor_run.argtypes = runargs + [C.POINTER(vp)]
        L.dref_executor_time.argtypes = runargs + [i32, C.POINTER(C.c_double)]
        L.dref_eval_eager.argtypes = [cp, i32, C.POINTER(cp), C.POINTER(vp), C.POINTER(vp),
                                      C.POINTER(i32), C.POINTER(vp)]
        L.dref_run_kernel.argtypes = [vp, i32, i32, i32, C.POINTER(vp), C.POINTER(vp),
                                      C.POINTER(i32), C.POINTER(i64), i32, C.POINTER(vp)]
        L.dref_guard_passes.argtypes = [vp, i32, i32, C.POINTER(i64), i32]
        L.dref_result_count.argtypes = [vp]
        L.dref_result_rank.argtypes = [vp, i32]
        L.dref_result_dims.argtypes = [vp, i32]
        L.dref_result_dims.restype = C.POINTER(i64)
        L.dref_result_data.argtypes = [vp, i32]
        L.dref_result_data.restype = C.POINTER(C.c_float)
        L.dref_result_stats.argtypes = [vp, C.POINTER(i64), C.POINTER(C.c_double)]
        L.dref_result_num_events.argtypes = [vp]
        L.dref_result_event.argtypes = [vp, i32, C.POINTER(i32)]
        L.dref_result_free.argtypes = [vp]
        L.dref_rng_new.argtypes = [C.c_uint64]
        L.dref_rng_new.restype = vp
        L.dref_rng_free.argtypes = [vp]
        L.dref_random_graph.argtypes = [C.c_uint64, i32, C.POINTER(vp)]
        L.dref_random_symbols.argtypes = [vp, cp, i32, C.POINTER(vp)]
        L.dref_make_binding.argtypes = [cp, cp, C.c_uint64, C.POINTER(vp)]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise RefError(rc, lib().dref_last_error().decode())


def _take_string(p: C.c_void_p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    lib().dref_free(p)
    return s


def _str_call(fn, *args) -> str:
    out = C.c_void_p()
    _check(fn(*args, C.byref(out)))
    return _take_string(out)


def compile(graph_json: str, inject: bool = True, fusion: bool = True,
            static_fallback: bool = False) -> str:
    return _str_call(lib().dref_compile, graph_json.encode(), int(inject), int(fusion),
                     int(static_fallback))


def static_specialize(graph_json: str) -> str:
    return _str_call(lib().dref_static_specialize, graph_json.encode())


def cache_key(graph_json: str, inject=True, fusion=True, static_fallback=False) -> str:
    return _str_call(lib().dref_cache_key, graph_json.encode(), int(inject), int(fusion),
                     int(static_fallback))


def dump_stage(graph_json: str, stage: str, inject=True, fusion=True) -> str:
    return _str_call(lib().dref_dump_stage, graph_json.encode(), int(inject), int(fusion),
                     stage.encode())


def lower_dhlo_json(graph_json: str) -> str:
    return _str_call(lib().dref_lower_dhlo_json, graph_json.encode())


def roundtrip_plan(plan_json: str) -> str:
    return _str_call(lib().dref_roundtrip_plan, plan_json.encode())


def _marshal(tensors: Sequence[np.ndarray], names: Optional[Sequence[str]] = None):
    arrs = [np.array(t, dtype=np.float32, order="C", copy=True) for t in tensors]  # keeps rank 0
    n = len(arrs)
    names_b = (C.c_char_p * max(n, 1))(*[(nm or "").encode() for nm in (names or [""] * n)])
    data = (C.c_void_p * max(n, 1))(*[a.ctypes.data for a in arrs])
    dims_arrs = [np.array(a.shape, dtype=np.int64) for a in arrs]
    dims = (C.c_void_p * max(n, 1))(*[d.ctypes.data for d in dims_arrs])
    ranks = (C.c_int * max(n, 1))(*[a.ndim for a in arrs])
    return arrs, dims_arrs, names_b, data, dims, ranks


class RefResult:
    def __init__(self, h: C.c_void_p):
        L = lib()
        self.outputs: List[np.ndarray] = []
        for i in range(L.dref_result_count(h)):
            r = L.dref_result_rank(h, i)
            dims = tuple(L.dref_result_dims(h, i)[k] for k in range(r))
            n = int(np.prod(dims)) if dims else 1
            if n:
                buf = np.ctypeslib.as_array(L.dref_result_data(h, i), shape=(n,)).copy()
            else:
                buf = np.zeros((0,), np.float32)
            self.outputs.append(buf.reshape(dims))
        s = (C.c_int64 * 7)()
        ms = (C.c_double * 2)()
        L.dref_result_stats(h, s, ms)
        self.stats: Dict[str, int] = dict(zip(STAT_KEYS, list(s)))
        self.host_ms, self.kernel_ms = ms[0], ms[1]
        self.events = []
        four = (C.c_int * 4)()
        for i in range(L.dref_result_num_events(h)):
            L.dref_result_event(h, i, four)
            self.events.append(tuple(four))
        L.dref_result_free(h)


class RefPlan:
    """A reference CompiledPlan (plan_from_json) plus one reference Executor."""

    def __init__(self, plan_json: str):
        self._h = C.c_void_p()
        _check(lib().dref_plan_load(plan_json.encode(), C.byref(self._h)))
        self._exec = C.c_void_p(lib().dref_executor_new())
        self.json = json.loads(plan_json)
        self.input_ids = [i["id"] for i in self.json["inputs"]]

    def __del__(self):
        try:
            lib().dref_executor_free(self._exec)
            lib().dref_plan_free(self._h)
        except Exception:
            pass

    def run(self, inputs: Dict[str, np.ndarray]) -> RefResult:
        names = list(inputs.keys())
        keep = _marshal([inputs[n] for n in names], names)
        _, _, names_b, data, dims, ranks = keep
        out = C.c_void_p()
        _check(lib().dref_executor_run(self._exec, self._h, len(names), names_b, data, dims,
                                       ranks, C.byref(out)))
        return RefResult(out)

    def time(self, inputs: Dict[str, np.ndarray], reps: int) -> float:
        names = list(inputs.keys())
        keep = _marshal([inputs[n] for n in names], names)
        _, _, names_b, data, dims, ranks = keep
        secs = C.c_double()
        _check(lib().dref_executor_time(self._exec, self._h, len(names), names_b, data, dims,
                                        ranks, reps, C.byref(secs)))
        return secs.value

    def run_kernel(self, kernel: int, version: int, externals: Sequence[np.ndarray],
                   regs: Sequence[int]) -> List[np.ndarray]:
        keep = _marshal(externals)
        _, _, _, data, dims, ranks = keep
        r = (C.c_int64 * max(len(regs), 1))(*regs)
        out = C.c_void_p()
        _check(lib().dref_run_kernel(self._h, kernel, version, len(externals), data, dims, ranks,
                                     r, len(regs), C.byref(out)))
        return RefResult(out).outputs

    def guard_passes(self, kernel: int, version: int, regs: Sequence[int]) -> bool:
        r = (C.c_int64 * max(len(regs), 1))(*regs)
        return lib().dref_guard_passes(self._h, kernel, version, r, len(regs)) == 1


def eval_eager(graph_json: str, inputs: Dict[str, np.ndarray]) -> RefResult:
    names = list(inputs.keys())
    keep = _marshal([inputs[n] for n in names], names)
    _, _, names_b, data, dims, ranks = keep
    out = C.c_void_p()
    _check(lib().dref_eval_eager(graph_json.encode(), len(names), names_b, data, dims, ranks,
                                 C.byref(out)))
    return RefResult(out)


class RefCompiler:
    def __init__(self, inject=True, fusion=True, static_fallback=False):
        self._h = C.c_void_p()
        _check(lib().dref_compiler_new(int(inject), int(fusion), int(static_fallback),
                                       C.byref(self._h)))

    def __del__(self):
        try:
            lib().dref_compiler_free(self._h)
        except Exception:
            pass

    def compile(self, graph_json: str) -> str:
        return _str_call(lambda *a: lib().dref_compiler_compile(self._h, *a), graph_json.encode())

    def stats(self) -> Tuple[int, int]:
        a, b = C.c_int64(), C.c_int64()
        lib().dref_compiler_stats(self._h, C.byref(a), C.byref(b))
        return a.value, b.value


class RefRng:
    """std::mt19937_64 shared across random_symbols calls (acceptance_main.cpp:60)."""

    def __init__(self, seed: int):
        self._h = C.c_void_p(lib().dref_rng_new(seed))

    def __del__(self):
        try:
            lib().dref_rng_free(self._h)
        except Exception:
            pass

    def random_symbols(self, graph_json: str, allow_zero: bool = True) -> Dict[str, int]:
        return json.loads(_str_call(lambda *a: lib().dref_random_symbols(self._h, *a),
                                    graph_json.encode(), int(allow_zero)))


def random_graph(seed: int, max_nodes: int = 12) -> str:
    return _str_call(lib().dref_random_graph, seed, max_nodes)


def make_binding(graph_json: str, syms: Dict[str, int], seed: int) -> Dict[str, np.ndarray]:
    out = C.c_void_p()
    _check(lib().dref_make_binding(graph_json.encode(), json.dumps(syms).encode(), seed,
                                   C.byref(out)))
    res = RefResult(out)
    ids = [i["id"] for i in json.loads(graph_json)["inputs"]]
    return dict(zip(ids, res.outputs))
