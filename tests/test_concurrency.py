"""Concurrency (SURVEY §8(b) threading): the reference's own concurrency cases plus the
thread-safety of the device layer's shared state.

* test_plan.cpp:215-226 -- 8 threads compiling the same graph coalesce into one compile
  (Compiler's shared_future; compile_count 1, cache_hits 7, one shared plan object);
* test_executor.cpp:115-131 -- a shared plan executes concurrently on 4 executors (one per
  thread), each within 1e-5 of the reference;
* a host-only dry run (capture mode) on one thread while other threads execute for real:
  capture mode is per thread, so the real executors still produce correct outputs;
* executors on several threads launching the same kernel instantiations with different
  dynamic shared-memory sizes (the smem attribute only ever grows per kernel).
"""
import json
import threading

import numpy as np
import pytest

from conftest import FIXTURES
from oracle import disc_oracle as O


def _run_threads(fns):
    errs = []

    def wrap(f):
        try:
            f()
        except BaseException as e:  # noqa: BLE001 - surfaced below
            errs.append(e)
    ts = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


def test_concurrent_compiles_coalesce(fixtures):
    import paper_2103_05288_b200 as D
    g = fixtures["transformer"]["graph"]
    comp = D.Compiler()
    plans = [None] * 8

    def one(t):
        plans[t] = comp.compile(g)
    _run_threads([lambda t=t: one(t) for t in range(8)])
    ids = {p.identity() for p in plans}
    assert len(ids) == 1 and 0 not in ids
    assert comp.stats() == {"compile_count": 1, "cache_hits": 7}


@pytest.mark.gpu
def test_shared_plan_executes_concurrently(gpu, ref, fixtures):
    g = fixtures["transformer"]["graph"]
    plan = gpu.compile_graph(g)
    errors = [1.0] * 4

    def one(t):
        inputs = ref.make_binding(g, {"S0": 3 + t}, 50 + t)
        ex = gpu.Executor()  # one executor (and allocator) per thread
        got = ex.run(plan, inputs)
        want = ref.eval_eager(g, inputs).outputs
        errors[t] = max(O.rel_err(a, b) for a, b in zip(got.outputs, want))
    _run_threads([lambda t=t: one(t) for t in range(4)])
    assert max(errors) <= 1e-5, errors


@pytest.mark.gpu
def test_dry_run_does_not_disturb_real_executors(gpu, ref, fixtures):
    """disc_plan_group_dry_run switches capture mode on for its own thread only."""
    g = fixtures["softmax"]["graph"]
    plan = gpu.compile_graph(g)
    stop = threading.Event()
    results = []

    def dry():
        while not stop.is_set():
            gpu.group_dry_run([(plan, {"x": (64, 8)})] * 300, host_threads=4)

    def real(t):
        ex = gpu.Executor()
        ex.set_host_threads(2)
        for i in range(20):
            inputs = ref.make_binding(g, {"S0": 200 + 13 * i + t}, 7 + i)
            got = ex.run(plan, inputs)
            want = ref.eval_eager(g, inputs).outputs
            results.append(max(O.rel_err(a, b) for a, b in zip(got.outputs, want)))
    d = threading.Thread(target=dry)
    d.start()
    try:
        _run_threads([lambda t=t: real(t) for t in range(3)])
    finally:
        stop.set()
        d.join()
    assert len(results) == 60 and max(results) <= 1e-5, max(results)


@pytest.mark.gpu
def test_concurrent_launches_with_different_smem(gpu, ref):
    """Same row-kernel instantiation, different row-cache sizes (R), on 4 threads at once."""
    g = json.dumps({"name": "sm", "inputs": [{"id": "x", "shape": ["B", "S"], "dtype": "f32"}], "outputs": ["y"],
                    "nodes": [{"id": "y", "op": "Softmax", "inputs": ["x"]}]})
    plan = gpu.compile_graph(g)
    errors = []

    def one(t):
        ex = gpu.Executor()
        for i in range(12):
            s = [64, 1024, 3000, 4096, 520, 2000][(i + t) % 6]
            x = np.random.default_rng(100 * t + i).uniform(0.25, 2, size=(37, s)).astype(np.float32)
            got = ex.run(plan, {"x": x}).outputs[0]
            e = np.exp(x.astype(np.float64) - x.max(axis=1, keepdims=True))
            errors.append(O.rel_err(got, (e / e.sum(axis=1, keepdims=True)).astype(np.float32)))
    _run_threads([lambda t=t: one(t) for t in range(4)])
    assert len(errors) == 48 and max(errors) <= 1e-5, max(errors)
