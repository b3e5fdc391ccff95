"""Grouped execution (disc_executor_run_grouped): many independent variable-shape
requests, the same plan kernel of all of them issued as ONE grouped launch per kernel
instantiation.  Outputs must be bit-identical to running the requests one by one through
disc_executor_run (same kernels bodies, same per-launch grids and reduction orders), and
within the north-star tolerance of the reference executor."""
import json

import numpy as np
import pytest

from oracle import disc_oracle as O

pytestmark = pytest.mark.gpu


def _inputs(g, syms, rng):
    from paper_2103_05288_b200 import workloads as W
    out = {}
    for i in g["inputs"]:
        shape = [syms[d] if isinstance(d, str) else d for d in i["shape"]]
        cv = W.CONST_INPUTS.get(i["id"]) if i["id"] != "inv_h" else 1.0 / syms.get("H", 1)
        out[i["id"]] = (np.full(shape, cv, np.float32) if cv is not None
                        else rng.uniform(0.25, 2.0, size=shape).astype(np.float32))
    return out


def _sequential(gpu, reqs):
    ex = gpu.Executor()
    return [ex.run(plan, inputs).outputs for plan, inputs in reqs]


def _assert_same(grouped, seq, ctx):
    assert len(grouped) == len(seq), ctx
    for r, (a, b) in enumerate(zip(grouped, seq)):
        assert len(a) == len(b), (ctx, r)
        for x, y in zip(a, b):
            assert x.shape == y.shape, (ctx, r)
            np.testing.assert_array_equal(x, y, err_msg=f"{ctx} request {r}")


def _workload_requests(gpu, name, shapes, seed=0):
    from paper_2103_05288_b200 import workloads as W
    g = {"ln_gelu": W.ln_gelu_graph, "colreduce": W.colreduce_graph, "bert": W.bert_graph}.get(name)
    g = g() if g else W.softmax_graph_for(0)
    plan = gpu.compile_graph(g)
    rng = np.random.default_rng(seed)
    return g, plan, [(plan, _inputs(g, s, rng)) for s in shapes]


@pytest.mark.parametrize("host_inputs", [True, False])
def test_grouped_ln_gelu_matches_sequential(gpu, host_inputs):
    shapes = [{"T": t, "H": h} for h in (768, 1024, 4096) for t in (1, 2, 7, 33, 100, 513, 2000)]
    g, plan, reqs = _workload_requests(gpu, "ln_gelu", shapes, 1)
    seq = _sequential(gpu, reqs)
    if not host_inputs:
        keep = []
        dreqs = []
        for p, inputs in reqs:
            d = {k: gpu.DeviceBuffer.from_numpy(v) for k, v in inputs.items()}
            keep.append(d)
            dreqs.append((p, d))
        reqs = dreqs
    ex = gpu.Executor()
    before = gpu.kernel_launches()
    got = ex.run_grouped(reqs)
    launched = gpu.kernel_launches() - before
    _assert_same(got, seq, "ln_gelu")
    # 3 plan kernels -> a handful of grouped launches, not 3 x len(shapes)
    assert launched <= 3 * 3, launched
    # and every request against the numpy oracle (oracle/disc_oracle.py) on its own inputs
    src = [(p, {k: v.numpy() if hasattr(v, "numpy") else v for k, v in i.items()}) for p, i in reqs]
    for r, (p, inputs) in enumerate(src):
        want, _, _ = O.Executor().run(plan.to_json(), {k: np.asarray(v) for k, v in inputs.items()})
        assert len(want) == len(got[r])
        for a, b in zip(got[r], want):
            assert O.rel_err(a, b) <= 1e-5, (r, shapes[r], O.rel_err(a, b))


@pytest.mark.parametrize("name,shapes", [
    ("softmax", [{"S0": b, "S1": s} for s, b in [(1, 100), (7, 3000), (31, 2048), (64, 517), (4096, 9), (1000, 33)]]),
    ("colreduce", [{"N": n, "C": c} for n, c in [(1, 5), (1000, 36), (64, 4096), (70000, 3), (5000, 260), (2, 1)]]),
    ("bert", [{"R": 12 * b * s, "S": s, "T": b * s, "H": 768, "F": 3072} for b, s in [(1, 8), (2, 64), (1, 128)]]),
])
def test_grouped_workloads_match_sequential(gpu, name, shapes):
    g, plan, reqs = _workload_requests(gpu, name, shapes, 2)
    seq = _sequential(gpu, reqs)
    got = gpu.Executor().run_grouped(reqs)
    _assert_same(got, seq, name)


@pytest.mark.parametrize("schedule", ["twopass", "atomic", "materialize"])
def test_grouped_alternate_schedules(gpu, schedule):
    g, plan, reqs = _workload_requests(gpu, "colreduce", [{"N": n, "C": c} for n, c in
                                                          [(3000, 36), (64, 4096), (70000, 3), (5000, 260)]], 3)
    ex1 = gpu.Executor()
    ex1.set_schedule(schedule)
    seq = [ex1.run(p, i).outputs for p, i in reqs]
    ex2 = gpu.Executor()
    ex2.set_schedule(schedule)
    _assert_same(ex2.run_grouped(reqs), seq, schedule)


def test_grouped_mixed_fixtures_and_oracle(gpu, ref, fixtures):
    """Heterogeneous requests (every fixture graph incl. standalone/library artifacts,
    several bindings each), grouped in one call: equal to sequential runs and to the
    reference executor."""
    reqs, want = [], []
    for name in sorted(fixtures):
        f = fixtures[name]
        plan = gpu.compile_graph(f["graph"])
        rp = ref.RefPlan(ref.compile(f["graph"]))
        for k, syms in enumerate(f["bindings"]):
            inputs = ref.make_binding(f["graph"], syms, 11 + k)
            reqs.append((plan, inputs))
            want.append(rp.run(inputs).outputs)
    sx = gpu.Executor()
    runs = [sx.run(plan, inputs) for plan, inputs in reqs]
    seq = [r.outputs for r in runs]
    ex = gpu.Executor()
    got = ex.run_grouped(reqs)
    _assert_same(got, seq, "fixtures")
    for r, (a, b) in enumerate(zip(got, want)):
        for x, y in zip(a, b):
            assert O.rel_err(x, y) <= 1e-5, r
    # per-request stats: launch / library-call / instruction counts and peak bytes follow
    # the plan (allocator hit counters differ: no block is reused inside a group)
    for r, run in enumerate(runs):
        st = ex.request_stats(r)
        for k in ("launch_count", "library_calls", "host_instruction_count", "peak_bytes", "aliased_allocs"):
            assert getattr(st, k) == getattr(run.stats, k), (r, k)


def test_grouped_random_graphs(gpu, ref):
    """Random reference graphs (acceptance_main.cpp seeds), 3 bindings each, all in one
    grouped call: bit-identical to sequential execution."""
    rng = ref.RefRng(20260810)
    reqs = []
    for seed in range(40):
        g = ref.random_graph(seed, 12)
        plan = gpu.compile_graph(g)
        for b in range(3):
            reqs.append((plan, ref.make_binding(g, rng.random_symbols(g), seed * 31 + b)))
    seq = _sequential(gpu, reqs)
    _assert_same(gpu.Executor().run_grouped(reqs), seq, "random")


def test_grouped_repeated_calls_and_records(gpu):
    """Back-to-back grouped calls reuse buffers safely; timing records are per grouped
    launch and their bytes add up to the executor's algorithmic bytes."""
    shapes = [{"T": t, "H": 1024} for t in (5, 50, 500, 5000)]
    g, plan, reqs = _workload_requests(gpu, "ln_gelu", shapes, 4)
    seq = _sequential(gpu, reqs)
    ex = gpu.Executor()
    for _ in range(3):
        _assert_same(ex.run_grouped(reqs), seq, "repeat")
    keep = [{k: gpu.DeviceBuffer.from_numpy(v) for k, v in inputs.items()} for _, inputs in reqs]
    ex.set_timing(True)
    ex.run_stream([(plan, d) for d in keep], grouped=True)
    ex.synchronize()
    recs = ex.launch_records()
    assert 3 <= len(recs) <= 6, recs  # 3 plan kernels, split only by kernel instantiation
    assert sum(r["bytes"] for r in recs) == ex.algorithmic_bytes()
    assert all(r["ms"] > 0 for r in recs)
    assert all(r["schedule"].startswith("group:") for r in recs)


def test_grouped_errors_are_reported(gpu, fixtures):
    """A request failing its runtime checks raises the reference's error; requests queued
    before it are still issued (valid work)."""
    from paper_2103_05288_b200 import workloads as W
    g = W.ln_gelu_graph()
    plan = gpu.compile_graph(g)
    rng = np.random.default_rng(0)
    good = _inputs(g, {"T": 4, "H": 768}, rng)
    bad = dict(good)
    bad["gamma"] = np.ones(5, np.float32)  # violates H
    ex = gpu.Executor()
    with pytest.raises(gpu.DiscError) as e:
        ex.run_stream([(plan, good), (plan, bad)], grouped=True)
    assert "shape constraint" in str(e.value) or "mismatch" in str(e.value)
    ex.synchronize()
    # the executor is usable afterwards
    got = ex.run_grouped([(plan, good)])
    want = gpu.Executor().run(plan, good).outputs
    _assert_same(got, [want], "after error")


@pytest.mark.parametrize("threads", [2, 4])
def test_grouped_host_threads_identical(gpu, ref, threads):
    """Multi-threaded host flow (worker sub-executors, merged queues): outputs and
    per-request stats identical to the single-threaded grouped call and to sequential runs."""
    rng = ref.RefRng(99)
    reqs = []
    for seed in range(60):
        g = ref.random_graph(seed, 10)
        plan = gpu.compile_graph(g)
        for b in range(5):
            reqs.append((plan, ref.make_binding(g, rng.random_symbols(g), seed * 7 + b)))
    seq = _sequential(gpu, reqs)
    one = gpu.Executor()
    base = one.run_grouped(reqs)
    _assert_same(base, seq, "1 thread")
    ex = gpu.Executor()
    ex.set_host_threads(threads)
    for _ in range(2):  # the second call reuses sub-executor caches
        _assert_same(ex.run_grouped(reqs), seq, f"{threads} threads")
    for r in range(len(reqs)):
        assert ex.request_stats(r).launch_count == one.request_stats(r).launch_count
    # the merged flush issues the same groups as one thread queueing everything
    one.set_timing(True)
    one.run_stream(reqs, grouped=True)
    one.synchronize()
    ex.set_timing(True)
    ex.run_stream(reqs, grouped=True)
    ex.synchronize()
    assert ex.algorithmic_bytes() == one.algorithmic_bytes()
    key = lambda recs: sorted((r["instr"], r["schedule"], r["bytes"], r["device_kernels"]) for r in recs)
    assert key(ex.launch_records()) == key(one.launch_records())


def test_grouped_mixed_alignment_rows(gpu):
    """Aligned and odd-width rows of one plan in one grouped call: separate kernel
    instantiations, never one group (odd widths run the float4-body row kernel)."""
    shapes = [{"S0": b, "S1": s} for s, b in [(64, 50), (255, 40), (1024, 9), (777, 11), (17, 300), (16, 300), (1, 500)]]
    g, plan, reqs = _workload_requests(gpu, "softmax", shapes, 5)
    _assert_same(gpu.Executor().run_grouped(reqs), _sequential(gpu, reqs), "mixed alignment")


def test_async_flush_matches_synchronous(gpu):
    """Grouped calls whose launches are issued by the background flusher (device inputs)
    give the same bits as synchronous flushes, call after call (memory reused in call
    order), and ExecStats are unchanged."""
    from paper_2103_05288_b200 import workloads as W
    graphs, reqs = W.mixed_stream(600, seed=5)
    plans = {k: gpu.compile_graph(g) for k, g in graphs.items()}
    rng = np.random.default_rng(8)
    batches = []
    for c in range(3):
        sub = reqs[c * 200:(c + 1) * 200]
        batches.append([(plans[k], {i["id"]: gpu.DeviceBuffer.from_numpy(rng.uniform(0.25, 2.0, size=tuple(
            s[d] if isinstance(d, str) else d for d in i["shape"])).astype(np.float32)) for i in graphs[k]["inputs"]})
            for k, s in sub])
    results = {}
    for mode in (False, True):
        ex = gpu.Executor()
        ex.set_host_threads(4)
        ex.set_async_flush(mode)
        out = []
        for b in batches:
            ex.run_stream(b, grouped=True)
            out.append((ex.fetch_request_outputs(), [ex.request_stats(r) for r in range(len(b))]))
        ex.synchronize()
        results[mode] = out
    for (oa, sa), (ob, sb) in zip(results[False], results[True]):
        assert sa == sb
        for ra, rb in zip(oa, ob):
            for a, b in zip(ra, rb):
                np.testing.assert_array_equal(a, b)
