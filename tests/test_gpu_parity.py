"""GPU parity through the C ABI (SURVEY §8a runtime rows a15-a23): the B200 runtime flow
and fused kernels against the reference executor (oracle/_ref) and the committed goldens.

Tolerances: f32 outputs within 1e-5 rel_err (tests/testutil.hpp:64-70); reductions
accumulate in f64 on both sides.  ExecStats and BufferEvents must match exactly."""
import json

import numpy as np
import pytest

from conftest import FIXTURES, OPTION_SETS, REF_FLAGS, fixture_binding
from oracle import disc_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-5


def check_outputs(got, want, tol=TOL, ctx=""):
    assert len(got) == len(want), ctx
    for a, b in zip(got, want):
        assert tuple(a.shape) == tuple(b.shape), ctx
        err = O.rel_err(a, b)
        assert err <= tol, f"{ctx}: rel err {err}"


def test_golden_fixture_io(gpu, fixture_io, fixture_plans):
    z, meta = fixture_io
    execs = {}
    for key, m in meta.items():
        name, _ = key.split("/")
        plan = gpu.CompiledPlan.from_json(fixture_plans[f"{name}/default"])
        ex = execs.setdefault(name, gpu.Executor())
        inputs = {k: z[f"{key}/in/{k}"] for k in m["inputs"]}
        r = ex.run(plan, inputs)
        assert r.stats.as_dict() == m["stats"], key
        check_outputs(r.outputs, [z[f"{key}/out/{i}"] for i in range(m["n_out"])], ctx=key)


@pytest.mark.parametrize("opt", list(OPTION_SETS))
def test_fixtures_vs_reference(gpu, ref, fixtures, opt):
    for name in FIXTURES:
        g = fixtures[name]["graph"]
        plan = gpu.compile_graph(g, gpu.CompileOptions(**OPTION_SETS[opt]))
        rp = ref.RefPlan(ref.compile(g, **REF_FLAGS[opt]))
        ex = gpu.Executor()
        for syms in fixtures[name]["bindings"]:
            inputs = ref.make_binding(g, syms, 7)
            r = rp.run(inputs)
            mine = ex.run(plan, inputs)
            assert mine.stats.as_dict() == r.stats, (name, opt)
            assert mine.buffer_events == r.events, (name, opt)
            check_outputs(mine.outputs, r.outputs, ctx=f"{name}/{opt}")


def test_random_graphs_oracle_equivalence(gpu, ref):
    """Acceptance criterion 1 on the GPU: 200 random graphs x 5 bindings <= 1e-5,
    with the reference's seeds (acceptance_main.cpp:58-87)."""
    rng = ref.RefRng(20260810)
    for seed in range(200):
        g = ref.random_graph(seed, 12)
        plan = gpu.compile_graph(g)
        ex = gpu.Executor()
        for b in range(5):
            syms = rng.random_symbols(g)
            inputs = ref.make_binding(g, syms, seed * 31 + b)
            want = ref.eval_eager(g, inputs).outputs
            got = ex.run(plan, inputs)
            check_outputs(got.outputs, want, ctx=f"seed {seed} binding {b}")


@pytest.mark.parametrize("schedule", ["materialize", "twopass", "atomic"])
def test_random_graphs_alternate_schedules(gpu, ref, schedule):
    rng = ref.RefRng(77)
    for seed in range(60):
        g = ref.random_graph(seed, 12)
        plan = gpu.compile_graph(g)
        ex = gpu.Executor()
        ex.set_schedule(schedule)
        syms = rng.random_symbols(g)
        inputs = ref.make_binding(g, syms, seed)
        check_outputs(ex.run(plan, inputs).outputs, ref.eval_eager(g, inputs).outputs, ctx=f"{schedule} {seed}")


def test_compile_once_adaptivity(gpu, ref, fixtures):
    """Criterion 2: 100 bindings per fixture through one cached plan."""
    for name in FIXTURES:
        g = fixtures[name]["graph"]
        c = gpu.Compiler()
        plan = c.compile(g)
        ex = gpu.Executor()
        for i in range(1, 101):
            inputs = ref.make_binding(g, fixture_binding(name, i), 1000 + i)
            check_outputs(ex.run(plan, inputs).outputs, ref.eval_eager(g, inputs).outputs, ctx=f"{name} {i}")
        for _ in range(99):
            c.compile(g)
        assert c.stats() == {"compile_count": 1, "cache_hits": 99}


def test_launch_counts_and_ablation(gpu, ref, fixtures):
    """Criteria 3 and 4."""
    tf = fixtures["transformer"]["graph"]
    r = gpu.Executor().run(gpu.compile_graph(tf), ref.make_binding(tf, {"S0": 8}, 3))
    assert r.stats.launch_count + r.stats.library_calls == 18
    sm = fixtures["softmax"]["graph"]
    r = gpu.Executor().run(gpu.compile_graph(sm), ref.make_binding(sm, {"S0": 4}, 4))
    assert r.stats.launch_count == 2
    sp = fixtures["split"]["graph"]
    b = ref.make_binding(sp, {"S0": 6, "T0": 6, "T1": 6}, 5)
    w = gpu.Executor().run(gpu.compile_graph(sp), b)
    wo = gpu.Executor().run(gpu.compile_graph(sp, gpu.CompileOptions(inject_constraints=False)), b)
    assert w.stats.launch_count < wo.stats.launch_count
    check_outputs(w.outputs, ref.eval_eager(sp, b).outputs)
    check_outputs(wo.outputs, ref.eval_eager(sp, b).outputs)


def test_buffer_safety_and_second_run(gpu, ref, fixtures):
    """Criterion 5 + test_buffers.cpp:220-230: events identical to the reference, no
    overlapping live intervals, and a second run allocates nothing."""
    for name in FIXTURES:
        g = fixtures[name]["graph"]
        plan = gpu.compile_graph(g)
        ex = gpu.Executor()
        for syms in fixtures[name]["bindings"]:
            inputs = ref.make_binding(g, syms, 7)
            r1 = ex.run(plan, inputs)
            r2 = ex.run(plan, inputs)
            assert r2.stats.alloc_calls == 0
            n_instr = plan.host_instruction_count
            by_block = {}
            for (_, phys, a, d) in r1.buffer_events:
                by_block.setdefault(phys, []).append((a, n_instr if d < 0 else d))
            for iv in by_block.values():
                iv.sort()
                assert all(iv[i - 1][1] <= iv[i][0] for i in range(1, len(iv)))


def test_static_fallback_agreement(gpu, ref, fixtures):
    """Criterion 7 at runtime: static == dynamic within 1e-6."""
    from test_compiler_parity import _static_variant
    for name in FIXTURES:
        g = _static_variant(fixtures, name)
        s = gpu.compile_graph(g, gpu.CompileOptions(static_fallback=True))
        d = gpu.compile_graph(g)
        inputs = ref.make_binding(g, {}, 11)
        check_outputs(gpu.Executor().run(s, inputs).outputs, gpu.Executor().run(d, inputs).outputs, tol=1e-6)


def test_version_soundness(gpu, ref, fixtures):
    """Criterion 8: every passing version of every kernel agrees with the scalar
    catch-all on the device (run_kernel), and exactly one effective guard matches."""
    checked = 0
    for name in FIXTURES:
        g = fixtures[name]["graph"]
        plan = gpu.compile_graph(g)
        pj = json.loads(plan.to_json())
        rp = ref.RefPlan(plan.to_json())
        ex = gpu.Executor()
        for b in range(0, 50, 5):
            inputs = ref.make_binding(g, fixture_binding(name, 1 + (b % 25)), 500 + b)
            regs = plan.eval_shapes([inputs[i["id"]].shape for i in pj["inputs"]])
            env = _buffer_values(ref, g, inputs)
            for ins in pj["instrs"]:
                if ins["k"] != "launch":
                    continue
                k = ins["kernel"]
                art = pj["kernels"][k]
                ext = [env[pj["buffer_values"][bf]] for bf in ins["inputs"]]
                ext = [x.reshape(O.resolve_dims(art["external_input_dims"][i], regs)) for i, x in enumerate(ext)]
                want = rp.run_kernel(k, art["versions"][-1]["id"], ext, regs)
                eff = 0
                for vi, v in enumerate(art["versions"]):
                    raw = gpu.guard_passes(plan, k, v["id"], regs)
                    assert raw == rp.guard_passes(k, v["id"], regs)
                    earlier = any(gpu.guard_passes(plan, k, u["id"], regs) for u in art["versions"][:vi])
                    eff += raw and not earlier
                    if raw:
                        got = ex.run_kernel(plan, k, v["id"], ext, regs)
                        check_outputs(got, want, tol=1e-6, ctx=f"{name} kernel {k} v{v['id']}")
                        checked += 1
                assert eff == 1
    assert checked > 0


def _buffer_values(ref, g, inputs):
    """Every DHLO value of the graph (plan buffers are named by these ids), evaluated
    eagerly with the numpy restatement of each op."""
    dh = json.loads(ref.lower_dhlo_json(g))
    # Evaluate the lowered DHLO eagerly through the numpy restatement of each op.
    vals = dict(inputs)
    for op in dh["ops"]:
        kind = op["kind"]
        args = [vals.get(a) for a in op["inputs"]]
        if kind == "constant":
            lit = op["literal"]
            vals[op["id"]] = np.array(lit.get("f32", lit.get("i64")), dtype=np.float32 if lit["dtype"] == "f32"
                                      else np.int64).reshape(lit["dims"])
        elif kind == "shape_of":
            vals[op["id"]] = np.array(args[0].shape, dtype=np.int64)
        elif kind == "extract_dim":
            vals[op["id"]] = np.array([args[0][op["index"]]], dtype=np.int64)
        elif kind == "scalar_arith":
            a, b = int(args[0][0]), int(args[1][0])
            f = {"add": a + b, "sub": a - b, "mul": a * b, "div": int(a / b) if b else 0,
                 "ceil_div": (a + b - 1) // b if b > 0 else 0}[op["arith"]]
            vals[op["id"]] = np.array([f], dtype=np.int64)
        elif kind == "concat" and op["dtype"] == "i64":
            vals[op["id"]] = np.concatenate(args)
        elif kind in ("add", "sub", "mul", "div", "maximum"):
            vals[op["id"]] = O.apply_binary(kind, args[0], args[1])
        elif kind in ("exp", "tanh", "neg"):
            vals[op["id"]] = O.apply_unary(kind, args[0])
        elif kind in ("reduce_sum", "reduce_max"):
            vals[op["id"]] = O.eval_reduce(kind, args[0], op["dims"])
        elif kind == "dynamic_broadcast_in_dim":
            vals[op["id"]] = O.eval_broadcast(args[0], [int(x) for x in args[1]], op["dims"])
        elif kind == "dynamic_reshape":
            vals[op["id"]] = args[0].reshape([int(x) for x in args[1]])
        elif kind == "dynamic_slice":
            st, li, sd = [list(map(int, a)) for a in args[1:4]]
            idx = tuple(slice(s, l, d) for s, l, d in zip(st, li, sd))
            vals[op["id"]] = np.array(args[0][idx], dtype=np.float32)
        elif kind == "dynamic_pad":
            vals[op["id"]] = O.eval_pad(args[0], float(args[1]), *[list(map(int, a)) for a in args[2:5]])
        elif kind == "transpose":
            vals[op["id"]] = O.eval_transpose(args[0], op["dims"])
        elif kind == "concat":
            vals[op["id"]] = O.eval_concat(args, op["axis"])
        elif kind == "matmul":
            vals[op["id"]] = O.eval_matmul(args[0], args[1])
    return vals


EDGE_CASES = [
    ('{"name": "sm1", "inputs": [{"id": "x", "shape": ["S0"], "dtype": "f32"}], "outputs": ["y"],'
     ' "nodes": [{"id": "y", "op": "Softmax", "inputs": ["x"]}]}', {"S0": 7}),
    ('{"name": "red2", "inputs": [{"id": "x", "shape": ["S0", 3, "S1"], "dtype": "f32"}], "outputs": ["y"],'
     ' "nodes": [{"id": "y", "op": "ReduceSum", "inputs": ["x"], "attrs": {"axes": [0, 2]}}]}', {"S0": 4, "S1": 5}),
    ('{"name": "cat3", "inputs": [{"id": "a", "shape": ["S0", 2], "dtype": "f32"},'
     ' {"id": "b", "shape": ["S0", 3], "dtype": "f32"}, {"id": "c", "shape": ["S0", 4], "dtype": "f32"}],'
     ' "outputs": ["y"], "nodes": [{"id": "y", "op": "Concat", "inputs": ["a", "b", "c"], "attrs": {"axis": 1}}]}',
     {"S0": 3}),
    ('{"name": "slice1", "inputs": [{"id": "x", "shape": [10], "dtype": "f32"}], "outputs": ["y"],'
     ' "nodes": [{"id": "y", "op": "Slice", "inputs": ["x"], "attrs": {"starts": [2], "limits": [9], "strides": [3]}}]}',
     {}),
    ('{"name": "mm_out", "inputs": [{"id": "a", "shape": ["S0", 6], "dtype": "f32"},'
     ' {"id": "b", "shape": [6, 5], "dtype": "f32"}], "outputs": ["y"],'
     ' "nodes": [{"id": "y", "op": "MatMul", "inputs": ["a", "b"]}]}', {"S0": 4}),
    ('{"name": "split4", "inputs": [{"id": "x", "shape": ["S0", 3], "dtype": "f32"}],'
     ' "outputs": ["a0", "a1", "a2", "a3"], "nodes": [{"id": "s", "op": "Split", "inputs": ["x"],'
     ' "attrs": {"num_splits": 4, "axis": 0}, "outputs": ["p0", "p1", "p2", "p3"]},'
     ' {"id": "a0", "op": "Exp", "inputs": ["p0"]}, {"id": "a1", "op": "Tanh", "inputs": ["p1"]},'
     ' {"id": "a2", "op": "Neg", "inputs": ["p2"]}, {"id": "a3", "op": "Exp", "inputs": ["p3"]}]}', {"S0": 8}),
    ('{"name": "idgraph", "inputs": [{"id": "x", "shape": ["S0", 2], "dtype": "f32"}], "outputs": ["x"],'
     ' "nodes": []}', {"S0": 3}),
    ('{"name": "pass", "inputs": [{"id": "x", "shape": ["S0"], "dtype": "f32"}], "outputs": ["y", "x", "y"],'
     ' "nodes": [{"id": "y", "op": "Exp", "inputs": ["x"]}]}', {"S0": 5}),
    ('{"name": "pad2", "inputs": [{"id": "x", "shape": ["S0", 3], "dtype": "f32"}], "outputs": ["y"],'
     ' "nodes": [{"id": "y", "op": "Pad", "inputs": ["x"], "attrs": {"low": [1, 0], "high": [0, 2],'
     ' "interior": [2, 1], "value": 0.5}}]}', {"S0": 4}),
    ('{"name": "tr3", "inputs": [{"id": "x", "shape": ["S0", 3, 5], "dtype": "f32"}], "outputs": ["y"],'
     ' "nodes": [{"id": "y", "op": "Transpose", "inputs": ["x"], "attrs": {"perm": [2, 0, 1]}}]}', {"S0": 6}),
    ('{"name": "colred", "inputs": [{"id": "x", "shape": ["N", "C"], "dtype": "f32"}, {"id": "b", "shape": ["C"]}],'
     ' "outputs": ["r"], "nodes": [{"id": "bb", "op": "Broadcast", "inputs": ["b"], "attrs": {"shape": ["N", "C"],'
     ' "broadcast_dims": [1]}}, {"id": "a", "op": "Add", "inputs": ["x", "bb"]},'
     ' {"id": "t", "op": "Tanh", "inputs": ["a"]}, {"id": "m", "op": "Mul", "inputs": ["t", "x"]},'
     ' {"id": "r", "op": "ReduceSum", "inputs": ["m"], "attrs": {"axes": [0]}}]}', {"N": 1000, "C": 36}),
    ('{"name": "midred", "inputs": [{"id": "x", "shape": ["A", "B", "C"], "dtype": "f32"}], "outputs": ["r", "e"],'
     ' "nodes": [{"id": "e", "op": "Exp", "inputs": ["x"]}, {"id": "r", "op": "ReduceMax", "inputs": ["e"],'
     ' "attrs": {"axes": [1]}}]}', {"A": 3, "B": 77, "C": 20}),
]


@pytest.mark.parametrize("i", range(len(EDGE_CASES)))
def test_edge_shapes(gpu, ref, i):
    g, syms = EDGE_CASES[i]
    inputs = ref.make_binding(g, syms, 91)
    for sched in ("auto", "materialize"):
        ex = gpu.Executor()
        ex.set_schedule(sched)
        check_outputs(ex.run(gpu.compile_graph(g), inputs).outputs, ref.eval_eager(g, inputs).outputs, tol=1e-6,
                      ctx=f"{i} {sched}")


def test_unfused_plans_bit_exact(gpu, ref, fixtures):
    """test_executor.cpp:317-332 restricted to IEEE ops: unfused add/sub/mul/div/max/neg
    plans are bit-exact; exp/tanh plans within 1e-6 (libdevice vs glibc ulp)."""
    g = ('{"name": "ieee", "inputs": [{"id": "x", "shape": ["S0", 4]}, {"id": "y", "shape": ["S0", 4]}],'
         ' "outputs": ["f"], "nodes": [{"id": "a", "op": "Add", "inputs": ["x", "y"]},'
         ' {"id": "b", "op": "Mul", "inputs": ["a", "x"]}, {"id": "c", "op": "Div", "inputs": ["b", "y"]},'
         ' {"id": "d", "op": "Maximum", "inputs": ["c", "x"]}, {"id": "e", "op": "Neg", "inputs": ["d"]},'
         ' {"id": "f", "op": "Sub", "inputs": ["e", "y"]}]}')
    inputs = ref.make_binding(g, {"S0": 5}, 81)
    got = gpu.Executor().run(gpu.compile_graph(g, gpu.CompileOptions(enable_fusion=False)), inputs).outputs
    np.testing.assert_array_equal(got[0], ref.eval_eager(g, inputs).outputs[0])
    # fused groups divide with a * rcp.approx(b) (<= 2 ulp): within 1e-6, not bit-exact
    got = gpu.Executor().run(gpu.compile_graph(g, gpu.CompileOptions(enable_fusion=True)), inputs).outputs
    check_outputs(got, ref.eval_eager(g, inputs).outputs, tol=1e-6)
    for name in ("chain", "softmax", "diamond"):
        fg = fixtures[name]["graph"]
        b = ref.make_binding(fg, {"S0": 5}, 81)
        got = gpu.Executor().run(gpu.compile_graph(fg, gpu.CompileOptions(enable_fusion=False)), b).outputs
        check_outputs(got, ref.eval_eager(fg, b).outputs, tol=1e-6)


def test_runtime_errors_match_reference(gpu, ref, fixtures):
    sp = fixtures["split"]["graph"]
    plan = gpu.compile_graph(sp)
    bad = ref.make_binding(sp, {"S0": 6, "T0": 6, "T1": 4}, 9)
    with pytest.raises(gpu.DiscError) as e:
        gpu.Executor().run(plan, bad)
    with pytest.raises(ref.RefError) as r:
        ref.RefPlan(ref.compile(sp)).run(bad)
    assert str(e.value) == str(r.value) and "violates a shape constraint" in str(e.value)
    ch = gpu.compile_graph(fixtures["chain"]["graph"])
    with pytest.raises(gpu.DiscError, match="missing input"):
        gpu.Executor().run(ch, {})
    with pytest.raises(gpu.DiscError, match="rank"):
        gpu.Executor().run(ch, {"x": np.ones(4, np.float32)})


def test_device_inputs_and_large_softmax_property(gpu):
    """Full-size property check: softmax rows sum to 1 and match a float64 numpy softmax."""
    g = '{"name": "sm", "inputs": [{"id": "x", "shape": ["B", "S"]}], "outputs": ["y"], "nodes": [{"id": "y", "op": "Softmax", "inputs": ["x"]}]}'
    plan = gpu.compile_graph(g)
    ex = gpu.Executor()
    for B, S in [(4096, 4096), (65536, 33), (3, 100003), (1, 1), (8, 4095)]:
        x = gpu.DeviceBuffer((B, S)).fill_uniform(B * 131 + S)
        ex.run_device(plan, {"x": x})
        y = ex.fetch_outputs()[0]
        xs = x.numpy().astype(np.float64)
        e = np.exp(xs - xs.max(axis=1, keepdims=True))
        want = e / e.sum(axis=1, keepdims=True)
        assert np.max(np.abs(y - want) / np.maximum(1.0, np.abs(want))) <= 1e-5
        np.testing.assert_allclose(y.sum(axis=1), 1.0, rtol=1e-4)


def test_generated_kernels_match_interpreter(gpu):
    """Generated straight-line kernels are used for the library patterns and produce
    results bit-identical to the interpreter (same ops, same order)."""
    from paper_2103_05288_b200 import workloads as W
    cases = [(W.ln_gelu_graph(), {"T": 333, "H": 768}), (W.ln_gelu_graph(), {"T": 5, "H": 1000}),
             (W.softmax_graph_for(0), {"S0": 77, "S1": 4096}), (W.softmax_graph_for(0), {"S0": 300, "S1": 7}),
             (W.colreduce_graph(), {"N": 5000, "C": 260}), (W.colreduce_graph(), {"N": 100000, "C": 3}),
             (W.bert_graph(), {"R": 12 * 2 * 64, "S": 64, "T": 128, "H": 768, "F": 3072})]
    rng = np.random.default_rng(5)
    for g, syms in cases:
        plan = gpu.compile_graph(g)
        inputs = {i["id"]: rng.uniform(0.25, 2.0, size=[syms[d] if isinstance(d, str) else d for d in i["shape"]])
                  .astype(np.float32) for i in g["inputs"]}
        ex = gpu.Executor()
        before = gpu.specialized_launches()
        fast = ex.run(plan, inputs).outputs
        assert gpu.specialized_launches() > before, (g["name"], syms)
        gpu.set_specialization(False)
        try:
            slow = ex.run(plan, inputs).outputs
        finally:
            gpu.set_specialization(True)
        for a, b in zip(fast, slow):
            np.testing.assert_array_equal(a, b)
        want, _, _ = O.Executor().run(plan.to_json(), inputs)
        check_outputs(fast, want)


def test_transcendental_accuracy(gpu):
    """exp/tanh on the device against float64 numpy over a dense argument sweep (incl.
    subnormal/tiny, large and saturating arguments), held to TRUE relative error (not the
    reference's floored rel_err): tanh <= 2e-6 everywhere and over every f32 in [2^-12, 1]
    (odd polynomial below 0.5, MUFU ex2/rcp form above; program.cuh tanh_fast), exp within
    2.5e-7 relative."""
    every = np.arange(np.float32(2 ** -12).view(np.int32), np.float32(1.0).view(np.int32), 7,
                      dtype=np.int32).view(np.float32)
    for op, ref_fn, tol in (("Tanh", np.tanh, 2e-6), ("Exp", np.exp, 2.5e-7)):
        g = json.dumps({"name": "t", "inputs": [{"id": "x", "shape": ["N"]}], "outputs": ["y"],
                        "nodes": [{"id": "y", "op": op, "inputs": ["x"]}]})
        lim = 20.0 if op == "Tanh" else 80.0
        x = np.concatenate([np.linspace(-lim, lim, 2_000_003, dtype=np.float32),
                            np.float32(1e-30) * np.arange(-50, 50, dtype=np.float32),
                            np.array([0.0, -0.0, 1e-7, -1e-7, 0.49999, 0.5, 0.50001, 0.59999, 0.6, 0.60001, 9.0,
                                      9.02, 88.0], np.float32), every, -every])
        y = gpu.Executor().run(gpu.compile_graph(g), {"x": x}).outputs[0].astype(np.float64)
        want = ref_fn(x.astype(np.float64))
        nz = want != 0
        err = np.abs(y[nz] - want[nz]) / np.abs(want[nz])
        assert float(err.max()) <= tol, (op, float(err.max()), float(x[nz][np.argmax(err)]))
        if op == "Tanh":  # tiny arguments are returned exactly (sign and value)
            tiny = np.abs(x) < 2.44140625e-4
            np.testing.assert_array_equal(y[tiny], x[tiny].astype(np.float64))
            assert np.array_equal(np.signbit(y[tiny]), np.signbit(x[tiny]))
            band = (np.abs(x) >= 2 ** -12) & (np.abs(x) <= 1.0)
            band_err = np.abs(y[band] - want[band]) / np.abs(want[band])
            print(f"tanh true-relative error on [2^-12, 1]: {band_err.max():.3g}")
            assert band_err.max() <= 2e-6


def test_gemm_library_call(gpu, ref):
    """kLibraryCall (eval_matmul, kernels.cpp:261-303) at transformer sizes: within 1e-5
    of the f64-accumulated product (floored rel_err), and the matmul fixture plan against
    the reference executor."""
    rng = np.random.default_rng(3)
    for m, k, n in ((512, 768, 3072), (333, 3072, 768), (1, 5, 7), (64, 0, 16)):
        g = json.dumps({"name": "mm", "inputs": [{"id": "a", "shape": ["M", k]}, {"id": "b", "shape": [k, "N"]}],
                        "outputs": ["c"], "nodes": [{"id": "c", "op": "MatMul", "inputs": ["a", "b"]}]})
        a = rng.uniform(0.25, 2.0, size=(m, k)).astype(np.float32)
        b = rng.uniform(-1.0, 1.0, size=(k, n)).astype(np.float32)
        got = gpu.Executor().run(gpu.compile_graph(g), {"a": a, "b": b}).outputs[0]
        want = (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
        assert O.rel_err(got, want) <= 1e-5, (m, k, n, O.rel_err(got, want))


def test_static_plans_replay_as_cuda_graphs(gpu, ref, fixtures):
    """Static plans (static_specialize: no shape program) are captured on the second
    identical run and replayed afterwards (one graph launch per run); outputs equal the
    graph-free executor's and the reference's, with new input values each run."""
    from test_compiler_parity import _static_variant
    for name in ("softmax", "transformer", "chain"):
        g = _static_variant(fixtures, name)
        plan = gpu.static_specialize(g)
        ex, plain = gpu.Executor(0, gpu.new_stream()), gpu.Executor(0, gpu.new_stream())
        plain.set_graphs(False)
        for it in range(7):
            inputs = ref.make_binding(g, {}, 100 + it)
            before = gpu.kernel_launches()
            got = ex.run(plan, inputs)
            launched = gpu.kernel_launches() - before
            want = plain.run(plan, inputs)
            for a, b in zip(got.outputs, want.outputs):
                np.testing.assert_array_equal(a, b)
            assert got.stats.as_dict() == want.stats.as_dict()
            if it >= 4:
                assert launched == 1, (name, it, launched)
        assert ex.graph_replays() >= 1, name
    # dynamic plans never use graphs
    dyn = gpu.compile_graph(fixtures["softmax"]["graph"])
    ex = gpu.Executor(0, gpu.new_stream())
    for it in range(3):
        ex.run(dyn, ref.make_binding(fixtures["softmax"]["graph"], {"S0": 5}, it))
    assert ex.graph_replays() == 0


def test_odd_width_rows(gpu, ref, fixtures):
    """Odd row widths (R % 4 != 0) run the float4 body + scalar head/tail row kernel;
    softmax and the BERT attention subgraph against the reference executor, every row's
    alignment phase covered (R = 33 .. 4095)."""
    from paper_2103_05288_b200 import workloads as W
    sm = fixtures["softmax"]["graph"]
    plan = gpu.compile_graph(sm)
    rp = ref.RefPlan(ref.compile(sm))
    for B, S in [(7, 33), (5, 255), (3, 777), (2, 1001), (2, 4095), (9, 65)]:
        g = json.loads(sm)
        inputs = {g["inputs"][0]["id"]: np.random.default_rng(S).uniform(0.25, 2.0, size=(B, S)).astype(np.float32)}
        check_outputs(gpu.Executor().run(plan, inputs).outputs, rp.run(inputs).outputs, ctx=f"softmax {B}x{S}")
    bg = W.bert_graph()
    bplan = gpu.compile_graph(bg)
    brp = ref.RefPlan(ref.compile(json.dumps(bg)))
    syms = {"R": 12 * 37, "S": 37, "T": 37, "H": 768, "F": 3072}
    rng = np.random.default_rng(1)
    inputs = {}
    for i in bg["inputs"]:
        shape = [syms[d] if isinstance(d, str) else d for d in i["shape"]]
        cv = W.CONST_INPUTS.get(i["id"]) if i["id"] != "inv_h" else 1.0 / 768
        inputs[i["id"]] = (np.full(shape, cv, np.float32) if cv is not None
                           else rng.uniform(0.25, 2.0, size=shape).astype(np.float32))
    check_outputs(gpu.Executor().run(bplan, inputs).outputs, brp.run(inputs).outputs, ctx="bert S=37")


SPLIT_ROW_CASES = [
    # full reduction [N] -> [] / [1]-like, column sums of [N, 1], a handful of long rows, max
    ('{"name": "full", "inputs": [{"id": "x", "shape": ["N"], "dtype": "f32"}], "outputs": ["r"],'
     ' "nodes": [{"id": "r", "op": "ReduceSum", "inputs": ["x"], "attrs": {"axes": [0]}}]}', {"N": 3000001}),
    ('{"name": "col1", "inputs": [{"id": "x", "shape": ["N", "C"], "dtype": "f32"}, {"id": "b", "shape": ["C"]}],'
     ' "outputs": ["r"], "nodes": [{"id": "bb", "op": "Broadcast", "inputs": ["b"], "attrs": {"shape": ["N", "C"],'
     ' "broadcast_dims": [1]}}, {"id": "a", "op": "Add", "inputs": ["x", "bb"]},'
     ' {"id": "t", "op": "Tanh", "inputs": ["a"]}, {"id": "m", "op": "Mul", "inputs": ["t", "x"]},'
     ' {"id": "r", "op": "ReduceSum", "inputs": ["m"], "attrs": {"axes": [0]}}]}', {"N": 1 << 21, "C": 1}),
    ('{"name": "rows", "inputs": [{"id": "x", "shape": ["K", "R"], "dtype": "f32"}], "outputs": ["r"],'
     ' "nodes": [{"id": "e", "op": "Exp", "inputs": ["x"]}, {"id": "r", "op": "ReduceSum", "inputs": ["e"],'
     ' "attrs": {"axes": [1]}}]}', {"K": 3, "R": 400003}),
    ('{"name": "rmax", "inputs": [{"id": "x", "shape": ["K", "R"], "dtype": "f32"}], "outputs": ["r"],'
     ' "nodes": [{"id": "r", "op": "ReduceMax", "inputs": ["x"], "attrs": {"axes": [1]}}]}', {"K": 100, "R": 65536}),
]


@pytest.mark.parametrize("i", range(len(SPLIT_ROW_CASES)))
def test_few_long_rows_split_across_ctas(gpu, ref, i):
    """Few long rows without an epilogue run on the column machinery (R split across CTAs,
    f64 partials joined in order): same results as the reference, and the schedule is not
    the one-group-per-row kernel."""
    g, syms = SPLIT_ROW_CASES[i]
    inputs = ref.make_binding(g, syms, 5)
    ex = gpu.Executor()
    got = ex.run(gpu.compile_graph(g), inputs)
    check_outputs(got.outputs, ref.eval_eager(g, inputs).outputs, ctx=g[:30])
    scheds = [r["schedule"] for r in ex.launch_records()]
    assert any(s.startswith("col") for s in scheds), scheds


COLRED = ('{"name": "colred", "inputs": [{"id": "x", "shape": ["N", "C"], "dtype": "f32"}, {"id": "b", "shape": ["C"]}],'
          ' "outputs": ["r"], "nodes": [{"id": "bb", "op": "Broadcast", "inputs": ["b"], "attrs": {"shape": ["N", "C"],'
          ' "broadcast_dims": [1]}}, {"id": "a", "op": "Add", "inputs": ["x", "bb"]},'
          ' {"id": "t", "op": "Tanh", "inputs": ["a"]}, {"id": "m", "op": "Mul", "inputs": ["t", "x"]},'
          ' {"id": "r", "op": "ReduceSum", "inputs": ["m"], "attrs": {"axes": [0]}}]}')
COLMAX = ('{"name": "colmax", "inputs": [{"id": "x", "shape": ["N", "C"], "dtype": "f32"}], "outputs": ["r"],'
          ' "nodes": [{"id": "e", "op": "Exp", "inputs": ["x"]}, {"id": "r", "op": "ReduceMax", "inputs": ["e"],'
          ' "attrs": {"axes": [0]}}]}')


@pytest.mark.parametrize("g", [COLRED, COLMAX])
@pytest.mark.parametrize("schedule", ["auto", "atomic"])
def test_folded_column_reduce(gpu, ref, g, schedule):
    """Column reduces with C % 4 != 0 fold 2 or 4 rows into float4 super rows (tiled bias,
    partial last super row, folded finalize): every N mod f tail and both finalize forms
    against the reference executor."""
    ex = gpu.Executor()
    ex.set_schedule(schedule)
    plan = gpu.compile_graph(g)
    if schedule == "atomic" and "ReduceMax" in g:
        pytest.skip("atomic schedules are sum-only")
    seen = set()
    for c in (1, 2, 3, 5, 6, 7, 33, 130):
        for n in (64, 65, 66, 67, 1001, 40003):
            inputs = ref.make_binding(g, {"N": n, "C": c}, n + c)
            got = ex.run(plan, inputs)
            check_outputs(got.outputs, ref.eval_eager(g, inputs).outputs, ctx=f"C={c} N={n}")
            seen |= {r["schedule"] for r in ex.launch_records()}
    assert any("fold" in s for s in seen), seen


def test_column_reduce_special_values(gpu, ref):
    """The XU-heavy column pass converts f32 -> f64 on the integer pipe (kernels.cuh
    f2d_bits); zeros, signed zeros, subnormals, infinities and NaNs must take the hardware
    conversion: every output equals the reference's (NaN where the reference has NaN,
    matching infinities), for columns with and without special values in one warp."""
    import numpy as np
    ex = gpu.Executor()
    plan = gpu.compile_graph(COLRED)
    rng = np.random.default_rng(11)
    for n, c in ((4096, 256), (777, 1024), (20000, 64)):
        x = rng.uniform(0.25, 2.0, size=(n, c)).astype(np.float32)
        b = rng.uniform(0.25, 2.0, size=(c,)).astype(np.float32)
        x[:, 1] = 0.0
        x[::7, 2] = -0.0
        x[::5, 3] = 1e-40  # subnormal
        x[3, 4] = np.inf
        x[5, 5] = -np.inf
        x[9, 6] = np.nan
        x[:, 8] = -x[:, 8]
        x[::3, 9] = np.float32(1e-39) * -1
        inputs = {"x": x, "b": b}
        got = ex.run(plan, inputs).outputs[0]
        want = ref.eval_eager(COLRED, inputs).outputs[0]
        assert np.array_equal(np.isnan(got), np.isnan(want)), (n, c)
        fin = np.isfinite(want)
        assert np.array_equal(got[~fin & ~np.isnan(want)], want[~fin & ~np.isnan(want)]), (n, c)
        check_outputs([np.where(fin, got, 0)], [np.where(fin, want, 0)], ctx=f"special N={n} C={c}")
