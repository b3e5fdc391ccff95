"""Host compile pipeline parity: shape propagation, constraints,
fusion plans, buffer plans and the generated runtime flow must be BIT-EXACT with the
reference -- checked as byte-identical plan JSON, stage dumps and cache keys."""
import json
import random

import numpy as np
import pytest

from conftest import FIXTURES, OPTION_SETS, REF_FLAGS


def opts(disc, name):
    return disc.CompileOptions(**OPTION_SETS[name])


@pytest.mark.parametrize("opt", list(OPTION_SETS))
def test_fixture_plans_byte_identical(disc, fixtures, fixture_plans, opt):
    for name in FIXTURES:
        mine = disc.compile_graph(fixtures[name]["graph"], opts(disc, opt)).to_json()
        assert mine == fixture_plans[f"{name}/{opt}"], f"{name}/{opt}"


def test_random_plans_byte_identical(disc, random_plans):
    for seed, v in random_plans.items():
        assert disc.compile_graph(v["graph"]).to_json() == v["plan"], seed


def test_reference_goldens(disc, fixtures, reference_goldens):
    """tests/golden/softmax_{ir.txt,dhlo.json,plan.json} pinned by test_dhlo.cpp:159-173,
    test_plan.cpp:144-150."""
    g = fixtures["softmax"]["graph"]
    assert disc.compile_graph(g).to_json() == reference_goldens["softmax_plan.json"]
    assert disc.lower_dhlo_json(g) == reference_goldens["softmax_dhlo.json"]
    assert disc.dump_stage(g, "dhlo") == reference_goldens["softmax_ir.txt"]
    assert disc.dhlo_roundtrip(reference_goldens["softmax_dhlo.json"]) == reference_goldens["softmax_dhlo.json"]


def test_plan_json_round_trip_and_check(disc, fixtures, fixture_plans):
    for k, text in fixture_plans.items():
        p = disc.CompiledPlan.from_json(text)
        assert p.to_json() == text
        assert p.check() == []


def test_launch_and_op_counts(disc, fixtures):
    """Structural KATs: softmax 2 kernels / 7 eager ops, transformer 14 kernels + 4 GEMMs /
    54 eager ops (acceptance_main.cpp:123-147)."""
    sm = disc.compile_graph(fixtures["softmax"]["graph"])
    assert sm.eager_op_count == 7 and sm.num_kernels == 2
    tf = disc.compile_graph(fixtures["transformer"]["graph"])
    assert tf.eager_op_count == 54 and tf.num_kernels == 14
    plan = json.loads(tf.to_json())
    assert sum(1 for i in plan["instrs"] if i["k"] == "library_call") == 4
    split = json.loads(disc.compile_graph(fixtures["split"]["graph"]).to_json())
    split_no = json.loads(disc.compile_graph(fixtures["split"]["graph"],
                                             disc.CompileOptions(inject_constraints=False)).to_json())
    assert len(split["kernels"]) == 1 and len(split_no["kernels"]) == 2


def test_compile_once_plan_cache(disc, fixtures):
    """Criterion 2 (compile side): graphs that differ only in dim values or symbol names
    share one plan; 99 recompiles are cache hits."""
    for name in FIXTURES:
        c = disc.Compiler()
        c.compile(fixtures[name]["graph"])
        for _ in range(99):
            c.compile(fixtures[name]["graph"])
        assert c.stats() == {"compile_count": 1, "cache_hits": 99}
    c = disc.Compiler()
    base = json.loads(fixtures["softmax"]["graph"])
    for i in range(1, 101):
        g = json.loads(json.dumps(base))
        g["inputs"][0]["shape"] = [f"Sym{i}", 8 + i]  # new names and constants: same key
        c.compile(json.dumps(g))
    assert c.stats() == {"compile_count": 1, "cache_hits": 99}


def test_determinism(disc, fixtures):
    for name in FIXTURES:
        g = fixtures[name]["graph"]
        assert disc.compile_graph(g).to_json() == disc.compile_graph(g).to_json()


def test_shape_program_slice_and_pad(disc):
    """Criterion 6 (acceptance_main.cpp:259-311), via the host EvalShape."""
    rng = random.Random(4242)
    for _ in range(300):
        start = rng.randrange(101)
        limit = start + rng.randrange(101 - start)
        stride = 1 + rng.randrange(5)
        g = {"name": "g", "inputs": [{"id": "x", "shape": [max(limit, 1)], "dtype": "f32"}], "outputs": ["s"],
             "nodes": [{"id": "s", "op": "Slice", "inputs": ["x"],
                        "attrs": {"starts": [start], "limits": [limit], "strides": [stride]}}]}
        p = json.loads(disc.compile_graph(g).to_json())
        assert p["outputs"][0]["dims"][0]["c"] == len(range(start, limit, stride))
    for _ in range(300):
        n, lo, hi, it = rng.randrange(30), rng.randrange(6), rng.randrange(6), rng.randrange(5)
        g = {"name": "g", "inputs": [{"id": "x", "shape": ["S"], "dtype": "f32"}], "outputs": ["p"],
             "nodes": [{"id": "p", "op": "Pad", "inputs": ["x"],
                        "attrs": {"low": [lo], "high": [hi], "interior": [it], "value": 0.0}}]}
        plan = disc.compile_graph(g)
        regs = plan.eval_shapes([[n]])
        out = json.loads(plan.to_json())["outputs"][0]["dims"][0]
        assert "r" in out
        assert regs[out["r"]] == lo + hi + n + max(n - 1, 0) * it


# --- live comparison against the reference build (test infrastructure) -------------

@pytest.mark.parametrize("opt", ["default", "no_inject", "no_fusion"])
def test_random_graphs_live(disc, ref, opt):
    for seed in range(200, 700):
        g = ref.random_graph(seed, 12)
        want = ref.compile(g, **REF_FLAGS[opt])
        assert disc.compile_graph(g, opts(disc, opt)).to_json() == want, seed


@pytest.mark.parametrize("stage", ["dhlo", "constraints", "simplified", "fused", "program"])
def test_stage_dumps_live(disc, ref, fixtures, stage):
    for name in FIXTURES:
        g = fixtures[name]["graph"]
        assert disc.dump_stage(g, stage) == ref.dump_stage(g, stage), (name, stage)
        assert disc.dump_stage(g, stage, disc.CompileOptions(inject_constraints=False)) == \
            ref.dump_stage(g, stage, inject=False), (name, stage)
    for seed in range(60):
        g = ref.random_graph(seed, 12)
        assert disc.dump_stage(g, stage) == ref.dump_stage(g, stage), (seed, stage)


def test_cache_keys_live(disc, ref, fixtures):
    for name in FIXTURES:
        for opt in OPTION_SETS:
            assert disc.cache_key(fixtures[name]["graph"], opts(disc, opt)) == \
                ref.cache_key(fixtures[name]["graph"], **REF_FLAGS[opt])
    for seed in range(100):
        g = ref.random_graph(seed, 12)
        assert disc.cache_key(g) == ref.cache_key(g)


def _static_variant(fx, name):
    syms = fx[name]["bindings"][-1]
    g = json.loads(fx[name]["graph"])
    sub = lambda shape: [syms.get(d, d) if isinstance(d, str) else d for d in shape]
    for i in g["inputs"]:
        i["shape"] = sub(i["shape"])
    for n in g["nodes"]:
        if "attrs" in n and "shape" in n["attrs"]:
            n["attrs"]["shape"] = sub(n["attrs"]["shape"])
    return json.dumps(g)


def test_static_specialization_live(disc, ref, fixtures):
    """Criterion 7 (compile side): static plans are byte-identical, zero EvalShape."""
    for name in FIXTURES:
        g = _static_variant(fixtures, name)
        mine = disc.compile_graph(g, disc.CompileOptions(static_fallback=True)).to_json()
        assert mine == ref.compile(g, static_fallback=True)
        assert not any(i["k"] == "eval_shape" for i in json.loads(mine)["instrs"])
        assert disc.static_specialize(g).to_json() == ref.static_specialize(g)
    with pytest.raises(disc.DiscError) as e:
        disc.static_specialize(fixtures["softmax"]["graph"])
    with pytest.raises(ref.RefError) as r:
        ref.static_specialize(fixtures["softmax"]["graph"])
    assert str(e.value) == str(r.value) and e.value.code == 3


BAD_GRAPHS = [
    "{not json",
    "[]",
    '{"inputs": [], "outputs": []}',
    '{"inputs": [{"id": "x", "shape": [2]}], "outputs": ["x"], "nodes": [{"id": "y", "op": "Foo", "inputs": ["x"]}]}',
    '{"inputs": [{"id": "x", "shape": [2]}], "outputs": ["y"], "nodes": [{"id": "y", "op": "Add", "inputs": ["x"]}]}',
    '{"inputs": [{"id": "x", "shape": [2, 3]}], "outputs": ["y"], "nodes": [{"id": "y", "op": "ReduceSum", "inputs": ["x"], "attrs": {"axes": [2]}}]}',
    '{"inputs": [{"id": "x", "shape": [2, 3]}], "outputs": ["y"], "nodes": [{"id": "y", "op": "ReduceSum", "inputs": ["x"]}]}',
    '{"inputs": [{"id": "x", "shape": [2, 3]}], "outputs": ["y"], "nodes": [{"id": "y", "op": "Transpose", "inputs": ["x"], "attrs": {"perm": [0, 0]}}]}',
    '{"inputs": [{"id": "x", "shape": [2, 3]}], "outputs": ["y"], "nodes": [{"id": "y", "op": "Reshape", "inputs": ["x"], "attrs": {"shape": [5]}}]}',
    '{"inputs": [{"id": "x", "shape": [2, 3]}], "outputs": ["y"], "nodes": [{"id": "y", "op": "Slice", "inputs": ["x"], "attrs": {"starts": [0, 0], "limits": [3, 3], "strides": [1, 1]}}]}',
    '{"inputs": [{"id": "x", "shape": [3, 3]}], "outputs": ["a"], "nodes": [{"id": "s", "op": "Split", "inputs": ["x"], "attrs": {"num_splits": 2, "axis": 0}, "outputs": ["a", "b"]}]}',
    '{"inputs": [{"id": "x", "shape": ["S", 2]}, {"id": "y", "shape": [3, 2]}], "outputs": ["z"], "nodes": [{"id": "z", "op": "Add", "inputs": ["x", "y"]}, {"id": "w", "op": "Add", "inputs": ["z", "z"], "bogus": 1}]}',
    '{"inputs": [{"id": "x", "shape": [2]}], "outputs": ["y"], "nodes": [{"id": "y", "op": "Broadcast", "inputs": ["x"], "attrs": {"shape": ["Q", 2]}}]}',
    '{"inputs": [{"id": "x", "shape": [2, 3]}], "outputs": ["y"], "nodes": [{"id": "y", "op": "Reshape", "inputs": ["x"], "attrs": {"shape": [-1, -1]}}]}',
    '{"inputs": [{"id": "x", "shape": [2], "dtype": "f16"}], "outputs": ["x"], "nodes": []}',
    '{"inputs": [{"id": "x", "shape": [-2]}], "outputs": ["x"], "nodes": []}',
    '{"inputs": [{"id": "x", "shape": [2]}], "outputs": ["q"], "nodes": []}',
    '{"inputs": [{"id": "x", "shape": [2]}, {"id": "x", "shape": [2]}], "outputs": ["x"], "nodes": []}',
    '{"inputs": [{"id": "x", "shape": [2, "S"]}, {"id": "y", "shape": [3, "S"]}], "outputs": ["z"], "nodes": [{"id": "z", "op": "MatMul", "inputs": ["x", "y"]}]}',
]


@pytest.mark.parametrize("i", range(len(BAD_GRAPHS)))
def test_error_parity_live(disc, ref, i):
    g = BAD_GRAPHS[i]
    try:
        ref.compile(g)
        ref_err = None
    except ref.RefError as e:
        ref_err = (e.code, str(e))
    try:
        disc.compile_graph(g)
        mine = None
    except disc.DiscError as e:
        mine = (e.code, str(e))
    assert mine == ref_err
