"""Grouped execution's flush plan, host only (no device): disc_plan_group_dry_run runs the
requests' runtime flows in capture mode and returns the actions the level-synchronous
flush would issue.  Pins the grouping rules of DESIGN.md §2.4 on CPU; the device-side
equivalence (bit-identical outputs) is tests/test_gpu_grouped.py."""
import json

import pytest


@pytest.fixture(scope="module")
def D():
    import paper_2103_05288_b200 as D
    D.lib()
    return D


def _reqs(D, graph, shape_list):
    from paper_2103_05288_b200 import workloads as W
    plan = D.compile_graph(graph)
    return plan, [(plan, W.input_shapes(graph, s)) for s in shape_list]


def test_c2_sweep_is_three_grouped_launches_per_phase(D):
    """192 variable-shape LN+GELU requests -> one grouped launch per plan kernel in each of
    the two flush phases (the largest eighth of the requests first, so the device starts
    while the host runs the other flows), members ordered by work (largest first), bytes =
    the requests' algorithmic bytes."""
    from paper_2103_05288_b200 import workloads as W
    g = W.ln_gelu_graph()
    plan, reqs = _reqs(D, g, W.ln_shapes())
    acts = D.group_dry_run(reqs)
    assert [a["action"] for a in acts] == ["group"] * 6
    assert [a["level"] for a in acts] == [0, 1, 2] * 2
    assert [a["kernel"] for a in acts] == [0, 1, 2] * 2
    assert [a["members"] for a in acts] == [len(reqs) // 8] * 3 + [len(reqs) - len(reqs) // 8] * 3
    assert all(a["generated"] for a in acts)
    assert min(acts[0]["order"]) >= max(acts[3]["order"])  # phase 1 = the largest requests
    for a in acts:
        assert a["order"] == sorted(a["order"], reverse=True)
        # compact member records: well under the full descriptor (4.6 / 9.3 KB)
        assert a["table_bytes"] / a["members"] < 4096
    want = sum(plan.algorithmic_bytes(shapes) for _, shapes in reqs)
    assert sum(a["bytes"] for a in acts) == want


def test_groups_split_by_kernel_instantiation(D):
    """Softmax over S = 1..4096: vec4 and scalar rows, staged short rows -- one group per
    kernel instantiation and level, every fused launch in exactly one group."""
    from paper_2103_05288_b200 import workloads as W
    g = W.softmax_graph_for(0)
    shapes = [{"S0": 64, "S1": s} for s in (1, 2, 3, 7, 8, 17, 31, 64, 100, 255, 256, 777, 1024, 4096)]
    plan, reqs = _reqs(D, g, shapes)
    acts = D.group_dry_run(reqs)
    fused = [a for a in acts if a["action"] in ("group", "alone")]
    for lv in (0, 1):
        assert sum(a["members"] for a in fused if a["level"] == lv) == len(reqs)
    # more than one instantiation per level (vector width / staging differ), fewer than requests
    assert 1 < sum(1 for a in fused if a["level"] == 0) < len(reqs)


def test_mixed_fixtures_and_host_threads_identical(D, fixtures):
    """Heterogeneous requests over every fixture graph, 20 bindings each: the plan is the
    same whether one thread or several worker threads queue them (merged queues)."""
    reqs = []
    for name in sorted(fixtures):
        f = fixtures[name]
        graph = json.loads(f["graph"]) if isinstance(f["graph"], str) else f["graph"]
        plan = D.compile_graph(graph)
        for syms in (f["bindings"] * 20)[:20]:
            shapes = {i["id"]: [syms.get(d, 2) if isinstance(d, str) else d for d in i["shape"]] for i in graph["inputs"]}
            reqs.append((plan, shapes))
    one = D.group_dry_run(reqs, host_threads=1)
    assert len(reqs) >= 128
    for t in (2, 4):
        assert D.group_dry_run(reqs, host_threads=t) == one
    kinds = {a["action"] for a in one}
    assert "group" in kinds
    # library calls and other non-fusible work are issued one by one, never grouped
    assert all(a["members"] == 1 for a in one if a["action"] == "single")


def test_stream_of_10k_requests_collapses(D):
    """C5: 10 000 distinct (graph, shape) requests over 10 graphs, one compile per graph;
    the flush issues a few hundred actions, not one launch per request kernel."""
    import bench
    wl = bench.make_workload("stream")
    graphs, reqs = wl.graphs, wl.requests(0)
    compiler = D.Compiler()
    plans = {k: compiler.compile(g) for k, g in graphs.items()}
    rq = [(plans[k], {i["id"]: bench.input_shape(i, s) for i in graphs[k]["inputs"]}) for k, s in reqs]
    assert compiler.stats()["compile_count"] == len(graphs)
    acts = D.group_dry_run(rq, host_threads=4)
    fused = sum(a["members"] for a in acts if a["action"] in ("group", "alone"))
    assert fused >= len(reqs)
    assert len(acts) < 600, len(acts)


@pytest.mark.parametrize("S,kind,vec", [(1, "loop", 4), (2, "row", 1), (777, "row", 4), (4095, "row", 4), (1024, "row", 4)])
def test_softmax_schedule_by_width(D, S, kind, vec):
    """Schedule selection by row width (host only, capture mode): single-element rows become
    one vectorised elementwise program, odd widths >= 32 the float4 body + scalar head/tail
    row kernel (vec 4), short odd rows stay scalar."""
    from paper_2103_05288_b200 import workloads as W
    plan = D.compile_graph(W.softmax_graph_for(0))
    recs = D.capture_programs(plan, {"x": [64, S]})
    assert [(r["kind"], r["vec"]) for r in recs] == [(kind, vec)] * 2


def test_odd_and_aligned_rows_never_share_a_group(D):
    from paper_2103_05288_b200 import workloads as W
    g = W.softmax_graph_for(0)
    plan, reqs = _reqs(D, g, [{"S0": 64, "S1": s} for s in (64, 255, 1024, 777)])
    acts = [a for a in D.group_dry_run(reqs) if a["action"] == "group" and a["level"] == 0]
    assert sorted(a["members"] for a in acts) == [2, 2]


@pytest.mark.parametrize("S,short,stage", [(2, 8, 0), (7, 8, 0), (9, 0, 0), (17, 0, 0), (31, 0, 0), (33, 0, 0)])
def test_softmax_short_rows(D, S, short, stage):
    """Scalar rows narrower than 8 floats run the register-resident thread-per-row kernel
    (unstaged: the warp-staged variant, stage 3, is an A/B knob, DISC_WARP_STAGE_MAX);
    wider ones the row kernels."""
    from paper_2103_05288_b200 import workloads as W
    plan = D.compile_graph(W.softmax_graph_for(0))
    recs = D.capture_programs(plan, {"x": [1000, S]})
    assert [(r["kind"], r["short"], r["stage"]) for r in recs] == [("row", short, stage)] * 2
