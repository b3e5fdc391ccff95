"""Multi-GPU request dispatch: host-side sharding logic on CPU, including a
world_size-2 gloo job; the in-process Dispatcher on the GPU.

The byte estimate that drives the sharding is checked against the §8d formula evaluated
by the oracle on the reference's own plan JSON (oracle/_ref), so the cost model is the
reference's, not ours.
"""
from __future__ import annotations

import json
import os
import random
import socket

import numpy as np
import pytest

import paper_2103_05288_b200 as D
from paper_2103_05288_b200 import workloads as W
from paper_2103_05288_b200.dispatch import shard, shard_loads


def test_shard_covers_disjoint_balanced():
    rng = random.Random(7)
    for world in (1, 2, 3, 8):
        costs = [rng.randint(0, 1 << 28) for _ in range(1000)]
        parts = shard(costs, world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(costs)))
        assert all(p == sorted(p) for p in parts)
        loads = shard_loads(costs, parts)
        # LPT bound: max load <= mean + largest item
        assert max(loads) <= sum(costs) / world + max(costs)
        assert parts == shard(costs, world)  # deterministic


def test_shard_edge_cases():
    assert shard([], 4) == [[], [], [], []]
    assert shard([5], 3) == [[0], [], []]
    assert shard([1, 1, 1, 1], 2) == [[0, 2], [1, 3]]
    with pytest.raises(ValueError):
        shard([1], 0)


def _stream_requests(n):
    graphs, reqs = W.mixed_stream(n)
    plans = {k: D.compile_graph(g) for k, g in graphs.items()}
    return graphs, plans, reqs


def test_plan_bytes_match_reference_formula(ref):
    """CompiledPlan.algorithmic_bytes == SURVEY §8d bytes on the reference plan."""
    from oracle import disc_oracle as O
    graphs, plans, reqs = _stream_requests(60)
    for kind, syms in reqs:
        g = graphs[kind]
        shapes = W.input_shapes(g, syms)
        got = plans[kind].algorithmic_bytes(shapes)
        pj = json.loads(ref.compile(json.dumps(g)))
        regs = plans[kind].eval_shapes([shapes[i["id"]] for i in g["inputs"]])
        want = 0
        for ins in pj["instrs"]:
            if ins["k"] != "launch":
                continue
            art = pj["kernels"][ins["kernel"]]
            ext = [O.resolve_dims(d, regs) for d in art["external_input_dims"]]
            for e, dims in enumerate(ext):
                whole = int(np.prod(dims))
                sliced, only = 0, True
                for m in art["tape"]:
                    for a in m["args"]:
                        if a["k"] == "e" and a["i"] == e:
                            if m["kind"] == "dynamic_slice":
                                sliced += int(np.prod(O.resolve_dims(m["out_dims"], regs)))
                            else:
                                only = False
                want += 4 * (min(sliced, whole) if only else whole)
            for t in art["outputs"]:
                want += 4 * int(np.prod(O.resolve_dims(art["tape"][t]["out_dims"], regs)))
        assert got == want, (kind, syms)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, n, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    graphs, plans, reqs = _stream_requests(n)
    costs = [plans[k].algorithmic_bytes(W.input_shapes(graphs[k], s)) for k, s in reqs]
    mine = shard(costs, world)[rank]
    # every rank's view of the full assignment must agree (no exchange on the data path,
    # the gather here only checks it)
    views = [None] * world
    dist.all_gather_object(views, {"rank": rank, "mine": mine, "all": shard(costs, world)})
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump({"views": views, "total": sum(costs), "mine_bytes": sum(costs[i] for i in mine)}, f)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_sharding(tmp_path):
    import torch.multiprocessing as mp
    world, n = 2, 400
    mp.spawn(_rank_main, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    res = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    views = res[0]["views"]
    assert res[1]["views"] == views
    for v in views:
        assert v["all"] == views[0]["all"]
        assert v["mine"] == v["all"][v["rank"]]
    parts = views[0]["all"]
    assert sorted(i for p in parts for i in p) == list(range(n))
    total = res[0]["total"]
    assert sum(r["mine_bytes"] for r in res) == total
    assert max(r["mine_bytes"] for r in res) <= 0.55 * total


@pytest.mark.gpu
def test_dispatcher_matches_executor():
    graphs, plans, reqs = _stream_requests(24)
    rng = np.random.default_rng(3)
    work = []
    for kind, syms in reqs:
        g = graphs[kind]
        inputs = {}
        for i in g["inputs"]:
            shape = tuple(syms[d] if isinstance(d, str) else d for d in i["shape"])
            inputs[i["id"]] = rng.uniform(0.25, 2.0, size=shape).astype(np.float32)
        work.append((plans[kind], inputs))
    with D.Dispatcher([0]) as disp:
        got = disp.map(work)
        assert disp.assigned == [len(work)]
    # two native workers sharing the GPU (separate streams, executors, CPU slices): LPT split
    with D.Dispatcher([0, 0]) as disp2:
        got2 = disp2.map(work)
        assert sum(disp2.assigned) == len(work) and min(disp2.assigned) > 0
        st = disp2.worker_stats()
        assert sum(w["requests"] for w in st) == len(work)
        costs = [p.algorithmic_bytes({k: v.shape for k, v in x.items()}) for p, x in work]
        assert [disp2.worker_of(r) for r in range(len(work))] == [
            next(w for w, part in enumerate(D.dispatch.shard(costs, 2)) if r in part) for r in range(len(work))]
    for a_res, b_res in zip(got, got2):
        for a, b in zip(a_res.outputs, b_res.outputs):
            np.testing.assert_array_equal(a, b)
    ex = D.Executor()
    for (plan, inputs), r in zip(work, got):
        want = ex.run(plan, inputs).outputs
        for a, b in zip(r.outputs, want):
            np.testing.assert_array_equal(a, b)


@pytest.mark.gpu
def test_run_stream_matches_single_runs():
    graphs, plans, reqs = _stream_requests(16)
    rng = np.random.default_rng(5)
    work = []
    for kind, syms in reqs:
        g = graphs[kind]
        inputs = {i["id"]: D.DeviceBuffer.from_numpy(rng.uniform(0.25, 2.0, size=tuple(
            syms[d] if isinstance(d, str) else d for d in i["shape"])).astype(np.float32)) for i in g["inputs"]}
        work.append((plans[kind], inputs))
    ex = D.Executor()
    ex.run_stream(work)
    last = ex.fetch_outputs()
    ex.synchronize()
    want = D.Executor().run(*work[-1]).outputs
    for a, b in zip(last, want):
        np.testing.assert_array_equal(a, b)
