"""The multi-process path on a GPU: a world_size-2 gloo job whose ranks
share the box's GPU (bench.py's BENCH_DEVICES_OVERRIDE mode) -- each rank derives the same
LPT shard cover locally (no data-path exchange), runs ITS requests as one grouped call on
the device and writes its outputs; the union equals a single-rank run of every request,
bit for bit.  Also the bench itself under torchrun with 2 ranks."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _requests(n=48):
    from paper_2103_05288_b200 import workloads as W
    graphs, reqs = W.mixed_stream(n, seed=99)
    return graphs, reqs


def _inputs(graphs, reqs):
    rng = np.random.default_rng(11)
    out = []
    for kind, syms in reqs:
        g = graphs[kind]
        out.append({i["id"]: rng.uniform(0.25, 2.0, size=tuple(syms[d] if isinstance(d, str) else d
                                                                  for d in i["shape"])).astype(np.float32)
                    for i in g["inputs"]})
    return out


def _rank_main(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_2103_05288_b200 as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    graphs, reqs = _requests()
    inputs = _inputs(graphs, reqs)
    plans = {k: D.compile_graph(g) for k, g in graphs.items()}
    costs = [plans[k].algorithmic_bytes({n: a.shape for n, a in x.items()}) for (k, _), x in zip(reqs, inputs)]
    mine = D.shard(costs, world)[rank]
    ex = D.Executor(0)  # both ranks on the visible GPU
    outs = ex.run_grouped([(plans[reqs[i][0]], inputs[i]) for i in mine])
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
             **{f"{i}_{o}": a for i, res in zip(mine, outs) for o, a in enumerate(res)})
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump({"mine": mine}, f)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_share_the_gpu_and_match_one_rank(gpu, tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_rank_main, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    graphs, reqs = _requests()
    inputs = _inputs(graphs, reqs)
    plans = {k: gpu.compile_graph(g) for k, g in graphs.items()}
    want = gpu.Executor().run_grouped([(plans[k], x) for (k, _), x in zip(reqs, inputs)])
    seen = []
    for r in range(2):
        mine = json.load(open(tmp_path / f"rank{r}.json"))["mine"]
        z = np.load(tmp_path / f"rank{r}.npz")
        seen += mine
        for i in mine:
            for o, a in enumerate(want[i]):
                np.testing.assert_array_equal(z[f"{i}_{o}"], a)
    assert sorted(seen) == list(range(len(reqs)))


def test_bench_two_ranks_shared_gpu(gpu):
    """bench.py under torchrun, 2 ranks sharing the GPU over gloo: barriers, max-over-ranks
    time, summed bytes -- the multi-GPU code path end to end (not a scaling number)."""
    port = _free_port()
    env = dict(os.environ, BENCH_DEVICES_OVERRIDE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--requests", "400", "--no-analysis", "--verify", "off", "--no-e2e", "--no-cpu-baseline",
           "--arena-gb", "8", "--reserve-gb", "8", "--cache-gb", "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    j = json.loads(line)
    assert j["n_gpus"] == 2 and j["value"] > 0 and j["recompiles"] == 0
    assert j["config"]["requests_per_step"] == 400
