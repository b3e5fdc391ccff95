"""Static plan as a CUDA graph vs per-launch issue: device inputs, same buffers each run,
wall time per run (host flow + launches) over 2000 runs of the transformer fixture."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05288_b200 as D  # noqa: E402

fx = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "fixtures.json")))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
from test_compiler_parity import _static_variant  # noqa: E402

for name in ("transformer", "softmax"):
    g = _static_variant(fx, name)
    graph = json.loads(g)
    plan = D.static_specialize(g)
    syms = {}
    rng = np.random.default_rng(0)
    bufs = {i["id"]: D.DeviceBuffer.from_numpy(rng.uniform(0.25, 2, size=[syms.get(d, 2) if isinstance(d, str) else d
                                                                          for d in i["shape"]]).astype(np.float32))
            for i in graph["inputs"]}
    for on in (False, True):
        ex = D.Executor(0, D.new_stream())
        ex.set_graphs(on)
        for _ in range(5):
            ex.run_device(plan, bufs)
        ex.synchronize()
        t = time.perf_counter()
        for _ in range(2000):
            ex.run_device(plan, bufs)
        ex.synchronize()
        dt = (time.perf_counter() - t) / 2000
        print(f"{name}: graphs={on} {dt * 1e6:.1f} us/run, replays {ex.graph_replays()}, "
              f"{plan.num_kernels} kernels")
