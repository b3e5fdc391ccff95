"""Small runs of every kernel family for compute-sanitizer (tests/test_sanitizer.py):
fused loop / row (plain, fused epilogue, arg-cached, staged, odd-width, single-element) /
column (single, two-pass, atomic) / generic reduces, pad, concat, transpose (gather),
reshape copies, the library GEMM, and the same through grouped launches with PDL on --
each checked against the numpy oracle so a sanitizer run is also a parity run."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2103_05288_b200 as D  # noqa: E402
from oracle import disc_oracle as O  # noqa: E402
from paper_2103_05288_b200 import workloads as W  # noqa: E402


def graphs():
    fx = json.load(open(os.path.join(ROOT, "tests", "golden", "fixtures.json")))
    out = [(f"fx_{k}", json.loads(v["graph"]), v["bindings"][:2]) for k, v in sorted(fx.items())]
    out += [("softmax", W.softmax_graph_for(0), [{"S0": 5, "S1": 7}, {"S0": 33, "S1": 1}, {"S0": 9, "S1": 23},
                                                 {"S0": 4, "S1": 300}, {"S0": 3, "S1": 37}]),
            ("ln_gelu", W.ln_gelu_graph(), [{"T": 5, "H": 768}, {"T": 2, "H": 4096}]),
            ("colreduce", W.colreduce_graph(), [{"N": 300, "C": 9}, {"N": 4000, "C": 33}, {"N": 20000, "C": 1}]),
            ("bert", W.bert_graph(), [{"R": 96, "S": 8, "T": 8, "H": 768, "F": 3072}])]
    return out


def inputs_for(g, syms, rng):
    out = {}
    for i in g["inputs"]:
        shape = tuple(syms.get(d, 2) if isinstance(d, str) else d for d in i["shape"])
        cv = W.CONST_INPUTS.get(i["id"]) if i["id"] in W.CONST_INPUTS else None
        if i["id"] == "inv_h":
            cv = 1.0 / syms.get("H", 1)
        out[i["id"]] = (np.full(shape, cv, np.float32) if cv is not None
                        else rng.uniform(0.25, 2.0, size=shape).astype(np.float32))
    return out


def main():
    rng = np.random.default_rng(0)
    D.set_pdl(1)
    comp = D.Compiler()
    reqs = []
    worst = 0.0
    for schedule in ("auto", "twopass", "atomic"):
        ex = D.Executor()
        ex.set_schedule(schedule)
        for name, g, binds in graphs():
            plan = comp.compile(g)
            for syms in binds:
                x = inputs_for(g, syms, rng)
                got = ex.run(plan, x).outputs
                want, _, _ = O.Executor().run(plan.to_json(), x)
                worst = max([worst] + [O.rel_err(a, b) for a, b in zip(got, want)])
                if schedule == "auto":
                    reqs.append((plan, x, want))
    ex = D.Executor()
    ex.set_host_threads(2)
    res = ex.run_grouped([(p, x) for p, x, _ in reqs])
    for (p, x, want), got in zip(reqs, res):
        worst = max([worst] + [O.rel_err(a, b) for a, b in zip(got, want)])
    print(f"sanitize smoke: {len(reqs)} grouped requests, worst rel_err {worst:.3g}")
    if worst > 1e-5:
        raise SystemExit(f"parity failure under the sanitizer: {worst}")


if __name__ == "__main__":
    main()
