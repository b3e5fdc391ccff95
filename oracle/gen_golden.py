"""TEST INFRASTRUCTURE ONLY -- regenerates tests/golden/ from the reference.

Run here (where /root/reference and oracle/_ref exist):  python oracle/gen_golden.py
Outputs (all small, committed):
  tests/golden/reference_goldens.json  the reference's own byte-exact goldens
        (proj/tests/golden/softmax_{ir.txt,dhlo.json,plan.json}) keyed by file name
  tests/golden/fixtures.json           proj/fixtures/*.json graphs + *.bindings.json
  tests/golden/fixture_plans.json      reference plan JSON per fixture x option set
  tests/golden/random_plans.json.gz     reference plan JSON for RandomGraphGen seeds 0..199
  tests/golden/fixture_io.npz          make_binding inputs + reference Executor outputs/stats
"""
from __future__ import annotations

import glob
import gzip
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

REF = "/root/reference/proj"
OUT = os.path.join(ROOT, "tests", "golden")

OPTION_SETS = {
    "default": dict(inject=True, fusion=True, static_fallback=False),
    "no_inject": dict(inject=False, fusion=True, static_fallback=False),
    "no_fusion": dict(inject=True, fusion=False, static_fallback=False),
    "static_fb": dict(inject=True, fusion=True, static_fallback=True),
}


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    goldens = {}
    for p in sorted(glob.glob(os.path.join(REF, "tests", "golden", "*"))):
        goldens[os.path.basename(p)] = open(p).read()
    json.dump(goldens, open(os.path.join(OUT, "reference_goldens.json"), "w"), indent=1, sort_keys=True)

    fixtures = {}
    for p in sorted(glob.glob(os.path.join(REF, "fixtures", "*.json"))):
        if p.endswith(".bindings.json"):
            continue
        name = os.path.basename(p)[:-5]
        fixtures[name] = {
            "graph": open(p).read(),
            "bindings": json.load(open(p[:-5] + ".bindings.json")),
        }
    json.dump(fixtures, open(os.path.join(OUT, "fixtures.json"), "w"), indent=1, sort_keys=True)

    plans = {}
    for name, fx in fixtures.items():
        for oname, o in OPTION_SETS.items():
            plans[f"{name}/{oname}"] = ref.compile(fx["graph"], **o)
    json.dump(plans, open(os.path.join(OUT, "fixture_plans.json"), "w"), indent=1, sort_keys=True)

    rnd = {}
    for seed in range(200):
        g = ref.random_graph(seed, 12)
        rnd[str(seed)] = {"graph": g, "plan": ref.compile(g)}
    with gzip.open(os.path.join(OUT, "random_plans.json.gz"), "wt") as f:
        json.dump(rnd, f, sort_keys=True)

    arrays = {}
    meta = {}
    for name, fx in fixtures.items():
        rp = ref.RefPlan(plans[f"{name}/default"])
        for bi, syms in enumerate(fx["bindings"]):
            inputs = ref.make_binding(fx["graph"], syms, 7)
            res = rp.run(inputs)
            key = f"{name}/{bi}"
            for k, v in inputs.items():
                arrays[f"{key}/in/{k}"] = v
            for oi, v in enumerate(res.outputs):
                arrays[f"{key}/out/{oi}"] = v
            meta[key] = {"syms": syms, "stats": res.stats, "inputs": list(inputs.keys()),
                         "n_out": len(res.outputs)}
    arrays["__meta__"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "fixture_io.npz"), **arrays)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
