"""TEST / BASELINE INFRASTRUCTURE ONLY -- the SURVEY §8(d) algorithmic byte count of one
request, computed from the REFERENCE's own plan JSON (oracle/_ref compile), so bench.py's
reference arm never loads the B200 package.

  bytes = 4 x sum over kLaunch of [ sum_external-inputs numel_read + sum_outputs numel ]

numel_read is the input's numel, or -- when the kernel reads that input only through
dynamic_slice members -- the sum of the slice outputs (capped at the input numel);
broadcast sources count at their source size (they are external inputs of the tape at
their own dims).  tests/test_dispatch.py pins this against CompiledPlan.algorithmic_bytes.

The register file comes from the plan's host shape program, restated from the reference
executor's kEvalShape (src/executor.cpp:303-341; ShapeInstr kinds shape_analysis.hpp:56-125).
"""
from __future__ import annotations

import json
from typing import Dict, List, Sequence


def _ref(r: dict, regs: Sequence[int]) -> int:  # resolve_ref, src/executor.cpp:46-51
    return int(r["c"]) if "c" in r else int(regs[r["r"]])


def eval_shape_program(plan: dict, input_dims: Dict[str, Sequence[int]]) -> List[int]:
    """Register file after EvalShape for the given input dims (by input id)."""
    sp = plan["shape_program"]
    regs = [0] * sp["num_regs"]
    ids = [i["id"] for i in plan["inputs"]]
    for si in sp["instrs"]:
        k = si["k"]
        if k == "read_input_dim":
            regs[si["dest"]] = int(input_dims[ids[si["input"]]][si["axis"]])
        elif k == "read_scalar":
            regs[si["dest"]] = plan["literals"][si["tensor"]][si["index"]]
        elif k == "load_const":
            regs[si["dest"]] = si["value"]
        elif k == "bin_op":
            a, b, op = regs[si["lhs"]], regs[si["rhs"]], si["op"]
            if op == "add":
                v = a + b
            elif op == "sub":
                v = a - b
            elif op == "mul":
                v = a * b
            elif op == "div":
                v = int(a / b)  # C++ truncation toward zero
            elif op == "ceil_div":
                v = int((a + b - 1) / b)
            else:
                v = max(a, b)
            regs[si["dest"]] = v
    return regs


def _numel(dims) -> int:
    n = 1
    for d in dims:
        n *= int(d)
    return n


class PlanBytes:
    """Byte model of one reference plan (JSON text or dict)."""

    def __init__(self, plan):
        self.plan = json.loads(plan) if isinstance(plan, str) else plan
        self.launches = [self.plan["kernels"][i["kernel"]] for i in self.plan["instrs"] if i["k"] == "launch"]

    def __call__(self, input_dims: Dict[str, Sequence[int]]) -> int:
        regs = eval_shape_program(self.plan, input_dims)
        total = 0
        for art in self.launches:
            for e, d in enumerate(art["external_input_dims"]):
                whole = _numel(_ref(x, regs) for x in d)
                sliced, only = 0, True
                for m in art["tape"]:
                    for a in m["args"]:
                        if a["k"] == "e" and a["i"] == e:
                            if m["kind"] == "dynamic_slice":
                                sliced += _numel(_ref(x, regs) for x in m["out_dims"])
                            else:
                                only = False
                total += 4 * (min(sliced, whole) if only else whole)
            for t in art["outputs"]:
                total += 4 * _numel(_ref(x, regs) for x in art["tape"][t]["out_dims"])
        return total
