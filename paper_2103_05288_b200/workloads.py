"""Benchmark workloads = BASELINE.json configs, as reference-format graph JSON plus the
dynamic-shape sweeps of SURVEY.md §8(d).  All graphs use only the reference's op set
(framework.cpp:38-61), so the reference executor runs them unmodified.

  C1 softmax        fixtures/softmax.json (Softmax over [B,S]), S = 1..4096
  C2 ln_gelu        LN-like (variance division) + bias + tanh-GELU over [T,H],
                    T log-uniform 1..16384 (64 samples) x H in {768, 1024, 4096}
  C3 colreduce      ReduceSum(axes=[0]) of Mul(Tanh(Add(x, bcast(b))), x) over [N,C]
  C4 bert           BERT-base non-GEMM subgraphs: scale+mask+softmax over scores
                    [B*12*S, S], bias+residual+LN-like over [B*S, 768], bias+GELU over
                    [B*S, 3072]; S in 8..512 step 8, B in {1, 8, 32}
  C5 stream         >= 10k distinct (graph, shape) requests across C1-C4 + fixtures
"""
from __future__ import annotations

import json
import math
import random
from typing import Dict, List, Tuple

SOFTMAX = {
    "name": "softmax",
    "inputs": [{"id": "x", "shape": ["S0", 8], "dtype": "f32"}],
    "outputs": ["y"],
    "nodes": [{"id": "y", "op": "Softmax", "inputs": ["x"]}],
}


def _bcast(nid, src, shape, bdims):
    return {"id": nid, "op": "Broadcast", "inputs": [src], "attrs": {"shape": shape, "broadcast_dims": bdims}}


def _bin(nid, op, a, b):
    return {"id": nid, "op": op, "inputs": [a, b]}


def ln_gelu_graph() -> dict:
    """C2.  y = gelu_tanh((x - mean) / (var + eps) * gamma + beta + bias); the reference
    op set has no sqrt, so normalisation divides by the variance."""
    TH = ["T", "H"]
    n = [
        {"id": "s1", "op": "ReduceSum", "inputs": ["x"], "attrs": {"axes": [1]}},
        _bcast("s1b", "s1", TH, [0]), _bcast("invhb", "inv_h", TH, [1]),
        _bin("mean", "Mul", "s1b", "invhb"), _bin("c", "Sub", "x", "mean"), _bin("sq", "Mul", "c", "c"),
        {"id": "s2", "op": "ReduceSum", "inputs": ["sq"], "attrs": {"axes": [1]}},
        _bcast("s2b", "s2", TH, [0]), _bin("var", "Mul", "s2b", "invhb"), _bcast("epsb", "eps", TH, [1]),
        _bin("ve", "Add", "var", "epsb"), _bin("nrm", "Div", "c", "ve"),
        _bcast("gb", "gamma", TH, [1]), _bcast("bb", "beta", TH, [1]), _bcast("biasb", "bias", TH, [1]),
        _bin("g1", "Mul", "nrm", "gb"), _bin("g2", "Add", "g1", "bb"), _bin("h", "Add", "g2", "biasb"),
        _bin("h2", "Mul", "h", "h"), _bin("h3", "Mul", "h2", "h"), _bcast("k1b", "k1", TH, [1]),
        _bin("t1", "Mul", "h3", "k1b"), _bin("u", "Add", "h", "t1"), _bcast("k2b", "k2", TH, [1]),
        _bin("v", "Mul", "u", "k2b"), {"id": "w", "op": "Tanh", "inputs": ["v"]}, _bcast("oneb", "one", TH, [1]),
        _bin("z", "Add", "w", "oneb"), _bin("hz", "Mul", "h", "z"), _bcast("halfb", "half", TH, [1]),
        _bin("y", "Mul", "hz", "halfb"),
    ]
    inputs = [{"id": "x", "shape": TH}] + [{"id": k, "shape": ["H"]} for k in ("gamma", "beta", "bias")] + \
             [{"id": k, "shape": [1]} for k in ("inv_h", "eps", "k1", "k2", "one", "half")]
    return {"name": "ln_gelu", "inputs": inputs, "outputs": ["y"], "nodes": n}


def colreduce_graph() -> dict:
    """C3: column reduction with an elementwise prologue."""
    return {"name": "colreduce", "inputs": [{"id": "x", "shape": ["N", "C"]}, {"id": "b", "shape": ["C"]}],
            "outputs": ["r"],
            "nodes": [_bcast("bb", "b", ["N", "C"], [1]), _bin("a", "Add", "x", "bb"),
                      {"id": "t", "op": "Tanh", "inputs": ["a"]}, _bin("m", "Mul", "t", "x"),
                      {"id": "r", "op": "ReduceSum", "inputs": ["m"], "attrs": {"axes": [0]}}]}


def bert_graph() -> dict:
    """C4: the non-GEMM part of one BERT-base layer over variable-length batches.
    scores [R=B*12*S, S] -> scale, mask add, softmax; attn_out [T=B*S, 768] -> bias +
    residual + LN-like; ffn [T, 3072] -> bias + tanh-GELU."""
    RS, TH, TF = ["R", "S"], ["T", "H"], ["T", "F"]
    n = [
        # attention probabilities
        _bcast("scb", "scale", RS, [1]), _bin("ss", "Mul", "scores", "scb"), _bin("sm_in", "Add", "ss", "mask"),
        {"id": "probs", "op": "Softmax", "inputs": ["sm_in"]},
        # attention output: bias + residual + LN-like
        _bcast("ab", "attn_bias", TH, [1]), _bin("ao", "Add", "attn", "ab"), _bin("res", "Add", "ao", "resid"),
        {"id": "s1", "op": "ReduceSum", "inputs": ["res"], "attrs": {"axes": [1]}},
        _bcast("s1b", "s1", TH, [0]), _bcast("invh", "inv_h", TH, [1]), _bin("mean", "Mul", "s1b", "invh"),
        _bin("c", "Sub", "res", "mean"), _bin("sq", "Mul", "c", "c"),
        {"id": "s2", "op": "ReduceSum", "inputs": ["sq"], "attrs": {"axes": [1]}},
        _bcast("s2b", "s2", TH, [0]), _bin("var", "Mul", "s2b", "invh"), _bcast("epsb", "eps", TH, [1]),
        _bin("ve", "Add", "var", "epsb"), _bin("nrm", "Div", "c", "ve"), _bcast("gb", "gamma", TH, [1]),
        _bin("g1", "Mul", "nrm", "gb"), _bcast("bb", "beta", TH, [1]), _bin("ln", "Add", "g1", "bb"),
        # FFN intermediate: bias + tanh-GELU
        _bcast("fb", "ffn_bias", TF, [1]), _bin("h", "Add", "ffn", "fb"), _bin("h2", "Mul", "h", "h"),
        _bin("h3", "Mul", "h2", "h"), _bcast("k1b", "k1", TF, [1]), _bin("t1", "Mul", "h3", "k1b"),
        _bin("u", "Add", "h", "t1"), _bcast("k2b", "k2", TF, [1]), _bin("v", "Mul", "u", "k2b"),
        {"id": "w", "op": "Tanh", "inputs": ["v"]}, _bcast("oneb", "one", TF, [1]), _bin("z", "Add", "w", "oneb"),
        _bin("hz", "Mul", "h", "z"), _bcast("halfb", "half", TF, [1]), _bin("gelu", "Mul", "hz", "halfb"),
    ]
    inputs = [{"id": "scores", "shape": RS}, {"id": "mask", "shape": RS}, {"id": "attn", "shape": TH},
              {"id": "resid", "shape": TH}, {"id": "ffn", "shape": TF}] + \
             [{"id": k, "shape": ["H"]} for k in ("attn_bias", "gamma", "beta")] + \
             [{"id": "ffn_bias", "shape": ["F"]}] + \
             [{"id": k, "shape": [1]} for k in ("scale", "inv_h", "eps", "k1", "k2", "one", "half")]
    return {"name": "bert_nongemm", "inputs": inputs, "outputs": ["probs", "ln", "gelu"], "nodes": n}


CONST_INPUTS = {"inv_h": None, "eps": 1e-5, "k1": 0.044715, "k2": 0.7978845608, "one": 1.0, "half": 0.5,
                "scale": 0.125}


def input_shapes(graph: dict, syms: Dict[str, int]) -> Dict[str, Tuple[int, ...]]:
    shapes = {}
    for i in graph["inputs"]:
        shapes[i["id"]] = tuple(syms[d] if isinstance(d, str) else d for d in i["shape"])
    return shapes


def ln_shapes(samples: int = 64, seed: int = 20261017) -> List[Dict[str, int]]:
    rng = random.Random(seed)
    ts = sorted({max(1, min(16384, int(round(math.exp(rng.uniform(0, math.log(16384))))))) for _ in range(samples * 4)})
    rng.shuffle(ts)
    ts = sorted(ts[:samples])
    return [{"T": t, "H": h} for h in (768, 1024, 4096) for t in ts]


def softmax_shapes(big: bool = True) -> List[Dict[str, int]]:
    """C1: S = 1..4096; roofline points use B = max(1, 2^26 / S) (256 MB/request)."""
    out = []
    for s in [1, 2, 3, 7, 8, 17, 31, 64, 100, 128, 255, 256, 500, 512, 777, 1000, 1024, 1500, 2048, 3000, 4000, 4096]:
        out.append({"S0": max(1, (1 << 26) // s) if big else 64, "_S": s})
    return out


def colreduce_shapes() -> List[Dict[str, int]]:
    return [{"N": n, "C": c} for (n, c) in [(1 << 22, 4), (1 << 20, 64), (1 << 18, 1024), (1 << 16, 4096),
                                            (65537, 1000), (4096, 4096), (1 << 14, 257), (100, 4096), (7, 3)]]


def bert_shapes() -> List[Dict[str, int]]:
    out = []
    for b in (1, 8, 32):
        for s in range(8, 513, 8):
            out.append({"R": b * 12 * s, "S": s, "T": b * s, "H": 768, "F": 3072})
    return out


def softmax_graph_for(s: int) -> dict:
    g = json.loads(json.dumps(SOFTMAX))
    g["inputs"][0]["shape"] = ["S0", "S1"]
    return g


def mixed_stream(n: int = 10000, seed: int = 20261017, max_bytes: int = 1 << 22, fixtures: Dict[str, tuple] = None,
                 valid=None):
    """C5: n distinct (graph, shape) requests, kinds drawn round-robin over C1-C4 plus the
    given fixtures {name: (graph, example bindings)} (Python's MT19937, seeded); each
    request's inputs are bounded by max_bytes.  Fixture symbols that are equal in every
    example binding stay tied (e.g. split's T0 = T1 = S0).  ``valid(kind, syms)``
    (optional) rejects shapes the caller finds invalid."""
    rng = random.Random(seed)
    graphs = {"softmax": softmax_graph_for(0), "ln_gelu": ln_gelu_graph(), "colreduce": colreduce_graph(),
              "bert": bert_graph()}
    ties = {}
    for name, (g, bindings) in (fixtures or {}).items():
        graphs[f"fx_{name}"] = g
        tie = {}
        for b in bindings:
            for x in b:
                if x not in tie:
                    tie[x] = next(y for y in b if all(bb.get(y) == bb.get(x) for bb in bindings))
        ties[f"fx_{name}"] = tie
    kinds = list(graphs)
    cap = max(1, max_bytes // 4)

    def draw(kind):
        if kind == "softmax":
            s = rng.randint(1, 4096)
            return {"S0": rng.randint(1, max(1, cap // s)), "S1": s}
        if kind == "ln_gelu":
            h = rng.choice([768, 1024, 4096])
            return {"T": rng.randint(1, max(1, min(16384, cap // h))), "H": h}
        if kind == "colreduce":
            c = rng.randint(1, 4096)
            return {"N": rng.randint(1, max(1, cap // c)), "C": c}
        if kind == "bert":
            b, s = rng.choice([1, 8, 32]), rng.randrange(8, 513, 8)
            if b * 12 * s * s > cap:
                return None
            return {"R": b * 12 * s, "S": s, "T": b * s, "H": 768, "F": 3072}
        g = graphs[kind]  # fixture: every symbolic dim drawn, constant dims kept
        tie = ties.get(kind, {})
        syms = {}
        for i in g["inputs"]:
            for d in i["shape"]:
                if isinstance(d, str) and d not in syms:
                    root = tie.get(d, d)
                    if root not in syms:
                        syms[root] = rng.randint(0 if rng.random() < 0.02 else 1, 4096)
                    syms[d] = syms[root]
        return syms

    seen = set()
    reqs = []
    k = 0
    while len(reqs) < n:
        kind = kinds[k % len(kinds)]
        k += 1
        for _ in range(64):
            syms = draw(kind)
            if syms is None:
                continue
            key = (kind, tuple(sorted(syms.items())))
            if key in seen:
                continue
            if valid is not None and not valid(kind, syms):
                continue
            seen.add(key)
            reqs.append((kind, syms))
            break
    return graphs, reqs


def _logu(rng: random.Random, lo: int, hi: int) -> int:
    """Integer log-uniform in [lo, hi] (every scale of the range equally likely)."""
    if hi <= lo:
        return lo
    v = int(math.exp(rng.uniform(math.log(lo), math.log(hi + 1))))
    return max(lo, min(hi, v))


SWEEP_KINDS = ("softmax", "ln_gelu", "colreduce", "bert")


def sweep_graphs(fixtures: Dict[str, tuple] = None) -> Dict[str, dict]:
    graphs = {"softmax": softmax_graph_for(0), "ln_gelu": ln_gelu_graph(), "colreduce": colreduce_graph(),
              "bert": bert_graph()}
    for name, (g, _) in (fixtures or {}).items():
        graphs[f"fx_{name}"] = g
    return graphs


def full_sweep(step: int, n: int = 10000, seed: int = 20261017, fixtures: Dict[str, tuple] = None,
               seen: set = None, fixture_numel_cap: int = 1 << 22):
    """The headline workload (BASELINE metric; SURVEY §8d C5 over the FULL C1-C4 ranges):
    n distinct (graph, shape) requests for one step, kinds round-robin over C1-C4 plus the
    reference fixtures, every dimension drawn log-uniformly over its whole configured range
    (Python MT19937 seeded with seed + 7919 * step, so each step draws FRESH shapes):

      C1 softmax    [B, S]: S in 1..4096, B in 1..2^26/S   (up to 256 MB per tensor)
      C2 ln_gelu    [T, H]: T in 1..16384, H in {768, 1024, 4096}
      C3 colreduce  [N, C]: C in 1..4096, N in 1..min(2^22, 2^26/C)
      C4 bert       B in 1..32, S in 8..512 (variable-length batches): scores [12BS, S], [BS, 768/3072]
      fixtures      every symbolic dim log-uniform (2% zero), inputs <= fixture_numel_cap elements

    Shapes are distinct within the step (``seen``, optional, may be shared to make them
    distinct over several steps -- that biases later steps towards large shapes, since the
    small end of every range is exhausted first).  Returns (graphs, [(kind, syms)])."""
    rng = random.Random(seed + 7919 * step)
    graphs = sweep_graphs(fixtures)
    ties = {}
    for name, (g, bindings) in (fixtures or {}).items():
        tie = {}
        for b in bindings:
            for x in b:
                if x not in tie:
                    tie[x] = next(y for y in b if all(bb.get(y) == bb.get(x) for bb in bindings))
        ties[f"fx_{name}"] = tie
    kinds = list(graphs)

    def draw(kind):
        if kind == "softmax":
            s = _logu(rng, 1, 4096)
            return {"S0": _logu(rng, 1, max(1, (1 << 26) // s)), "S1": s}
        if kind == "ln_gelu":
            return {"T": _logu(rng, 1, 16384), "H": rng.choice([768, 1024, 4096])}
        if kind == "colreduce":
            c = _logu(rng, 1, 4096)
            return {"N": _logu(rng, 1, min(1 << 22, (1 << 26) // c)), "C": c}
        if kind == "bert":
            b, s = _logu(rng, 1, 32), _logu(rng, 8, 512)
            return {"R": b * 12 * s, "S": s, "T": b * s, "H": 768, "F": 3072}
        g = graphs[kind]
        tie = ties.get(kind, {})
        roots = sorted({tie.get(d, d) for i in g["inputs"] for d in i["shape"] if isinstance(d, str)})
        hi = 4096 if len(roots) > 1 else max(1, fixture_numel_cap // 8)
        syms = {r: (0 if rng.random() < 0.02 else _logu(rng, 1, hi)) for r in roots}
        for i in g["inputs"]:
            for d in i["shape"]:
                if isinstance(d, str):
                    syms[d] = syms[tie.get(d, d)]
        for i in g["inputs"]:
            m = 1
            for d in i["shape"]:
                m *= syms[d] if isinstance(d, str) else d
            if m > fixture_numel_cap:
                return None
        return syms

    seen = set() if seen is None else seen
    reqs = []
    k = 0
    while len(reqs) < n:
        kind = kinds[k % len(kinds)]
        k += 1
        for _ in range(64):
            syms = draw(kind)
            if syms is None:
                continue
            key = (kind, tuple(sorted(syms.items())))
            if key in seen:
                continue
            seen.add(key)
            reqs.append((kind, syms))
            break
    return graphs, reqs
