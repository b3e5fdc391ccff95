"""TEST INFRASTRUCTURE ONLY -- parity checker for the benchmarked sweeps.

bench.py (--verify, outside the timed region) and tests/test_gpu_sweeps.py hand this
module the host copies of a request's inputs and of the B200 outputs of the EXACT grouped
pass the bench times; it runs the reference executor (oracle/_ref, the unmodified
reference build: disc::Executor::run, src/executor.cpp:221-465) on the same inputs and
compares.  Nothing here touches the device or imports the B200 package.

Which requests are checked:
  * every request whose inputs all have <= 2^22 elements: the whole request;
  * larger ones (all of them with mode "full", a seeded fraction otherwise): a seeded
    sample of rows (row-independent patterns C1 softmax, C2 LN+GELU, C4 BERT parts) or
    columns (C3 column reduce) -- the reference computes exactly those rows / columns
    from exactly those inputs.

Metrics per output element (a = B200, b = reference):
  * rel_err_floored = |a-b| / max(1, |a|, |b|)   -- the reference's own test metric
    (tests/testutil.hpp:64-70), north-star bound 1e-5;
  * rel_err_true    = |a-b| / |b| over |b| > 0    -- true relative error (reported);
  * ulp             = |a-b| / ulp_f32(b)          -- units in the last place (reported).
"""
from __future__ import annotations

import json
import threading
from concurrent.futures import ThreadPoolExecutor
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import ref

SMALL_NUMEL = 1 << 22
TOL = 1e-5

# Row structure of the benchmark patterns: {input: row axis group} and {output: group}.
# A group's rows are sampled together (same row indices in every member).
ROW_SPEC = {
    "softmax": ({"x": "r"}, ["r"]),
    "ln_gelu": ({"x": "r"}, ["r"]),
    "bert": ({"scores": "R", "mask": "R", "attn": "T", "resid": "T", "ffn": "T"}, ["R", "T", "T"]),
}
COL_SPEC = {"colreduce": ({"x": 1, "b": 0}, [0])}  # input -> axis of the column index; outputs' axis


def errors(a: np.ndarray, b: np.ndarray) -> Dict[str, float]:
    a = np.asarray(a, dtype=np.float32).ravel()
    b = np.asarray(b, dtype=np.float32).ravel()
    if a.shape != b.shape:
        return {"floored": 1.0, "true": float("inf"), "ulp": float("inf"), "n": int(b.size), "shape_mismatch": True}
    if a.size == 0:
        return {"floored": 0.0, "true": 0.0, "ulp": 0.0, "n": 0, "over_1e-5_true": 0}
    ad, bd = a.astype(np.float64), b.astype(np.float64)
    both_nan = np.isnan(ad) & np.isnan(bd)
    inf = np.isinf(ad) | np.isinf(bd)
    same_inf = inf & (ad == bd)
    diff = np.abs(ad - bd)
    diff[both_nan | same_inf] = 0.0
    bad_inf = inf & ~same_inf
    floored = diff / np.maximum(1.0, np.maximum(np.abs(ad), np.abs(bd)))
    floored[bad_inf] = 1.0
    nz = (bd != 0) & np.isfinite(bd) & ~both_nan
    true = np.zeros_like(diff)
    true[nz] = diff[nz] / np.abs(bd[nz])
    true[(bd == 0) & (diff != 0)] = np.inf
    ulp = diff / np.spacing(np.abs(b).astype(np.float32)).astype(np.float64)
    ulp[both_nan | same_inf] = 0.0
    ulp[bad_inf] = np.inf
    return {"floored": float(floored.max()), "true": float(true.max()), "ulp": float(ulp.max()), "n": int(b.size),
            "over_1e-5_true": int((true > TOL).sum())}


def _merge(acc: Dict, e: Dict) -> None:
    for k in ("floored", "true", "ulp"):
        acc[k] = max(acc.get(k, 0.0), e[k])
    acc["elements"] = acc.get("elements", 0) + e["n"]
    acc["over_1e-5_true"] = acc.get("over_1e-5_true", 0) + e.get("over_1e-5_true", 0)


class Plan:
    """How one request is checked: 'full', or sampled 'rows' / 'cols' of a pattern."""

    def __init__(self, mode: str, pick: Optional[Dict[str, np.ndarray]] = None):
        self.mode = mode
        self.pick = pick or {}


def check_plan(kind: str, shapes: Dict[str, Tuple[int, ...]], large_checked: bool, rng: np.random.Generator,
               rows: int = 64) -> Optional[Plan]:
    """None: not checked.  Small requests are checked whole; large ones by rows/columns."""
    if max((int(np.prod(s)) for s in shapes.values()), default=0) <= SMALL_NUMEL:
        return Plan("full")
    if not large_checked:
        return None
    if kind in ROW_SPEC:
        ins, _ = ROW_SPEC[kind]
        groups = {}
        for name, g in ins.items():
            groups[g] = shapes[name][0]
        return Plan("rows", {g: np.sort(rng.choice(n, min(rows, n), replace=False)) for g, n in groups.items()})
    if kind in COL_SPEC:
        ncol = shapes["x"][1]
        return Plan("cols", {"c": np.sort(rng.choice(ncol, min(16, ncol), replace=False))})
    return Plan("full")  # fixtures are capped small; anything else is checked whole


class Checker:
    """Runs reference checks on a thread pool (ctypes releases the GIL inside the
    reference executor; one reference executor per thread).  submit() takes host copies
    of inputs and B200 outputs already reduced to the checked rows/columns."""

    def __init__(self, graphs: Dict[str, dict], threads: int = 8, max_pending: int = 256):
        self.graphs = graphs
        self.plan_json = {k: ref.compile(json.dumps(g)) for k, g in graphs.items()}
        self.pool = ThreadPoolExecutor(max(1, threads))
        self.local = threading.local()
        self.sem = threading.Semaphore(max_pending)
        self.lock = threading.Lock()
        self.futures = []
        self.per_kind: Dict[str, Dict] = {}
        self.failures: List[str] = []
        self.requests = {"full": 0, "rows": 0, "cols": 0}

    def _plans(self):
        if not hasattr(self.local, "plans"):
            self.local.plans = {}
        return self.local.plans

    def _run(self, kind: str, inputs: Dict[str, np.ndarray]) -> List[np.ndarray]:
        plans = self._plans()
        if kind not in plans:
            plans[kind] = ref.RefPlan(self.plan_json[kind])
        return plans[kind].run(inputs).outputs

    def _job(self, tag: str, kind: str, mode: str, inputs, got: Sequence[np.ndarray]) -> None:
        try:
            want = self._run(kind, inputs)
            acc = {}
            for o, (a, b) in enumerate(zip(got, want)):
                e = errors(a, b)
                _merge(acc, e)
                if e["floored"] > TOL or e.get("shape_mismatch"):
                    with self.lock:
                        self.failures.append(f"{tag} output {o}: floored rel_err {e['floored']:.3g}")
            if len(got) != len(want):
                with self.lock:
                    self.failures.append(f"{tag}: {len(got)} outputs, reference {len(want)}")
            with self.lock:
                _merge(self.per_kind.setdefault(kind, {}), {"floored": acc.get("floored", 0.0),
                                                            "true": acc.get("true", 0.0),
                                                            "ulp": acc.get("ulp", 0.0), "n": acc.get("elements", 0),
                                                            "over_1e-5_true": acc.get("over_1e-5_true", 0)})
                self.per_kind[kind]["requests"] = self.per_kind[kind].get("requests", 0) + 1
                self.requests[mode] += 1
        except Exception as ex:  # a reference error on the same inputs is a parity failure too
            with self.lock:
                self.failures.append(f"{tag}: {type(ex).__name__}: {ex}")
        finally:
            self.sem.release()

    def submit(self, tag: str, kind: str, mode: str, inputs: Dict[str, np.ndarray], got: Sequence[np.ndarray]) -> None:
        self.sem.acquire()
        self.futures.append(self.pool.submit(self._job, tag, kind, mode, inputs, list(got)))

    def finish(self) -> Dict:
        for f in self.futures:
            f.result()
        self.pool.shutdown()
        allk = {}
        for v in self.per_kind.values():
            _merge(allk, {"floored": v["floored"], "true": v["true"], "ulp": v["ulp"], "n": v["elements"],
                          "over_1e-5_true": v["over_1e-5_true"]})
        r = lambda x: float(f"{x:.4g}") if np.isfinite(x) else str(x)
        return {
            "requests_checked": dict(self.requests),
            "tol_floored": TOL,
            "max_rel_err_floored": r(allk.get("floored", 0.0)),
            "max_rel_err_true": r(allk.get("true", 0.0)),
            "max_ulp": r(allk.get("ulp", 0.0)),
            "elements_over_1e-5_true": allk.get("over_1e-5_true", 0),
            "elements": allk.get("elements", 0),
            "per_pattern": {k: {"requests": v["requests"], "floored": r(v["floored"]), "true": r(v["true"]),
                                "ulp": r(v["ulp"]), "over_1e-5_true": v["over_1e-5_true"]}
                            for k, v in sorted(self.per_kind.items())},
            "failures": self.failures[:20],
            "pass": not self.failures,
        }


def expected_output_rows(kind: str, plan: Plan, n_outputs: int) -> List[Optional[np.ndarray]]:
    """Row (or column) indices of each output the B200 side must gather for `plan`."""
    if plan.mode == "full":
        return [None] * n_outputs
    if plan.mode == "rows":
        _, outs = ROW_SPEC[kind]
        return [plan.pick[g] for g in outs]
    return [plan.pick["c"]] * n_outputs
