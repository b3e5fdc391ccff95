"""TEST INFRASTRUCTURE ONLY -- a numpy restatement of the reference's runtime path.

This is the CPU *checker* for the B200 backend: it interprets a plan JSON exactly the way
the reference executor does, and is itself pinned against the reference build
(oracle/_ref/libdisc_ref.so) and the committed goldens by tests/test_oracle.py.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import it.

Restated (file:line relative to /root/reference/proj):
  resolve_ref                      src/executor.cpp:46-51
  guard_passes                     src/executor.cpp:78-98
  elementwise_loop (flat index)    src/executor.cpp:102-133
  run_kernel (tape, own out_dims)  src/executor.cpp:137-219
  Executor::run (instruction loop) src/executor.cpp:221-465
  CachedAllocator (exact-size)     src/executor.cpp:53-76
  apply_binary / apply_unary       src/kernels.cpp:26-44   (f32, std::max = (a<b)?b:a)
  reduce_identity / reduce_step    src/kernels.cpp:46-54   (f64 accumulate)
  eval_slice_gather / eval_pad / eval_broadcast / eval_reshape / eval_transpose /
  eval_concat / eval_reduce        src/kernels.cpp:103-259
  eval_matmul (f64 accumulate)     src/kernels.cpp:261-303

Numerics: f32 elementwise via numpy float32 (no FMA contraction); exp/tanh use numpy's
float32 ufuncs (may differ from glibc by an ulp -- parity for those ops is the 1e-5
rel_err of tests/testutil.hpp:64-70).  Reductions accumulate in float64 in flat order.
"""
from __future__ import annotations

import json
from typing import Dict, List, Sequence

import numpy as np


class OracleError(RuntimeError):
    pass


def resolve_ref(r: dict, regs: Sequence[int]) -> int:
    if "c" in r:
        return int(r["c"])
    return int(regs[r["r"]])


def resolve_dims(refs, regs) -> List[int]:
    return [resolve_ref(r, regs) for r in refs]


def guard_passes(art: dict, version: dict, regs) -> bool:
    for t in version["guards"]:
        k = t["k"]
        if k == "total_div4":
            total = 1
            for d in art["space"]:
                total *= resolve_ref(d, regs)
            if total % 4 != 0:
                return False
        elif k == "eq":
            if resolve_ref(t["a"], regs) != resolve_ref(t["b"], regs):
                return False
        elif k == "never":
            return False
    return True


def apply_binary(kind: str, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = a.astype(np.float32, copy=False)
    b = b.astype(np.float32, copy=False)
    with np.errstate(all="ignore"):
        if kind == "add":
            return a + b
        if kind == "sub":
            return a - b
        if kind == "mul":
            return a * b
        if kind == "div":
            return a / b
        if kind == "maximum":
            return np.where(a < b, b, a)  # std::max(a, b) returns a unless a < b
    raise OracleError("not a binary op")


def apply_unary(kind: str, a: np.ndarray) -> np.ndarray:
    with np.errstate(all="ignore"):
        if kind == "exp":
            return np.exp(a.astype(np.float32))
        if kind == "tanh":
            return np.tanh(a.astype(np.float32))
        if kind == "neg":
            return -a.astype(np.float32)
    raise OracleError("not a unary op")


def eval_reduce(kind: str, x: np.ndarray, axes: Sequence[int]) -> np.ndarray:
    axes = tuple(int(a) for a in axes)
    x64 = x.astype(np.float64)
    out_shape = tuple(d for i, d in enumerate(x.shape) if i not in axes)
    if x.size == 0:
        ident = 0.0 if kind == "reduce_sum" else -np.inf
        return np.full(out_shape, ident, dtype=np.float64).astype(np.float32)
    if kind == "reduce_sum":
        r = x64.sum(axis=axes)
    else:
        # NaN never wins std::max(acc, v) with acc starting at -inf (kernels.cpp:52-54).
        r = np.where(np.isnan(x64), -np.inf, x64).max(axis=axes)
    return np.asarray(r, dtype=np.float64).reshape(out_shape).astype(np.float32)


def eval_broadcast(x: np.ndarray, out_dims: Sequence[int], bdims: Sequence[int]) -> np.ndarray:
    for i, bd in enumerate(bdims):
        if x.shape[i] != 1 and x.shape[i] != out_dims[bd]:
            raise OracleError("broadcast dim incompatible at runtime")
    shape = [1] * len(out_dims)
    for i, bd in enumerate(bdims):
        shape[bd] = x.shape[i]
    return np.broadcast_to(x.reshape(shape), tuple(out_dims)).astype(np.float32)


def eval_slice_gather(x: np.ndarray, starts, strides, out_dims) -> np.ndarray:
    r = x.ndim
    for i in range(r):
        if strides[i] <= 0:
            raise OracleError("slice stride <= 0")
        if starts[i] < 0:
            raise OracleError("slice index out of range")
        if out_dims[i] > 0 and starts[i] + (out_dims[i] - 1) * strides[i] >= x.shape[i]:
            raise OracleError("slice index out of range")
    idx = tuple(slice(starts[i], starts[i] + out_dims[i] * strides[i], strides[i]) for i in range(r))
    return np.array(x[idx], dtype=np.float32).reshape(out_dims)


def eval_pad(x: np.ndarray, value: float, low, high, interior) -> np.ndarray:
    r = x.ndim
    out_dims = []
    for i in range(r):
        if low[i] < 0 or high[i] < 0 or interior[i] < 0:
            raise OracleError("negative padding")
        n = x.shape[i]
        out_dims.append(low[i] + high[i] + n + ((n - 1) * interior[i] if n > 0 else 0))
    out = np.full(out_dims, np.float32(value), dtype=np.float32)
    idx = tuple(slice(low[i], low[i] + (x.shape[i] - 1) * (1 + interior[i]) + 1 if x.shape[i] else low[i],
                      1 + interior[i]) for i in range(r))
    if x.size:
        out[idx] = x
    return out


def eval_transpose(x: np.ndarray, perm) -> np.ndarray:
    return np.array(np.transpose(x, [int(p) for p in perm]), dtype=np.float32)


def eval_concat(parts: List[np.ndarray], axis: int) -> np.ndarray:
    r = parts[0].ndim
    for p in parts:
        for i in range(r):
            if i != axis and p.shape[i] != parts[0].shape[i]:
                raise OracleError("concat non-axis dim mismatch at runtime")
    return np.concatenate(parts, axis=axis).astype(np.float32)


def eval_matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    if a.ndim != 2 or b.ndim != 2:
        raise OracleError("matmul operands must be rank-2")
    if a.shape[1] != b.shape[0]:
        raise OracleError("matmul inner dim mismatch at runtime")
    return (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)


def _numel(d) -> int:
    n = 1
    for x in d:
        n *= int(x)
    return n


def run_kernel(art: dict, version: dict, externals: List[np.ndarray], regs) -> List[np.ndarray]:
    """executor.cpp:137-219: every member materialised at its own out_dims; members
    combine by flat index."""
    scratch: List[np.ndarray] = [None] * len(art["tape"])  # type: ignore

    def arg(ref):
        return externals[ref["i"]] if ref["k"] == "e" else scratch[ref["i"]]

    vec4 = version["vectorized4"]
    for t, ins in enumerate(art["tape"]):
        kind = ins["kind"]
        out_dims = resolve_dims(ins["out_dims"], regs)
        n = _numel(out_dims)
        if kind in ("add", "sub", "mul", "div", "maximum"):
            a, b = arg(ins["args"][0]), arg(ins["args"][1])
            if a.size != n or b.size != n:
                raise OracleError("fused elementwise operand size mismatch")
            if vec4 and n % 4:
                raise OracleError("vectorized kernel launched with ragged extent")
            scratch[t] = apply_binary(kind, a.reshape(-1), b.reshape(-1)).reshape(out_dims)
        elif kind in ("exp", "tanh", "neg"):
            a = arg(ins["args"][0])
            if a.size != n:
                raise OracleError("fused elementwise operand size mismatch")
            if vec4 and n % 4:
                raise OracleError("vectorized kernel launched with ragged extent")
            scratch[t] = apply_unary(kind, a.reshape(-1)).reshape(out_dims)
        elif kind in ("reduce_sum", "reduce_max"):
            scratch[t] = eval_reduce(kind, arg(ins["args"][0]), ins.get("dims", []))
        elif kind == "dynamic_broadcast_in_dim":
            x = arg(ins["args"][0])
            if version["implicit_broadcast"]:
                scratch[t] = eval_broadcast(x, out_dims, ins.get("dims", []))
            else:
                if x.size != n:
                    raise OracleError("no-broadcast version launched with non-identity shape")
                scratch[t] = x.reshape(out_dims)
        elif kind == "dynamic_slice":
            scratch[t] = eval_slice_gather(arg(ins["args"][0]), resolve_dims(ins["starts"], regs),
                                           resolve_dims(ins["strides"], regs), out_dims)
        elif kind == "transpose":
            scratch[t] = eval_transpose(arg(ins["args"][0]), ins.get("dims", []))
        elif kind == "dynamic_reshape":
            x = arg(ins["args"][0])
            if n != x.size:
                raise OracleError("reshape element count mismatch at runtime")
            scratch[t] = x.reshape(out_dims)
        elif kind == "dynamic_pad":
            scratch[t] = eval_pad(arg(ins["args"][0]), ins["value"], resolve_dims(ins["low"], regs),
                                  resolve_dims(ins["high"], regs), resolve_dims(ins["interior"], regs))
        elif kind == "concat":
            scratch[t] = eval_concat([arg(a) for a in ins["args"]], ins.get("axis", 0))
        else:
            raise OracleError("unexpected op in kernel tape")
    return [scratch[i] for i in art["outputs"]]


class Executor:
    """executor.cpp:221-465 with the exact-size CachedAllocator (53-76) and ExecStats."""

    def __init__(self):
        self.free_list: Dict[int, List[int]] = {}
        self.block_bytes: List[int] = []
        self.block_data: List[np.ndarray] = []

    def _alloc(self, nbytes: int, stats: dict) -> int:
        fl = self.free_list.get(nbytes)
        if fl:
            stats["allocator_cache_hits"] += 1
            return fl.pop()
        stats["alloc_calls"] += 1
        floats = max((nbytes + 3) // 4, 1)
        floats = (floats + 3) // 4 * 4
        self.block_bytes.append(nbytes)
        self.block_data.append(np.zeros(floats, np.float32))
        return len(self.block_bytes) - 1

    def _free(self, block: int) -> None:
        self.free_list.setdefault(self.block_bytes[block], []).append(block)

    def run(self, plan, inputs: Dict[str, np.ndarray]):
        if isinstance(plan, str):
            plan = json.loads(plan)
        stats = dict(launch_count=0, library_calls=0, host_instruction_count=len(plan["instrs"]),
                     peak_bytes=0, alloc_calls=0, allocator_cache_hits=0, aliased_allocs=0)
        sp = plan["shape_program"]
        regs = [0] * sp["num_regs"]
        nbuf = plan["num_buffers"]
        slot_input: List = [None] * nbuf
        slot_block = [-1] * nbuf
        slot_bytes = [0] * nbuf
        versions: Dict[int, int] = {}
        live = 0
        events: Dict[int, list] = {}
        outputs: List = [None] * len(plan["outputs"])

        def input_asserts():
            for i, pi in enumerate(plan["inputs"]):
                t = slot_input[i]
                for d, ref in enumerate(pi["dims"]):
                    want = resolve_ref(ref, regs)
                    if t.shape[d] != want:
                        raise OracleError(f"input {pi['id']} dim {d} violates a shape constraint: "
                                          f"expected {want}, got {t.shape[d]}")

        def tensor_from_slot(buf, dims):
            if slot_input[buf] is not None:
                return slot_input[buf].reshape(dims) if list(slot_input[buf].shape) != list(dims) \
                    else slot_input[buf]
            n = _numel(dims)
            return self.block_data[slot_block[buf]][:n].copy().reshape(dims)

        def write_to_slot(buf, t):
            if slot_input[buf] is not None:
                raise OracleError("write into an input buffer")
            if t.size * 4 > slot_bytes[buf]:
                raise OracleError("kernel output exceeds planned buffer size")
            if t.size:
                self.block_data[slot_block[buf]][: t.size] = t.reshape(-1)

        for pc, ins in enumerate(plan["instrs"]):
            k = ins["k"]
            if k == "bind_input":
                pi = plan["inputs"][ins["io"]]
                if pi["id"] not in inputs:
                    raise OracleError("missing input " + pi["id"])
                x = np.asarray(inputs[pi["id"]], dtype=np.float32)
                if x.ndim != len(pi["dims"]):
                    raise OracleError(f"input {pi['id']} rank mismatch")
                slot_input[ins["buffer"]] = x
            elif k == "eval_shape":
                for si in sp["instrs"][ins["from"]:ins["to"]]:
                    sk = si["k"]
                    if sk == "read_input_dim":
                        regs[si["dest"]] = slot_input[si["input"]].shape[si["axis"]]
                    elif sk == "read_scalar":
                        regs[si["dest"]] = plan["literals"][si["tensor"]][si["index"]]
                    elif sk == "load_const":
                        regs[si["dest"]] = si["value"]
                    elif sk == "bin_op":
                        a, b = regs[si["lhs"]], regs[si["rhs"]]
                        op = si["op"]
                        if op == "add":
                            v = a + b
                        elif op == "sub":
                            v = a - b
                        elif op == "mul":
                            v = a * b
                        elif op == "div":
                            if b == 0:
                                raise OracleError("shape computation divided by zero")
                            v = int(a / b)  # C++ truncation toward zero
                        elif op == "ceil_div":
                            if b <= 0:
                                raise OracleError("shape ceil_div by non-positive stride")
                            v = int((a + b - 1) / b)
                        else:
                            v = max(a, b)
                        regs[si["dest"]] = v
                input_asserts()
            elif k == "alloc":
                elems = ins["size"]["const_elems"]
                for r in ins["size"]["regs"]:
                    elems *= regs[r]
                b = ins["buffer"]
                slot_block[b] = self._alloc(elems * 4, stats)
                slot_bytes[b] = elems * 4
                live += elems * 4
                stats["peak_bytes"] = max(stats["peak_bytes"], live)
                events[b] = [b, slot_block[b], pc, -1]
            elif k == "dealloc":
                b = ins["buffer"]
                if not ins.get("reserve", False):
                    self._free(slot_block[b])
                    live -= slot_bytes[b]
                events[b][3] = pc
            elif k == "alias":
                b, s = ins["buffer"], ins["source"]
                slot_block[b] = slot_block[s]
                slot_bytes[b] = slot_bytes[s]
                stats["aliased_allocs"] += 1
                events[b] = [b, slot_block[b], pc, -1]
            elif k == "select_version":
                art = plan["kernels"][ins["kernel"]]
                chosen = next((v["id"] for v in art["versions"] if guard_passes(art, v, regs)), -1)
                if chosen < 0:
                    raise OracleError("no kernel version guard matched")
                versions[ins["kernel"]] = chosen
            elif k == "compute_launch":
                pass  # launch config only (tile 256/1024); no effect on values
            elif k == "launch":
                art = plan["kernels"][ins["kernel"]]
                vid = ins.get("version", -1)
                if vid < 0:
                    vid = versions[ins["kernel"]]
                version = next(v for v in art["versions"] if v["id"] == vid)
                ext = [tensor_from_slot(b, resolve_dims(art["external_input_dims"][a], regs))
                       for a, b in enumerate(ins["inputs"])]
                outs = run_kernel(art, version, ext, regs)
                stats["launch_count"] += 1
                for o, b in enumerate(ins["outputs"]):
                    write_to_slot(b, outs[o])
            elif k == "library_call":
                m, kk, n = resolve_dims(ins["dims"], regs)
                a = tensor_from_slot(ins["inputs"][0], [m, kk])
                b = tensor_from_slot(ins["inputs"][1], [kk, n])
                stats["library_calls"] += 1
                write_to_slot(ins["outputs"][0], eval_matmul(a, b))
            elif k == "bind_output":
                po = plan["outputs"][ins["io"]]
                outputs[ins["io"]] = tensor_from_slot(ins["buffer"], resolve_dims(po["dims"], regs)).copy()
        if not sp["instrs"]:
            input_asserts()
        returned = set()
        for b, ev in events.items():
            if ev[3] >= 0:
                continue
            if ev[1] not in returned:
                returned.add(ev[1])
                self._free(ev[1])
        return outputs, stats, [tuple(events[b]) for b in sorted(events)]


def rel_err(a: np.ndarray, b: np.ndarray) -> float:
    """tests/testutil.hpp:64-82 (max over elements; inf/nan match by kind)."""
    a = np.asarray(a, dtype=np.float32).reshape(-1).astype(np.float64)
    b = np.asarray(b, dtype=np.float32).reshape(-1).astype(np.float64)
    if a.shape != b.shape:
        return 1.0
    if a.size == 0:
        return 0.0
    both_nan = np.isnan(a) & np.isnan(b)
    inf_a, inf_b = np.isinf(a), np.isinf(b)
    any_inf = inf_a | inf_b
    inf_ok = inf_a & inf_b & (np.sign(a) == np.sign(b))
    with np.errstate(all="ignore"):
        denom = np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
        err = np.abs(a - b) / denom
    err = np.where(any_inf, np.where(inf_ok, 0.0, 1.0), err)
    err = np.where(both_nan, 0.0, err)
    err = np.where(np.isnan(err), 1.0, err)
    return float(err.max())
