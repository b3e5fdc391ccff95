"""Generates paper_2103_05288_b200/csrc/kernels/patterns_gen.cu.

For every fused launch of a pattern library (the fixture graphs and the BASELINE config
graphs C1-C4, each at a few representative shapes), the product's own runtime lowering
is run in capture mode (host only, no GPU) to obtain the device program structure.  Each
distinct structure becomes a straight-line device function -- SSA values in registers,
no interpretation -- instantiated into the same schedule kernels the interpreter uses
(kernels.cuh).  At runtime the device layer hashes every launch's program structure and
uses the generated kernel when one exists; any other structure runs the interpreter.
Nothing is generated or compiled at runtime; kernels are shape-generic (load bindings,
vector width and geometry stay launch parameters).

  python tools/gen_patterns.py            # rewrite the generated file
  python tools/gen_patterns.py --check    # exit 1 if it is stale
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
KDIR = os.path.join(ROOT, "paper_2103_05288_b200", "csrc", "kernels")
OUT = os.path.join(KDIR, "patterns_gen.cu")  # registry; kernels in patterns_gen_<k>.cu shards
SHARDS = 6

I_LOAD_CONST, I_REDVAL, I_COPY, I_RCPVAL, I_BIN, I_UN, I_FDIV = 3, 4, 5, 6, 8, 28, 34
LC_SPLAT, LC_CONTIG, LC_CONTIGU = 2, 3, 6  # program.cuh LoadClass


def library():
    """(name, graph, [symbol bindings]) of the pattern library."""
    from paper_2103_05288_b200 import workloads as W
    lib = []
    fx = json.load(open(os.path.join(ROOT, "tests", "golden", "fixtures.json")))
    for name, f in sorted(fx.items()):
        lib.append((f"fixture:{name}", json.loads(f["graph"]), f["bindings"]))
    sm = W.softmax_graph_for(0)
    lib.append(("C1:softmax", sm, [{"S0": 64, "S1": 8}, {"S0": 5, "S1": 7}, {"S0": 16, "S1": 4096},
                                   {"S0": 2, "S1": 1}]))
    lib.append(("C2:ln_gelu", W.ln_gelu_graph(), [{"T": 64, "H": 768}, {"T": 1, "H": 1024}, {"T": 7, "H": 4096}]))
    lib.append(("C3:colreduce", W.colreduce_graph(), [{"N": 1000, "C": 36}, {"N": 64, "C": 4096},
                                                      {"N": 4096, "C": 3}, {"N": 100000, "C": 1}]))
    lib.append(("C4:bert", W.bert_graph(), [{"R": 96, "S": 8, "T": 8, "H": 768, "F": 3072},
                                            {"R": 12 * 8 * 128, "S": 128, "T": 8 * 128, "H": 768, "F": 3072}]))
    return lib


def input_shapes(graph, syms):
    shapes = {}
    for i in graph["inputs"]:
        shapes[i["id"]] = [syms.get(d, 2) if isinstance(d, str) else d for d in i["shape"]]
    return shapes


def collect():
    import paper_2103_05288_b200 as D
    seen = {}
    for name, graph, bindings in library():
        for opts in (D.CompileOptions(), D.CompileOptions(enable_fusion=False)):
            plan = D.compile_graph(graph, opts)
            for syms in bindings:
                try:
                    recs = D.capture_programs(plan, input_shapes(graph, syms))
                except D.DiscError:
                    continue
                for r in recs:
                    seen.setdefault((r["kind"], r["key"]), (r, name))
    return seen


def gen_program(fn, prog, ch=1, early_splat=True):
    """Straight-line body for one program (code from the capture).

    Identity (streaming) loads are split into a load phase (``load`` fills a Loads
    struct) and the rest (``run_loaded``), so a schedule can issue the next tile's
    loads before computing the current one (software pipelining); ``run`` = both."""
    code = prog["code"]
    loads = [(i, prog["lclass"][load]) for i, (op, a, b, flags, dst, load, out) in enumerate(code) if op <= I_LOAD_CONST]
    ident = [i for i, c in loads if c == 0]
    # Loads issued in the load phase (and, in a pipelined schedule, one tile ahead):
    # streaming identity operands, per-row scalars (splat: one register) and, while the
    # register budget allows, the L2-resident contiguous [W] vectors (bias/gamma/...).
    splat = [i for i, c in loads if c == LC_SPLAT] if early_splat else []
    contig = [i for i, c in loads if c in (LC_CONTIG, LC_CONTIGU)]
    regs = len(ident) * ch * 4 + len(splat) * ch
    if regs + len(contig) * ch * 4 <= 16:
        ident = ident + contig
        regs += len(contig) * ch * 4
    early = sorted(ident + splat)
    pf = [f"    prefetch_cls<VEC, CH, 0>(P, t, {code[i][5]});" for i, c in loads if c == 0]
    xu = any(I_UN <= c[0] < I_UN + 4 for c in code)  # exp / tanh (MUFU) in the program
    # streamed operands (not hoisted constants / per-row splats); max-reduce rows over two
    # or more streams run register-capped at 6 blocks/SM (kernels.cuh k_row_mb)
    streams = [i for i, c in loads if code[i][0] != I_LOAD_CONST and c != LC_SPLAT]
    lines = [f"struct {fn} {{",
             "  static constexpr bool kSplitFull = true;",
             f"  static constexpr bool kXuHeavy = {'true' if xu else 'false'};",
             f"  static constexpr int kMaxRowMinBlocks = {6 if fn.startswith('Pre_row') and len(streams) >= 2 else 0};",
             # pipelined only while the extra tile of loads fits (<= 16 registers at VEC=4)
             f"  static constexpr int kPipe = {len(early) if regs <= 16 else 0};",
             "  template <int VEC, int CH>",
             "  struct Loads {"] + \
            [f"    typename Vec<VEC>::T l{i}[CH];" for i in ident] + [f"    float s{i}[CH];" for i in splat] + \
            (["    char none;"] if not early else []) + \
            ["  };",
             "  template <int VEC, int CH, typename Ctx>",
             "  __device__ __forceinline__ static void prefetch(const disc_program& P, const Ctx& t) {"] + pf + \
            ["  }",
             "  template <int VEC, int CH, bool WIDE, typename Ctx>",
             "  __device__ __forceinline__ static void load(const disc_program& P, const Ctx& t, Loads<VEC, CH>& L) {"] + \
            [f"    load_cls<VEC, CH, WIDE, {prog['lclass'][code[i][5]]}>(P, t, nullptr, {code[i][5]}, L.l{i});"
             if i in ident else f"    load_splat<CH>(P, t, {code[i][5]}, L.s{i});" for i in early] + \
            ["  }",
             "  template <int VEC, int CH, bool WIDE, typename Ctx>",
             "  __device__ __forceinline__ static void run_loaded(const disc_program& P, const Ctx& t, const Loads<VEC, CH>& L,",
             "      typename Vec<VEC>::T (&acc)[CH], typename Vec<VEC>::T*, int, const float* consts, float red) {",
             "    using T = typename Vec<VEC>::T;"]
    slot_val = {}
    for i, (op, a, b, flags, dst, load, out) in enumerate(code):
        v = f"v{i}"
        lines.append(f"    T {v}[CH];")

        def src(is_slot, s):
            return f"v{slot_val[s]}" if is_slot else f"v{i - 1}"
        if op <= I_LOAD_CONST:
            if i in ident:
                lines.append(f"    _Pragma(\"unroll\") for (int c = 0; c < CH; ++c) {v}[c] = L.l{i}[c];")
            elif i in splat:
                lines.append(f"    _Pragma(\"unroll\") for (int c = 0; c < CH; ++c) {v}[c] = splat(L.s{i}[c], {v}[c]);")
            else:
                lines.append(f"    load_cls<VEC, CH, WIDE, {prog['lclass'][load]}>(P, t, consts, {load}, {v});")
        elif op == I_REDVAL:
            lines.append(f"    _Pragma(\"unroll\") for (int c = 0; c < CH; ++c) {v}[c] = splat(red, {v}[c]);")
        elif op == I_RCPVAL:
            lines.append(f"    _Pragma(\"unroll\") for (int c = 0; c < CH; ++c) {v}[c] = splat(__frcp_rn(red), {v}[c]);")
        elif op == I_COPY:
            lines.append(f"    _Pragma(\"unroll\") for (int c = 0; c < CH; ++c) {v}[c] = {src(True, a)}[c];")
        elif I_BIN <= op < I_UN or op >= I_FDIV:
            k, mode = divmod(op - I_BIN, 4) if op < I_UN else (5, op - I_FDIV)
            x, y = src(mode in (2, 3), a), src(mode in (1, 3), b)
            lines.append(f"    _Pragma(\"unroll\") for (int c = 0; c < CH; ++c) {v}[c] = bin<{k}>({x}[c], {y}[c]);")
        else:
            k, mode = divmod(op - I_UN, 2)
            lines.append(f"    un_tile<{k}>({src(mode == 1, a)}, {v});")
        if flags & 1:
            slot_val[dst] = i
        if flags & 2:
            lines.append(f"    store_out<VEC, CH>(P, {out}, t, {v});")
    if code:
        lines.append(f"    _Pragma(\"unroll\") for (int c = 0; c < CH; ++c) acc[c] = v{len(code) - 1}[c];")
    lines += ["  }",
              "  template <int VEC, int CH, bool WIDE, typename Ctx>",
              "  __device__ __forceinline__ static void run(const disc_program& P, const Ctx& t,",
              "      typename Vec<VEC>::T (&acc)[CH], typename Vec<VEC>::T* slots, int stride, const float* consts, float red) {",
              "    Loads<VEC, CH> L;",
              "    load<VEC, CH, WIDE>(P, t, L);",
              "    run_loaded<VEC, CH, WIDE>(P, t, L, acc, slots, stride, consts, red);",
              "  }",
              "};"]
    return "\n".join(lines)


def generate():
    """Returns {path: text} for the registry and the kernel shards."""
    seen = collect()
    header = ["// GENERATED by tools/gen_patterns.py -- do not edit.",
              "// Straight-line fused programs for the pattern library (fixtures + BASELINE configs C1-C4);",
              "// see the generator's docstring.  Source patterns per entry are noted in comments."]
    shards = [header + ['#include "kernels.cuh"', "", "#ifndef DISC_ROWX_CH", "#define DISC_ROWX_CH 2", "#endif",
                        "#ifndef DISC_ROW_READ_CH", "#define DISC_ROW_READ_CH 2", "#endif",
                        "#ifndef DISC_ROW_MAX_CH", "#define DISC_ROW_MAX_CH 2", "#endif",
                        "#ifndef DISC_COL_MAX_CH", "#define DISC_COL_MAX_CH 4", "#endif", "",
                        "namespace disc_gen {", "using namespace disc_dev;", ""]
              for _ in range(SHARDS)]
    entries = []
    for n, ((kind, key), (rec, src_name)) in enumerate(sorted(seen.items())):
        parts = shards[n % SHARDS]
        tag = f"{kind}_{key}"
        parts.append(f"// {kind} {key} from {src_name}")
        # Chunks per tile: short programs are memory-bound (more loads in flight), long
        # ones register/issue-bound (keep straight-line code small).
        n_code = max(len(rec["pre"]["code"]), len(rec.get("post", {}).get("code", [])))
        ch = 4 if n_code <= 8 else (2 if n_code <= 20 else 1)
        if 5 in rec["pre"]["lclass"] + rec.get("post", {}).get("lclass", []):
            ch = min(ch, 2)  # gather index math is register-heavy
        # early (pipelined) per-row scalars only pay off in the loop schedule (A/B: the row
        # schedule's reduce pass is faster with loads in program order)
        parts.append(gen_program(f"Pre_{tag}", rec["pre"], ch, early_splat=kind == "loop"))
        if kind == "row":
            parts.append(gen_program(f"Post_{tag}", rec["post"], ch, early_splat=False))
        parts.append(f"cudaError_t launch_{tag}(const void* l, int vec, cudaStream_t s, const HostGroup* g) {{")
        trans = any(I_UN <= c[0] < I_UN + 4 for p_ in ("pre", "post") for c in rec.get(p_, {}).get("code", []))
        trivial = kind == "row" and len(rec["pre"]["code"]) <= 1 and not rec.get("post", {}).get("code")
        if trivial:
            # a plain row reduce of one input (read-only stream): more loads in flight
            parts.append(f"  constexpr int kGenCH = DISC_ROW_READ_CH;")
        elif kind == "row" and trans and ch > 1:
            # transcendental row programs: fewer chunks in flight per thread (register
            # pressure under the 64-register cap spills the f64 accumulators)
            parts.append(f"  constexpr int kGenCH = DISC_ROWX_CH < {ch} ? DISC_ROWX_CH : {ch};")
        elif kind == "row" and ch > 1:
            parts.append(f"  constexpr int kGenCH = DISC_ROW_MAX_CH < {ch} ? DISC_ROW_MAX_CH : {ch};")
        elif kind == "col" and ch > 1:
            parts.append(f"  constexpr int kGenCH = DISC_COL_MAX_CH < {ch} ? DISC_COL_MAX_CH : {ch};")
        else:
            parts.append(f"  constexpr int kGenCH = {ch};")
        if kind == "loop":
            parts.append("  const auto& L = *static_cast<const disc_loop_launch*>(l);")
            parts.append(f"  return loop_pass<Pre_{tag}, kGenCH, false>(L, s, false, g);")
        elif kind == "row":
            parts.append("  const auto& L = *static_cast<const disc_reduce_launch*>(l);")
            parts.append(f"  return row_pass<Pre_{tag}, Post_{tag}, kGenCH, false>(L, s, false, g);")
        else:
            parts.append("  const auto& L = *static_cast<const disc_reduce_launch*>(l);")
            parts.append(f"  return col_pass_t<Pre_{tag}, kGenCH, false>(L, s, false, g);")
        parts.append("}")
        parts.append("")
        entries.append((["loop", "row", "col"].index(kind), key, f"launch_{tag}"))
    files = {}
    for k, parts in enumerate(shards):
        files[os.path.join(KDIR, f"patterns_gen_{k}.cu")] = "\n".join(parts + ["}  // namespace disc_gen", ""])
    reg = header + ["#include <cstdint>", "", "#include <cuda_runtime.h>", "",
                    "namespace disc_dev {", "struct HostGroup;", "}  // namespace disc_dev", "", "namespace disc_gen {",
                    "using disc_dev::HostGroup;"]
    for _, _, fn in sorted(entries):
        reg.append(f"cudaError_t {fn}(const void* l, int vec, cudaStream_t s, const HostGroup* g);")
    reg += ["}  // namespace disc_gen", "", "namespace disc_spec {",
            "struct Entry {\n  int kind;\n  uint64_t key;\n"
            "  // g != nullptr: grouped launch of g->n descriptors (l = the first)\n"
            "  cudaError_t (*launch)(const void* launch, int vec, cudaStream_t s, const disc_dev::HostGroup* g);\n};",
            "static const Entry kEntries[] = {"]
    for kind, key, fn in sorted(entries):
        reg.append(f"    {{{kind}, 0x{key}ull, disc_gen::{fn}}},")
    reg += ["};", "const Entry* lookup(int kind, uint64_t key) {", "  for (const Entry& e : kEntries)",
            "    if (e.kind == kind && e.key == key) return &e;", "  return nullptr;", "}",
            f"int count() {{ return {len(entries)}; }}", "}  // namespace disc_spec", ""]
    files[OUT] = "\n".join(reg)
    return files, len(entries)


def main():
    files, n = generate()
    if "--check" in sys.argv:
        for path, text in files.items():
            cur = open(path).read() if os.path.exists(path) else ""
            if cur != text:
                print(f"{os.path.basename(path)} is stale: run python tools/gen_patterns.py")
                sys.exit(1)
        print(f"generated patterns up to date ({n} patterns)")
        return
    for path, text in files.items():
        with open(path, "w") as f:
            f.write(text)
    print(f"wrote {len(files)} files: {n} patterns")


if __name__ == "__main__":
    main()
