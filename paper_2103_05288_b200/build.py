"""Builds paper_2103_05288_b200/libdisc_b200.so in-tree (host C++ + sm_100a CUDA).

    python -m paper_2103_05288_b200.build        # incremental
    python -m paper_2103_05288_b200.build --clean

Host C++ is compiled with the system g++ (C++20), CUDA with nvcc for
-gencode arch=compute_100a,code=sm_100a only (no PTX fallback, no JIT), IEEE f32 math
(--fmad=false, precise div/sqrt; the reference's CPU objects contain no FMA) and
-lineinfo for ncu source mapping.  cudart is linked statically so the .so is
self-contained on the GPU box.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
import site
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libdisc_b200.so")
# A/B experiment builds: DISC_BUILD_VARIANT=<name> DISC_NVCC_DEFS="-DKNOB=0" builds
# libdisc_b200_<name>.so in its own object dir (selected at run time by DISC_LIB_VARIANT).
_VARIANT = os.environ.get("DISC_BUILD_VARIANT")
if _VARIANT:
    BUILD = os.path.join(PKG, f"_build_{_VARIANT}")
    LIB = os.path.join(PKG, f"libdisc_b200_{_VARIANT}.so")

CXX = shutil.which("g++", path="/usr/bin") or "g++"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter",
            "-ffp-contract=off"]
NVCCFLAGS = ["-std=c++17", "-O3", "-lineinfo", "--fmad=false", "-prec-div=true", "-prec-sqrt=true",
             "-Xcompiler", "-fPIC", "-Xptxas", "-O3", "--expt-relaxed-constexpr"] + ARCH + \
    os.environ.get("DISC_NVCC_DEFS", "").split()


def _json_header() -> str:
    """nlohmann/json 3.11.3 from the image (cudnn_frontend's copy), with its local
    one-line-int-array printing patch reverted to stock pretty-printing."""
    out = os.path.join(BUILD, "include", "json.hpp")
    if os.path.exists(out):
        return os.path.dirname(out)
    src = None
    for p in site.getsitepackages() + [site.getusersitepackages()]:
        cand = os.path.join(p, "include", "cudnn_frontend", "thirdparty", "nlohmann", "json.hpp")
        if os.path.exists(cand):
            src = cand
            break
    if src is None:
        raise RuntimeError("nlohmann/json.hpp not found in site-packages")
    text = open(src).read()
    patched = text.replace(
        "if (pretty_print && (elementType != value_t::number_integer) &&\n"
        "                    (elementType != value_t::number_unsigned))", "if (pretty_print)")
    if patched == text:
        raise RuntimeError("json.hpp patch point not found")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        f.write(patched)
    return os.path.dirname(out)


def _sources():
    cpp, cu = [], []
    for d, _, files in os.walk(CSRC):
        for f in sorted(files):
            p = os.path.join(d, f)
            if f.endswith(".cpp"):
                cpp.append(p)
            elif f.endswith(".cu"):
                cu.append(p)
    return sorted(cpp), sorted(cu)


def _headers_digest() -> str:
    h = hashlib.sha1()
    for d, _, files in os.walk(CSRC):
        for f in sorted(files):
            if f.endswith((".hpp", ".h", ".cuh")):
                h.update(open(os.path.join(d, f), "rb").read())
    h.update(open(os.path.join(ROOT, "include", "disc_b200.h"), "rb").read())
    h.update(open(os.path.join(ROOT, "include", "disc_cuda.h"), "rb").read())
    h.update(" ".join(CXXFLAGS + NVCCFLAGS).encode())
    return h.hexdigest()[:12]


def _compile(src: str, inc: list, tag: str) -> str:
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    obj = os.path.join(BUILD, "obj", f"{rel}.{tag}.o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= os.path.getmtime(src):
        return obj
    os.makedirs(os.path.dirname(obj), exist_ok=True)
    incs = [f"-I{i}" for i in inc]
    if src.endswith(".cu"):
        cmd = [NVCC, *NVCCFLAGS, *incs, "-c", src, "-o", obj]
    else:
        cmd = [CXX, *CXXFLAGS, *incs, "-I/usr/local/cuda/include", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj


def build(clean: bool = False, verbose: bool = True) -> str:
    if clean and os.path.exists(BUILD):
        shutil.rmtree(BUILD)
    os.makedirs(BUILD, exist_ok=True)
    inc = [_json_header(), CSRC, os.path.join(ROOT, "include")]
    tag = _headers_digest()
    cpp, cu = _sources()
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, inc, tag), cpp + cu))
    keep = set(objs)
    for f in os.listdir(os.path.join(BUILD, "obj")):  # objects of older header digests
        path = os.path.join(BUILD, "obj", f)
        if path not in keep:
            os.remove(path)
    exports = os.path.join(CSRC, "exports.map")
    newest = max([os.path.getmtime(o) for o in objs] + [os.path.getmtime(exports)])
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread", "-ldl", "-lrt",
               f"-Xlinker=--version-script={exports}"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"built {LIB}")
    if not _VARIANT:
        build_cli(inc, verbose)
    return LIB


CLI_SRC = os.path.join(PKG, "cli", "disc_main.cpp")
CLI_BIN = os.path.join(PKG, "disc")


def build_cli(inc: list, verbose: bool = True) -> str:
    """The `disc` command-line tool (cli/disc_main.cpp), linked against the in-tree
    library with an $ORIGIN rpath so it runs from the package directory."""
    if os.path.exists(CLI_BIN) and os.path.getmtime(CLI_BIN) >= max(os.path.getmtime(CLI_SRC), os.path.getmtime(LIB)):
        return CLI_BIN
    cmd = [CXX, *[f for f in CXXFLAGS if f != "-fPIC"], *[f"-I{i}" for i in inc], CLI_SRC, LIB,
           "-Wl,-rpath,$ORIGIN", "-o", CLI_BIN]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"cli build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {CLI_BIN}")
    return CLI_BIN


if __name__ == "__main__":
    build(clean="--clean" in sys.argv)
