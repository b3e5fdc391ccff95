"""The drop-in boundary: the C-ABI library loads (no GPU needed) and exports every symbol
include/*.h declares; compute entry points fail cleanly without a device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = []
    for h in ("disc_b200.h", "disc_cuda.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        syms += re.findall(r"\b(disc_[a-z0-9_]+)\s*\(", text)
    return sorted(set(syms))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "disc_executor_run" in syms and "disc_cuda_launch_loop" in syms and len(syms) > 60


def test_library_exports_every_declared_symbol(disc):
    lib = ctypes.CDLL(disc.api.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert missing == []


def test_compute_calls_fail_loudly_without_device(disc):
    if disc.cuda_available():
        pytest.skip("device present")
    with pytest.raises(disc.DiscError) as e:
        disc.Executor()
    assert e.value.code == 4


def test_sass_is_sm100a(disc):
    """The fatbin carries sm_100a SASS only (no PTX to JIT)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", disc.api.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ptx = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-ptx", disc.api.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert ".ptx" not in ptx


def test_generated_patterns_up_to_date(disc):
    """patterns_gen.cu must match what the current lowering produces for the library."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_patterns.py"), "--check"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
