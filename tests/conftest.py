"""Shared test plumbing.

Markers: ``gpu`` -- needs a CUDA device (run on the B200 box).  Everything else runs on
CPU here.  The reference oracle (oracle/_ref/libdisc_ref.so, test infrastructure only)
is used as the checker wherever it is built; committed goldens under tests/golden/ pin
the same facts when it is not.
"""
from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running sweep")


def load_json(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rt") as f:
            return json.load(f)
    with open(path) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def fixtures():
    return load_json("fixtures.json")


@pytest.fixture(scope="session")
def fixture_plans():
    return load_json("fixture_plans.json")


@pytest.fixture(scope="session")
def random_plans():
    return load_json("random_plans.json.gz")


@pytest.fixture(scope="session")
def reference_goldens():
    return load_json("reference_goldens.json")


@pytest.fixture(scope="session")
def fixture_io():
    z = np.load(os.path.join(GOLDEN, "fixture_io.npz"))
    meta = json.loads(bytes(z["__meta__"]).decode())
    return z, meta


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("reference oracle not built (make -C oracle)")
    return R


@pytest.fixture(scope="session")
def disc():
    import paper_2103_05288_b200 as D
    D.lib()  # fails loudly if the CUDA library is missing
    return D


@pytest.fixture(scope="session")
def gpu(disc):
    if not disc.cuda_available():
        pytest.fail("GPU test requested but no CUDA device is visible")
    return disc


OPTION_SETS = {
    "default": dict(inject_constraints=True, enable_fusion=True, static_fallback=False),
    "no_inject": dict(inject_constraints=False, enable_fusion=True, static_fallback=False),
    "no_fusion": dict(inject_constraints=True, enable_fusion=False, static_fallback=False),
    "static_fb": dict(inject_constraints=True, enable_fusion=True, static_fallback=True),
}
REF_FLAGS = {
    "default": dict(inject=True, fusion=True, static_fallback=False),
    "no_inject": dict(inject=False, fusion=True, static_fallback=False),
    "no_fusion": dict(inject=True, fusion=False, static_fallback=False),
    "static_fb": dict(inject=True, fusion=True, static_fallback=True),
}
FIXTURES = ["chain", "softmax", "split", "reshape", "matmul", "diamond", "empty", "transformer"]


def fixture_binding(name, i):
    """acceptance_main.cpp:43-46"""
    if name == "split":
        return {"S0": i, "T0": i, "T1": i}
    return {"S0": i}
