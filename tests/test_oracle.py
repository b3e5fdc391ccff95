"""Pins the oracle before trusting it: the numpy restatement (oracle/disc_oracle.py) must
reproduce the reference build's outputs, ExecStats and BufferEvents, and both must match
the committed golden vectors (tests/golden/fixture_io.npz)."""
import json

import numpy as np
import pytest

from conftest import REF_FLAGS, FIXTURES
from oracle import disc_oracle as O


def test_golden_io_vs_numpy_oracle(fixture_io, fixture_plans):
    z, meta = fixture_io
    executors = {}  # one executor per fixture, reused across bindings like the generator
    for key, m in meta.items():
        name, bi = key.split("/")
        plan = fixture_plans[f"{name}/default"]
        inputs = {k: z[f"{key}/in/{k}"] for k in m["inputs"]}
        outs, stats, _ = executors.setdefault(name, O.Executor()).run(plan, inputs)
        assert stats == m["stats"], key
        for oi in range(m["n_out"]):
            assert O.rel_err(outs[oi], z[f"{key}/out/{oi}"]) <= 1e-6, key


def test_golden_io_vs_reference_build(ref, fixture_io, fixture_plans):
    z, meta = fixture_io
    plans = {}
    for key, m in meta.items():
        name, _ = key.split("/")
        rp = plans.setdefault(name, ref.RefPlan(fixture_plans[f"{name}/default"]))
        inputs = {k: z[f"{key}/in/{k}"] for k in m["inputs"]}
        r = rp.run(inputs)
        assert r.stats == m["stats"]
        for oi in range(m["n_out"]):
            np.testing.assert_array_equal(r.outputs[oi], z[f"{key}/out/{oi}"])


def test_reference_goldens_reproduce(ref, reference_goldens, fixtures):
    g = fixtures["softmax"]["graph"]
    assert ref.compile(g) == reference_goldens["softmax_plan.json"]
    assert ref.lower_dhlo_json(g) == reference_goldens["softmax_dhlo.json"]
    assert ref.dump_stage(g, "dhlo") == reference_goldens["softmax_ir.txt"]


@pytest.mark.parametrize("opt", list(REF_FLAGS))
def test_numpy_oracle_matches_reference_on_fixtures(ref, fixtures, fixture_plans, opt):
    for name in FIXTURES:
        plan = fixture_plans[f"{name}/{opt}"]
        rp = ref.RefPlan(plan)
        ex = O.Executor()
        for syms in fixtures[name]["bindings"]:
            inputs = ref.make_binding(fixtures[name]["graph"], syms, 7)
            try:
                r = rp.run(inputs)
            except ref.RefError as e:
                with pytest.raises(O.OracleError):
                    ex.run(plan, inputs)
                continue
            outs, stats, events = ex.run(plan, inputs)
            assert stats == r.stats, (name, opt)
            assert events == r.events, (name, opt)
            for a, b in zip(outs, r.outputs):
                assert a.shape == b.shape
                assert O.rel_err(a, b) <= 1e-6


def test_numpy_oracle_matches_reference_on_random_graphs(ref):
    """Acceptance criterion 1's seeds (acceptance_main.cpp:58-87), 40 graphs x 3 bindings."""
    rng = ref.RefRng(20260810)
    for seed in range(40):
        g = ref.random_graph(seed, 12)
        plan = ref.compile(g)
        rp = ref.RefPlan(plan)
        ex = O.Executor()
        for b in range(3):
            syms = rng.random_symbols(g)
            inputs = ref.make_binding(g, syms, seed * 31 + b)
            r = rp.run(inputs)
            outs, stats, events = ex.run(plan, inputs)
            assert stats == r.stats and events == r.events, seed
            for a, c in zip(outs, r.outputs):
                assert O.rel_err(a, c) <= 1e-5, seed


def test_rel_err_metric():
    """testutil.hpp:64-70: floor of 1, inf/nan matched by kind."""
    assert O.rel_err(np.float32([1.0]), np.float32([1.0 + 1e-6])) <= 1.1e-6
    assert O.rel_err(np.float32([np.inf]), np.float32([np.inf])) == 0.0
    assert O.rel_err(np.float32([np.inf]), np.float32([-np.inf])) == 1.0
    assert O.rel_err(np.float32([np.nan]), np.float32([np.nan])) == 0.0
    assert O.rel_err(np.float32([1e-8]), np.float32([2e-8])) < 1e-7
