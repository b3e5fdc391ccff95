"""Parity of the EXACT benchmarked passes (bench.py): every BASELINE config's sweep is run
the way bench.py times it -- one step's requests through disc_executor_run_grouped in the
bench's chunks, with its host threads and two flush phases, inputs in the device arena --
and the outputs are checked against the reference executor (oracle/_ref) by
oracle/verify.py: every request whose inputs have <= 2^22 elements in full, sampled rows /
columns of every larger one.  Gate: the reference's floored rel_err <= 1e-5
(tests/testutil.hpp:64-70); the true relative error and ulp error are printed per config.
"""
import os
import types

import pytest

pytestmark = pytest.mark.gpu


def _bench_args(**kw):
    a = types.SimpleNamespace(schedule="auto", host_threads=min(16, os.cpu_count() or 1), cache_gb=8.0,
                              arena_gb=48.0, chunk_gb=128.0)
    a.__dict__.update(kw)
    return a


@pytest.mark.parametrize("workload,requests", [("ln_gelu", None), ("softmax", None), ("colreduce", None),
                                               ("bert", None), ("stream", None), ("sweep", 3000)])
def test_benchmarked_sweep_matches_reference(gpu, ref, workload, requests):
    import bench
    wl = bench.make_workload(workload, 0, requests or 10000)
    B = bench.Bench(gpu, _bench_args(), 0, wl)
    try:
        reqs = wl.requests(3)  # a step the bench would time (warmup 3): fresh shapes for the sweep
        batch = B.batch(reqs)
        batch.run(B.ex)  # warm pass, as the bench's warmup
        res = bench.verify_pass(B, wl, batch, "full", threads=max(1, (os.cpu_count() or 2) - 1))
    finally:
        B.close()
    print(f"\n{workload}: {res['requests_checked']} max floored {res['max_rel_err_floored']} true "
          f"{res['max_rel_err_true']} ulp {res['max_ulp']} over1e-5(true) {res['elements_over_1e-5_true']} "
          f"of {res['elements']}; per pattern {res['per_pattern']}")
    assert res["pass"], res["failures"]
    assert sum(res["requests_checked"].values()) > 0
