"""The `disc` command-line tool (paper_2103_05288_b200/cli/disc_main.cpp) against the
reference CLI's contract, tests/cli_test.cmake (exit codes, stats plumbing, dump-ir
stages, ablation, bench lines).  Host-only steps run on CPU; steps that execute a plan
need the GPU."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2103_05288_b200", "disc")

# cli_test.cmake:37-38: printable payload bytes, 'AAAA' = 0x41414141 = 12.078431f
ROW8 = b"shape: 1,8\n" + b"A" * 32
ROW4 = b"shape: 1,4\n" + b"A" * 16
ROWS28 = b"shape: 2,8\n" + b"A" * 64


@pytest.fixture(scope="module")
def work(tmp_path_factory, fixtures):
    if not os.path.exists(BIN):
        from paper_2103_05288_b200 import build
        build.build(verbose=False)
    d = tmp_path_factory.mktemp("cli")
    for name, f in fixtures.items():
        (d / f"{name}.json").write_text(f["graph"] if isinstance(f["graph"], str) else json.dumps(f["graph"]))
    (d / "x.tensor").write_bytes(ROW8)
    (d / "w.tensor").write_bytes(ROW4)
    (d / "x28.tensor").write_bytes(ROWS28)
    return d


def disc(work, *args, rc=0, env=None):
    e = dict(os.environ, DISC_STATS_FILE=str(work / "stats.json"))
    e.update(env or {})
    r = subprocess.run([BIN, *map(str, args)], cwd=work, capture_output=True, text=True, env=e, timeout=300)
    assert r.returncode == rc, (args, r.returncode, r.stdout, r.stderr)
    return r.stdout + r.stderr


def test_compile_and_stats(work):
    out = disc(work, "compile", "softmax.json", "-o", "plan_c.json", "--stats-file", "c.json")
    assert "compiled" in out and "2 kernels" in out and "12 host instructions" in out
    assert "compile_count=1" in disc(work, "stats", "--stats-file", "c.json")
    disc(work, "compile", "softmax.json", "-o", "plan_c.json", "--stats-file", "c.json")
    j = json.loads(disc(work, "stats", "--json", "--stats-file", "c.json"))
    assert j["compile_count"] == 2 and j["host_instruction_count"] == 12 and j["launch_count"] == 0
    # the plan file is the library's plan JSON (plan_from_json round trip)
    import paper_2103_05288_b200 as D
    text = (work / "plan_c.json").read_text()
    assert D.CompiledPlan.from_json(text).to_json() == text


def test_dump_ir_stages(work):
    assert "dims:" in disc(work, "dump-ir", "split.json", "--stage=constraints")
    assert "elementwise-loop" in disc(work, "dump-ir", "split.json", "--stage", "fused")
    assert "reduce_max" in disc(work, "dump-ir", "softmax.json", "--stage=dhlo")
    disc(work, "compile", "softmax.json", "-o", "plan_d.json", "--stats-file", "d.json",
         env={"DISC_DUMP_DIR": str(work / "dumps")})
    import paper_2103_05288_b200 as D
    graph = (work / "softmax.json").read_text()
    for st in ("dhlo", "constraints", "simplified", "fused", "program"):  # softmax: no constraint sets
        assert (work / "dumps" / f"{st}.txt").read_text() == D.dump_stage(graph, st)


def test_error_exit_codes(work):
    disc(work, "compile", rc=2)
    disc(work, rc=2)
    disc(work, "frobnicate", rc=2)
    disc(work, "compile", "does_not_exist.json", rc=2)
    disc(work, "dump-ir", "softmax.json", "--stage=bogus", rc=2)
    disc(work, "run", "plan_c.json", "--input", "x_no_equals", rc=2)
    (work / "bad.json").write_text("{ not json")
    assert "error[parse]" in disc(work, "compile", "bad.json", rc=3)
    (work / "invalid.json").write_text(json.dumps({
        "name": "g", "inputs": [{"id": "x", "shape": [4], "dtype": "f32"}], "outputs": ["y"],
        "nodes": [{"id": "y", "op": "Exp", "inputs": ["zz"]}]}))
    assert "error[validation]" in disc(work, "compile", "invalid.json", rc=3)
    disc(work, "compile", "softmax.json", "-o", "plan_e.json", "--stats-file", "e.json")
    assert "error[runtime]" in disc(work, "run", "plan_e.json", "--input", "x=missing.tensor", rc=4)
    assert disc(work, "--help").startswith("disc")


def test_ablation_compiles_differ(work):
    disc(work, "compile", "split.json", "-o", "split_with.json", "--stats-file", "s1.json")
    disc(work, "compile", "split.json", "-o", "split_without.json", "--no-injected-constraints",
         "--stats-file", "s2.json")
    a = json.loads((work / "split_with.json").read_text())
    b = json.loads((work / "split_without.json").read_text())
    assert len(a["kernels"]) == 1 and len(b["kernels"]) == 2


@pytest.mark.gpu
def test_run_stats_accumulate(work):
    disc(work, "compile", "softmax.json", "-o", "plan.json", "--stats-file", "r.json")
    out = disc(work, "run", "plan.json", "--input", "x=x.tensor", "--out-dir", "out", "--stats-file", "r.json")
    assert "output y shape=[1,8]" in out
    disc(work, "run", "plan.json", "--input", "x=x.tensor", "--stats-file", "r.json")
    st = disc(work, "stats", "--stats-file", "r.json")
    assert "compile_count=1" in st and "launch_count=4" in st  # two runs, two launches each
    raw = (work / "out" / "y.tensor").read_bytes()
    head, data = raw.split(b"\n", 1)
    assert head == b"shape: 1,8"
    np.testing.assert_array_equal(np.frombuffer(data, "<f4"), np.full(8, 0.125, np.float32))


@pytest.mark.gpu
def test_run_outputs_match_oracle(work, fixtures, ref):
    """`run` output tensors equal the reference executor's (oracle/_ref) on the transformer
    fixture, GEMMs included (1e-5 rel_err, testutil.hpp:64-70)."""
    gtext = fixtures["transformer"]["graph"]
    disc(work, "compile", "transformer.json", "-o", "tf.json", "--stats-file", "t.json")
    binding = ref.make_binding(gtext, {"S0": 5}, 7)
    args = []
    for name, arr in binding.items():
        a = np.ascontiguousarray(arr, np.float32)
        (work / f"in_{name}.tensor").write_bytes(
            f"shape: {','.join(map(str, a.shape))}\n".encode() + a.astype("<f4").tobytes())
        args += ["--input", f"{name}=in_{name}.tensor"]
    disc(work, "run", "tf.json", *args, "--out-dir", "tf_out", "--stats-file", "t.json")
    want = ref.eval_eager(gtext, binding).outputs
    for oid, w in zip(json.loads(gtext)["outputs"], want):
        raw = (work / "tf_out" / f"{oid}.tensor").read_bytes()
        got = np.frombuffer(raw.split(b"\n", 1)[1], "<f4")
        w = np.asarray(w, np.float32).ravel()
        assert got.shape == w.shape
        assert np.max(np.abs(got - w) / np.maximum(1.0, np.abs(w))) <= 1e-5, oid


@pytest.mark.gpu
def test_ablation_launch_counts(work):
    disc(work, "compile", "split.json", "-o", "sw.json", "--stats-file", "a1.json")
    disc(work, "compile", "split.json", "-o", "swo.json", "--no-injected-constraints", "--stats-file", "a2.json")
    ins = ["--input", "x=x.tensor", "--input", "w0=w.tensor", "--input", "w1=w.tensor"]
    disc(work, "run", "sw.json", *ins, "--stats-file", "a1.json")
    disc(work, "run", "swo.json", *ins, "--stats-file", "a2.json")
    assert "launch_count=1" in disc(work, "stats", "--stats-file", "a1.json")
    assert "launch_count=2" in disc(work, "stats", "--stats-file", "a2.json")


@pytest.mark.gpu
def test_bench_lines(work):
    disc(work, "compile", "softmax.json", "-o", "plan_b.json", "--stats-file", "b.json")
    (work / "shapes.json").write_text('[{"S0": 2}, {"S0": 5}]')
    out = disc(work, "bench", "plan_b.json", "--shapes", "shapes.json", "--reps", "20", "--stats-file", "b.json")
    assert "launch_count=2" in out and "not" in out
    assert out.count("shape {") == 2
    rep = disc(work, "bench", "plan_b.json", "--shapes", "shapes.json", "--json", "--stats-file", "b.json")
    rows = json.loads(rep[rep.index("["):])
    assert [r["binding"] for r in rows] == [{"S0": 2}, {"S0": 5}]
    assert all(r["launch_count"] == 2 and r["kernel_ms"] > 0 for r in rows)
    disc(work, "compile", "transformer.json", "-o", "tf_plan.json", "--stats-file", "b.json")
    (work / "tf_shapes.json").write_text('[{"S0": 4}]')
    out = disc(work, "bench", "tf_plan.json", "--shapes", "tf_shapes.json", "--reps", "20", "--stats-file", "b.json")
    assert "eager_op_count=54" in out and "launch_ratio=0.333333" in out


@pytest.mark.gpu
def test_eager_and_static(work):
    out = disc(work, "run", "--eager", "softmax.json", "--input", "x=x28.tensor", "--out-dir", "eager_out")
    assert "output y shape=[2,8]" in out
    got = np.frombuffer((work / "eager_out" / "y.tensor").read_bytes().split(b"\n", 1)[1], "<f4")
    np.testing.assert_allclose(got, np.full(16, 0.125, np.float32), rtol=1e-6)
    (work / "static.json").write_text(json.dumps({
        "name": "s", "inputs": [{"id": "x", "shape": [1, 8], "dtype": "f32"}], "outputs": ["y"],
        "nodes": [{"id": "y", "op": "Exp", "inputs": ["x"]}]}))
    disc(work, "compile", "static.json", "-o", "static_plan.json", "--static-fallback", "--stats-file", "st.json")
    out = disc(work, "run", "static_plan.json", "--input", "x=x.tensor", "--out-dir", "st_out", "--stats-file", "st.json")
    assert "output y shape=[1,8]" in out
    got = np.frombuffer((work / "st_out" / "y.tensor").read_bytes().split(b"\n", 1)[1], "<f4")
    np.testing.assert_allclose(got, np.exp(np.full(8, np.frombuffer(b"AAAA", "<f4")[0])), rtol=1e-6)
