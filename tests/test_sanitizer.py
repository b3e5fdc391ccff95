"""compute-sanitizer over every kernel family (memcheck, racecheck, synccheck), single and
grouped launches with programmatic dependent launch on: tools/sanitize_smoke.py, which
also checks every output against the numpy oracle."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(gpu, tool):
    if not os.path.exists(SAN):
        pytest.fail("compute-sanitizer not found")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20", "python",
           os.path.join(ROOT, "tools", "sanitize_smoke.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT,
                       env=dict(os.environ, DISC_PIN_THREADS="0"))
    out = r.stdout + r.stderr
    print(out[-3000:])
    if r.returncode != 0 and "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses to run (pool policy); the same
        # smoke runs without it in test_sanitize_smoke_outputs below
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert r.returncode == 0, out[-3000:]
    assert "sanitize smoke:" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-2000:]


def test_sanitize_smoke_outputs(gpu):
    """The sanitizer smoke itself (every kernel family, single and grouped launches, PDL on),
    each output checked against the numpy oracle -- without the sanitizer."""
    r = subprocess.run(["python", os.path.join(ROOT, "tools", "sanitize_smoke.py")], capture_output=True, text=True,
                       timeout=900, cwd=ROOT, env=dict(os.environ, DISC_PIN_THREADS="0"))
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "sanitize smoke:" in out
