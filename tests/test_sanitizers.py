"""compute-sanitizer over every kernel family (the GPU analogue of the
reference's by-construction race freedom): memcheck (out-of-bounds / misaligned
accesses, leaks of device errors), racecheck (shared-memory hazards of the
warp-synchronous tables and CTA-tier bitmaps) and synccheck (barrier misuse) on
tools/sanitize_target.py, which also checks every count against the oracle."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    env = dict(os.environ, SMG_HEAVY_MIN="0", SMG_HEAVY_STREAM="1")
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "9", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_target.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=3000)
    out = p.stdout + p.stderr
    log = os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    with open(log, "w") as f:
        f.write(out)
    if "compute-sanitizer is closed" in out:
        # the GPU pool disables the tool (its wrapper says so and exits non-zero):
        # run the same target bare -- every count is still compared with the oracle
        q = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_target.py")], env=env,
                           capture_output=True, text=True, timeout=3000)
        assert q.returncode == 0 and "sanitize target: OK" in q.stdout + q.stderr, (q.stdout + q.stderr)[-4000:]
        pytest.skip("compute-sanitizer is closed on this GPU pool; target ran bare and matched the oracle")
    assert p.returncode == 0, out[-4000:]
    assert "sanitize target: OK" in out
    assert "ERROR SUMMARY: 0 errors" in out
