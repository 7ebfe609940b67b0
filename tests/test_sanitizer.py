"""compute-sanitizer over the emitted kernels (race
detection): the reference checks races dynamically with write footprints in
its simulator (SRC/eval_imp.py:252-263, SRC/opencl.py:450-470); on the B200
the same guarantee is checked on the hardware.

* racecheck -- shared-memory RAW/WAR/WAW hazards, i.e. the BarrierPlanner's
  barrier placement (loop-carried hazards, rotated pipelined stagings);
* memcheck  -- out-of-bounds / misaligned global and shared accesses (vec4
  views, 64-bit indices, scratch slices);
* synccheck -- divergent or invalid __syncthreads (fused grid tails).

The workload (tests/sanitize_run.py) also checks every result against the
oracle."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["racecheck", "memcheck", "synccheck"])
def test_compute_sanitizer(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, DPIA_SANITIZE_FUZZ="40")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "97"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "tests", "sanitize_run.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env)
    out = r.stdout + r.stderr
    assert "SANITIZE WORKLOAD DONE" in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    assert ("ERROR SUMMARY: 0 errors" in out or "(0 errors, 0 warnings)" in out), out[-4000:]


def test_racecheck_detects_missing_barriers():
    """Negative control: with the planned barriers stripped from the emitted
    mm kernel, racecheck must report hazards (so a clean run above means the
    barrier plan is what keeps the kernels race-free)."""
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, "--tool", "racecheck", "--error-exitcode", "97", sys.executable,
           os.path.join(ROOT, "tests", "sanitize_run.py"), "--broken"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert "BROKEN WORKLOAD DONE" in out, out[-4000:]
    assert r.returncode == 97, out[-4000:]
