"""compute-sanitizer over every kernel family (SURVEY.md §4.2 / §5 race detection).

memcheck (out-of-bounds and misaligned accesses), racecheck (shared-memory hazards
between the warp-specialised tail and DP warps, which hand buffers over through
named barriers) and synccheck (barrier misuse) on small solves of each variant in
tests/sanitize_driver.py, plus the NEXT-2 state/re-plan path and the NEXT-3
reassignment kernel; only the library's kernels are instrumented.
"""
import os
import re
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "3", "--kernel-name", "kns=ic_dp_kernel",
           "--kernel-name", "kns=reassign_kernel", "--kernel-name", "kns=ic_solo_kernel",
           sys.executable, os.path.join(ROOT, "tests", "sanitize_driver.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-4000:]
    if r.returncode == 86 and "closed" in tail:
        # the GPU pool's compute-sanitizer wrapper refuses to run (it has left GPUs needing a
        # reset); the same driver still runs un-instrumented in test_sanitize_driver_plain
        pytest.skip("compute-sanitizer closed on this GPU pool: " + tail.strip().splitlines()[0][:160])
    assert r.returncode == 0, f"{tool} exit {r.returncode}:\n{tail}"
    # memcheck/synccheck print "ERROR SUMMARY: 0 errors", racecheck "RACECHECK SUMMARY: 0 hazards ..."
    assert re.search(r"ERROR SUMMARY: 0 errors|RACECHECK SUMMARY: 0 hazards displayed \(0 errors, 0 warnings\)",
                     r.stdout + r.stderr), tail
    assert r.stdout.count("ok ") >= 10, tail


@pytest.mark.gpu
def test_sanitize_driver_plain():
    """The sanitizer's driver without instrumentation: every kernel family, both drop modes,
    the state/re-plan path and the reassignment kernel against the oracle."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_driver.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert r.stdout.count("ok ") >= 10, tail
