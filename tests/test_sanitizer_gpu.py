"""compute-sanitizer over every kernel on tiny shapes (SURVEY §4 tier T1): memcheck (including
the guard-page tables), racecheck (shared-memory kernels: TMA bulk, bucket histograms, scans)
and synccheck. API error returns that the library handles are not reported.

Opt-in (UT_SANITIZE=1): the GPU pool closed compute-sanitizer late in round 2 (runs under it had
left GPUs needing a reset, the pool's stub now refuses to start), so the round-end GPU suite does
not run it. Its last green runs at HEAD's kernels are in profiles/r2/r2pos/. The same cases run
without the sanitizer, against the oracle and with guard pages, in the other GPU tests."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(900)
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if os.environ.get("UT_SANITIZE") != "1":
        pytest.skip("opt-in (UT_SANITIZE=1): compute-sanitizer is closed on this GPU pool")
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    cmd = [cs, "--tool", tool, "--report-api-errors", "no",
           sys.executable, os.path.join(ROOT, "scripts", "sanitize_cases.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=850)
    out = p.stdout + p.stderr
    if "compute-sanitizer is closed" in out:
        pytest.skip(out.strip().splitlines()[0])
    assert "SANITIZE-CASES-DONE bad=0" in out, out[-3000:]
    assert ("ERROR SUMMARY: 0 errors" in out or
            "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out), out[-3000:]
