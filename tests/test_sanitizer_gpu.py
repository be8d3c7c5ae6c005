"""compute-sanitizer over every kernel on tiny shapes (SURVEY §4 tier T1): memcheck (including
the guard-page tables), racecheck (shared-memory kernels: TMA bulk, bucket histograms, scans)
and synccheck. API error returns that the library handles are not reported."""
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
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    cmd = [cs, "--tool", tool, "--report-api-errors", "no",
           sys.executable, os.path.join(ROOT, "scripts", "sanitize_cases.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=850)
    out = p.stdout + p.stderr
    assert "SANITIZE-CASES-DONE bad=0" in out, out[-3000:]
    assert ("ERROR SUMMARY: 0 errors" in out or
            "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out), out[-3000:]
