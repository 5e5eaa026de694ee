"""compute-sanitizer over the step kernels: memcheck, racecheck and synccheck on c1
and c1-evict (tools/sanitize_case.py: both call paths, flat and hierarchical index)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(tool):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99",
           sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "sanitize case ok" in r.stdout, tail
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr or "RACECHECK SUMMARY: 0 hazards" in r.stdout + r.stderr, tail
