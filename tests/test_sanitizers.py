"""compute-sanitizer over small runs of every kernel (VERDICT r1
#9): memcheck (out-of-bounds / misaligned global and shared accesses — K1s
reads a window's negatives as a fixed-size group into a zeroed pad past the
batch end), racecheck (shared-memory hazards: the staged sample rows, the g
exchange, the d=512 two-warp dot exchange), synccheck (barrier use) and
initcheck (reads of uninitialised device memory)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for p in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if p and os.path.exists(p):
            return p
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool,extra", [("memcheck", ["--leak-check", "no"]),
                                        ("racecheck", ["--racecheck-report", "hazard"]),
                                        ("synccheck", []),
                                        ("initcheck", [])])
def test_sanitizer_clean(tool, extra):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "97", "--print-limit", "20", *extra,
           sys.executable, os.path.join(ROOT, "tools", "sanitize_probe.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    print(out[-3000:])
    assert r.returncode == 0, out[-6000:]
    assert "sanitize probe ok" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-3000:]
