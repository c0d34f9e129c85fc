"""compute-sanitizer over every kernel family at tiny sizes (race
detection and memory checking on small configurations).  memcheck catches
out-of-bounds / misaligned accesses (the TMA boxes, the cp.async windows, the
swizzled FFT slots); racecheck shared-memory hazards between the staging and
the marching / accumulation phases; synccheck barrier misuse.  Where the GPU pool refuses compute-sanitizer,
these skip and tests/test_guardband_gpu.py (guard-band sentinels around every
device entry point's input and output) covers out-of-bounds access."""
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
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "17", sys.executable,
           os.path.join(ROOT, "tools", "sanitize_probe.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    out = r.stdout + r.stderr
    if "sanitize probe done" not in out and "compute-sanitizer is closed" in out:
        # the GPU pool refuses compute-sanitizer runs (its wrapper prints this and runs nothing);
        # tests/test_guardband_gpu.py checks out-of-bounds reads and writes without it
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert "sanitize probe done" in out, out[-3000:]
    clean = "ERROR SUMMARY: 0 errors" in out or "SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out
    assert r.returncode == 0 and clean, out[-3000:]
