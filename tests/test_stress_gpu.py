"""Randomised parity sweeps as regression tests (fixed seeds, a few seconds each):
tools/stress_parity.py (projector / FBP over random geometries, batch sizes, storage
dtypes, steps, device and host paths) and tools/stress_solvers.py (estimate_alpha,
Landweber, CGNE, shearlets on any square grid, ADMM) against the reference, extreme
geometries (tools/stress_extreme.py) and concurrent callers across plan-cache evictions
(tools/stress_concurrency.py, bitwise against serial).  The sweeps
found the r2 geometry gaps."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool,args", [("stress_parity.py", ["250", "31", "300"]),
                                       ("stress_parity.py", ["250", "32", "520"]),
                                       ("stress_solvers.py", ["16", "33"]),
                                       ("stress_extreme.py", ["8", "34"]),
                                       ("stress_concurrency.py", ["8", "25", "35"])])
def test_randomised_sweep(tool, args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", tool), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
