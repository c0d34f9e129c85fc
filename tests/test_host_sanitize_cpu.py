"""Host planners under AddressSanitizer + UndefinedBehaviorSanitizer (CPU):
tests/cpp/host_sanitize.cpp drives plan.cpp / fwd_plan.cpp / shearlet_plan.cpp
(geometry resolution, fp64 ray tables, forward schedule with its self-check,
backprojection windows, ramp filters, shearlet plans) over fixed and random
geometries; any heap overflow, use-after-free, leak or UB aborts the run."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2009_14788_b200", "csrc")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


@pytest.mark.timeout(900)
def test_host_planners_asan_ubsan(tmp_path):
    if shutil.which("g++") is None or not os.path.exists(os.path.join(CUDA, "include", "cuda_runtime.h")):
        pytest.skip("g++ / CUDA headers not available")
    exe = str(tmp_path / "host_sanitize")
    cmd = ["g++", "-std=c++20", "-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=undefined",
           "-fno-omit-frame-pointer", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "tests", "cpp", "host_sanitize.cpp")]
    cmd += [os.path.join(CSRC, f) for f in ("plan.cpp", "fwd_plan.cpp", "plan_cache.cpp", "shearlet_plan.cpp")]
    cmd += ["-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lpthread", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    env = dict(os.environ, RK_VERIFY_PLAN="1", ASAN_OPTIONS="detect_leaks=1:abort_on_error=0",
               UBSAN_OPTIONS="print_stacktrace=1")
    r = subprocess.run([exe], env=env, capture_output=True, text=True, timeout=800)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "host planners clean" in r.stdout
    assert "runtime error" not in r.stderr, r.stderr[-4000:]
