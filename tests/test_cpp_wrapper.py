"""The C++ drop-in layer (include/radonkit_b200.hpp) compiles against the C ABI
and links the in-tree library; on a GPU the demo's checks pass."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2009_14788_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "wrapper_demo.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "wrapper_demo")


def build():
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-L", PKG, "-lradon_b200",
           f"-Wl,-rpath,{PKG}", "-o", BIN]
    subprocess.run(cmd, check=True)
    return BIN


def test_cpp_wrapper_builds_and_validates_on_cpu(rk):
    exe = build()
    out = subprocess.run([exe, "--validate-only"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") == 4


@pytest.mark.gpu
def test_cpp_wrapper_runs_on_gpu(rk, cuda):
    exe = build()
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "FAIL" not in out.stdout
