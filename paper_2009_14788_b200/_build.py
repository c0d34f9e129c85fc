"""In-tree build of the CUDA extension (sm_100a) and of the oracle checkers.

``build_library()`` compiles ``csrc/*.cu`` + ``csrc/*.cpp`` with nvcc into
``paper_2009_14788_b200/libradon_b200.so`` (the C-ABI library declared in
``include/radon_b200.h``).  nvcc cross-compiles for sm_100a without a GPU.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libradon_b200.so")
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def build_library(verbose: bool = False, force: bool = False) -> str:
    srcs = sources()
    deps = srcs + glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(d) for d in deps):
        return LIB
    tmp = LIB + ".tmp"
    cmd = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off",
           "-I", INCLUDE, "-I", CSRC, "--threads", "0", "-o", tmp, *srcs]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


def build_oracles(verbose: bool = False) -> None:
    """Checkers only (oracle/Makefile): the C restatement always; the reference
    compiled in place only where /root/reference exists (this container)."""
    make = shutil.which("make") or "make"
    odir = os.path.join(ROOT, "oracle")
    subprocess.run([make, "-s", "-C", odir, "port"], check=True)
    if os.path.isdir("/root/reference/proj/core/src"):
        subprocess.run([make, "-s", "-C", odir, "ref"], check=True)
        # the reference's own program over the B200 projector
        subprocess.run([make, "-s", "-j8", "-C", os.path.join(ROOT, "integration")], check=True)


if __name__ == "__main__":
    build_library(verbose="-v" in sys.argv, force="-f" in sys.argv)
    build_oracles()
    print(LIB)
