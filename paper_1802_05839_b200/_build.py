"""In-tree build of libhftw.so (nvcc, sm_100a).  No JIT cache: the built .so
lives next to this file so it travels to the GPU box with the snapshot."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhftw.so")
SOURCES = [os.path.join(CSRC, "hftw.cu")]
DEPS = SOURCES + sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")) + [
    os.path.join(ROOT, "include", "hftw.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    # bitwise parity with the reference's -ffp-contract=off build
    # (proj/CMakeLists.txt:14-16): no FMA contraction on device or host
    "--fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-shared", "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libhftw.so if missing or out of date; returns its path."""
    if not force and not stale():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-Xptxas", "-v", "-o", LIB, *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "build_ptxas.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")
    if verbose:
        print(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
