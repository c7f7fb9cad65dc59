"""Build the native library in-tree with nvcc for sm_100a (no JIT, no torch extension).

Output: paper_2104_08571_b200/libripple_fv.so (git-ignored; travels to the GPU box
with the gpurun snapshot).  Flags:
  -gencode arch=compute_100a,code=sm_100a   B200 only
  -fmad=false    no implicit FMA contraction: every fma() in scheme.cuh is explicit,
                 so all kernels (split / fused, any partitioning) are bitwise identical
  -lineinfo      ncu source view
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libripple_fv.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")) +
                  glob.glob(os.path.join(HERE, "csrc", "*.cpp")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(HERE, "csrc", "*.h*")) +
                              glob.glob(os.path.join(HERE, "csrc", "*.cuh")) +
                              [os.path.join(ROOT, "include", "ripple_fv.h"), __file__])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, "-shared", "-Xcompiler", "-fPIC", "-O3", "-std=c++17", "-lineinfo",
           "-fmad=false", *ARCH, "-I", os.path.join(ROOT, "include"),
           "-Xptxas", "-v" if verbose else "-O3",
           "-o", tmp, *sources(), "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
