"""Builds libmla_b200.so in-tree with nvcc for sm_100a (no other architecture, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmla_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# -cudart shared: the library uses the process's libcudart.so.12 (the one torch has already loaded, or the
# toolkit's through the rpath) instead of embedding a private copy of the whole runtime.
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17", "-shared",
         "-cudart", "shared", "-Xlinker", "-rpath=/usr/local/cuda/lib64",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--use_fast_math=false"]


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))] + \
        [os.path.join(os.path.dirname(HERE), "include", "mla_b200.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    flags = [f for f in FLAGS if f != "--use_fast_math=false"]
    cmd = [NVCC, *flags, "-o", LIB, os.path.join(CSRC, "mla_b200.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed building libmla_b200.so")
    with open(os.path.join(HERE, "ptxas_report.txt"), "w") as f:
        # resource usage per kernel (registers, spills, shared memory); compile times left out so the
        # tracked file only changes when the code does
        f.write("".join(l for l in (res.stdout + res.stderr).splitlines(True) if "Compile time" not in l))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
