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


def check_sass(lib: str) -> None:
    """Guard against a ptxas (12.9) mis-encoding seen when the tile engine is compiled out of line: the bulk
    reduction of the update's epilogue must be UBLKRED...ADD.F64.RN; with its address operands allocated in
    uniform registers >= UR32 it came out as ADD.U64 (integer adds into C).  Also require the FP64 tensor
    instruction to be present at all."""
    cuobjdump = os.path.join(os.path.dirname(NVCC), "cuobjdump")
    sass = subprocess.run([cuobjdump, "-sass", lib], capture_output=True, text=True).stdout
    red = [l for l in sass.splitlines() if "UBLKRED" in l]
    bad = [l.strip() for l in red if "ADD.F64.RN" not in l]
    if not red or bad or "DMMA.8x8x4" not in sass:
        raise RuntimeError(f"libmla_b200.so: unexpected SASS (bulk reductions: {len(red)}, not F64: {bad[:2]})")


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    flags = [f for f in FLAGS if f != "--use_fast_math=false"]
    # three translation units compiled in parallel: the operator kernels + C ABI, the persistent LU kernel
    # (alone, so nothing else can change its code generation) and its traced twin
    cmd = [NVCC, *flags, "--threads", "3", "-o", LIB, os.path.join(CSRC, "mla_b200.cu"),
           os.path.join(CSRC, "mla_getrf_prod.cu"), os.path.join(CSRC, "mla_getrf_traced.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed building libmla_b200.so")
    try:
        check_sass(LIB)
    except RuntimeError:
        os.replace(LIB, LIB + ".rejected")
        raise
    with open(os.path.join(HERE, "ptxas_report.txt"), "w") as f:
        # resource usage per kernel (registers, spills, shared memory); compile times left out so the
        # tracked file only changes when the code does
        f.write("".join(l for l in (res.stdout + res.stderr).splitlines(True) if "Compile time" not in l))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
