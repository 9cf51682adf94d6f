"""Build libpd.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2605_06408_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpd.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-Wno-deprecated-declarations", "--expt-relaxed-constexpr",
         "-Xcudafe", "--diag_suppress=177"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + \
        [os.path.join(HERE, "..", "include", "pd.h")]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every csrc/*.cu for sm_100a and link libpd.so (or `out`, with extra -D defines)."""
    LIB_OUT = out or LIB
    if not force and os.path.exists(LIB_OUT):
        t = os.path.getmtime(LIB_OUT)
        if all(os.path.getmtime(d) <= t for d in deps()):
            return LIB_OUT
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(d.replace("=", "") for d in defines))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc()] + ARCH + FLAGS + ["-D" + d for d in defines] + ["-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        objs.append(obj)
    cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB_OUT + ".tmp"] + objs + ["-lcudart", "-ldl"]
    subprocess.check_call(cmd)
    os.replace(LIB_OUT + ".tmp", LIB_OUT)
    return LIB_OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
