"""Build the in-tree CUDA library libdmsgm.so for sm_100a (nvcc, no torch extension).

    python -m paper_1702_05156_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB_PATH = os.path.join(PKG, "libdmsgm.so")
SOURCES = [os.path.join(CSRC, "dmsgm.cu"), os.path.join(CSRC, "dmsgm_klt.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
    [os.path.join(INCLUDE, "dmsgm.h"), os.path.join(INCLUDE, "dmsgm_klt.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",              # no FMA contraction: bitwise parity with the oracle
    "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-shared",
    "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False, out: str = LIB_PATH, defines=()) -> str:
    """Build libdmsgm.so (or, with `out` / `defines`, a variant for A/B timing)."""
    newest = max(os.path.getmtime(p) for p in DEPS)
    if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-I", CSRC, "-o", tmp, *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else LIB_PATH
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args or out != LIB_PATH, verbose="--verbose" in args, out=out, defines=defs))
