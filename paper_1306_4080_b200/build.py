"""Build libpcdn.so in-tree for sm_100a (nvcc -gencode arch=compute_100a,code=sm_100a)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "pcdn_api.cu")]
DEPS = SRC + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "pcdn.h"), __file__]
LIB = os.path.join(HERE, "libpcdn.so")
# the same library with the sparse kernel's profiling instrumentation (-DPCDN_PROFILE=1), for the
# profiling scripts (loaded through PCDN_LIB); never the product path
LIB_PROF = os.path.join(HERE, "libpcdn_prof.so")
# ... and with device-side bounds / protocol checks (-DPCDN_CHECKS=1): the GPU tests run against it
# (scripts/checked_run.sh) in place of compute-sanitizer, which is closed on this pool
LIB_CHECKED = os.path.join(HERE, "libpcdn_checked.so")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false",          # no FMA contraction: same op sequence as the written formulas
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False, profile: bool = False, checks: bool = False) -> str:
    lib = LIB_CHECKED if checks else LIB_PROF if profile else LIB
    stale = force or not os.path.exists(lib) or any(os.path.getmtime(d) > os.path.getmtime(lib) for d in DEPS)
    if stale:
        tmp = lib + f".tmp{os.getpid()}"
        cmd = [nvcc()] + NVCC_FLAGS + (["-DPCDN_PROFILE=1"] if profile else []) + (["-DPCDN_CHECKS=1"] if checks else []) + \
              (["-Xptxas", "-v"] if verbose else []) + ["-o", tmp] + SRC
        subprocess.check_call(cmd)
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, profile="--profile" in sys.argv,
                checks="--checks" in sys.argv))
