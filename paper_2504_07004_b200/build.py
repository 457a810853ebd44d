"""Build libcypress_b200.so in-tree with nvcc for sm_100a (no torch involved)."""
from __future__ import annotations

import glob
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
CSRC = os.path.join(_HERE, "csrc")
OUT = os.path.join(_HERE, "libcypress_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-I" + os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(ROOT, "include", "cypress_b200.h")])


def build(force: bool = False, verbose: bool = False, defines=(), out: str = OUT) -> str:
    """Compile the product library (no ``defines``) or, for timing experiments only, a separate
    library at ``out`` with extra ``-D`` switches (scripts/build_experiment.py).  The product
    library never carries experiment switches."""
    if defines and out == OUT:
        raise ValueError("experiment switches must go to a separate library, not the product .so")
    stale = force or not os.path.exists(out) or any(os.path.getmtime(s) > os.path.getmtime(out) for s in sources())
    if stale:
        tmp = out + f".tmp{os.getpid()}"
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], os.path.join(CSRC, "cy_gemm.cu"),
               os.path.join(CSRC, "cy_attention.cu"), os.path.join(CSRC, "cy_comm.cu"), "-o", tmp]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
