"""Build libfvb.so in-tree with nvcc for sm_100a (FP64, no FMA contraction).

The library is the product's compute path; there is no fallback.  It is
built next to this file so that the snapshot gpurun ships (and the
driver's "which .so was loaded" check) sees it.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfvb.so")
SOURCES = ["setup.cpp", "meshio.cpp", "fvb_ops.cu", "fvb_solvers.cu", "fvb_team.cu", "fvb_api.cu"]
HEADERS = ["common.h", "fvb_internal.cuh", os.path.join("..", "..", "include", "fvb.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                      # numpy never fuses a*b+c
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-shared",
]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not stale():
        return LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    cmd = [NVCC, *FLAGS, "-o", LIB + ".tmp", *srcs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc build of libfvb.so failed")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
