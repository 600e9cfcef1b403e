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
SOURCES = ["setup.cpp", "meshio.cpp", "fvb_ops.cu", "fvb_cg.cu", "fvb_bicgstab.cu", "fvb_team.cu", "fvb_api.cu"]
HEADERS = ["common.h", "fvb_internal.cuh", "fvb_solvers_common.cuh", os.path.join("..", "..", "include", "fvb.h")]

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


def _compile(src, obj):
    flags = [f for f in FLAGS if f != "-shared"]
    cmd = [NVCC, *flags, "-c", "-o", obj, src]
    return subprocess.run(cmd, capture_output=True, text=True)


def build(force=False, verbose=False):
    """Compile every source to an object in parallel (the solver unit with
    its kernel instantiations is the long pole), then link libfvb.so."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in srcs]
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        results = list(ex.map(_compile, srcs, objs))
    for src, res in zip(srcs, results):
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc build of {os.path.basename(src)} failed")
        if verbose:
            sys.stderr.write(res.stderr)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp", *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link of libfvb.so failed")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
