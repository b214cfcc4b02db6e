"""Builds liblinoct_b200.so in-tree for sm_100a (nvcc -> objects -> one shared library).

No JIT cache: the .so lands next to this file so it travels with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# LO_BUILD_DIR / LO_NVCC_EXTRA: side builds of tuning variants (objects + library elsewhere)
OBJ = os.path.join(os.environ.get("LO_BUILD_DIR", HERE), "_build")
LIB = os.path.join(os.environ.get("LO_BUILD_DIR", HERE), "liblinoct_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CUDA_SOURCES = ["context.cu", "reorder.cu", "octree.cu", "radius.cu", "radius_struct.cu", "knn.cu", "io.cu", "centres.cu", "comm.cu"]
CXX_SOURCES = ["gen.cpp"]

# -fmad=false: no DFMA contraction anywhere, the FP64 predicates must be the reference's
# exact expression trees.  -ffp-contract=off for the host side (generators, Discretizer).
NVCC_FLAGS = [
    "-std=c++20", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
    "-fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
] + os.environ.get("LO_NVCC_EXTRA", "").split()


def _stale(src: str, obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src, *deps])


def _compile(src: str) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "linoct_b200.h"))
    if not _stale(path, obj, deps):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC, *NVCC_FLAGS, "-c", path, "-o", obj]
    else:
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = CUDA_SOURCES + CXX_SOURCES
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(_compile, srcs))
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB, *objs,
               "-Xlinker", "-z,defs", "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose=True)
