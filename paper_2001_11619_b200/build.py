"""In-tree nvcc build of libskelb200.so (sm_100a).

The shared library travels with the repo snapshot to the GPU box; there is no
JIT path.  ``assemble.cu`` is compiled with ``-fmad=false`` so kernel entries
follow NumPy's per-operation rounding.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libskelb200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = {
    "assemble.cu": ["-fmad=false"],
    "gemm.cu": [],
    "qr.cu": [],
    "lu.cu": [],
    "misc.cu": [],
    "matvec.cu": [],
    "level.cu": [],
    "engine.cu": [],
}
# native host runtime (no CUDA): plain g++, no FP contraction (NumPy rounding)
HOST_SOURCES = {"host.cpp": []}
CXX = os.environ.get("CXX", "g++")
HOST_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-g"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
          "--expt-relaxed-constexpr", *os.environ.get("SKB_NVCC_EXTRA", "").split()]


def _stale(objs) -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "skelb200.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, s.replace(".cu", ".o")) for s in SOURCES]
    hobjs = [os.path.join(objdir, s.replace(".cpp", ".o")) for s in HOST_SOURCES]
    if not force and not _stale(objs):
        return LIB
    shared = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    shared += [os.path.join(HERE, "..", "include", "skelb200.h"), __file__]
    cmds = []
    for (src, extra), obj in zip(SOURCES.items(), objs):
        deps = [os.path.join(CSRC, src), *shared]
        if (force or not os.path.exists(obj)
                or any(os.path.getmtime(d) > os.path.getmtime(obj) for d in deps if os.path.exists(d))):
            cmds.append([NVCC, *ARCH, *COMMON, *extra, "-c", os.path.join(CSRC, src), "-o", obj])
    for (src, extra), obj in zip(HOST_SOURCES.items(), hobjs):
        deps = [os.path.join(CSRC, src), *shared]
        if (force or not os.path.exists(obj)
                or any(os.path.getmtime(d) > os.path.getmtime(obj) for d in deps if os.path.exists(d))):
            cmds.append([CXX, *HOST_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj])
    # translation units compile in parallel (qr.cu dominates)
    from concurrent.futures import ThreadPoolExecutor
    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        list(ex.map(run, cmds))
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, *hobjs, "-lcudart"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
