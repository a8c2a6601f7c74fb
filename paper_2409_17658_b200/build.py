"""Builds librd.so in-tree for sm_100a (nvcc + g++), so the library travels with the repo
snapshot to the GPU box.  Run: python -m paper_2409_17658_b200.build"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "librd.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES = ["rd_host.cpp", "rd_cuda.cu"]
HEADERS = ["rd_internal.h", os.path.join(INCLUDE, "rd.h")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    bdir = os.path.join(PKG, "build")
    os.makedirs(bdir, exist_ok=True)
    host_o = os.path.join(bdir, "rd_host.o")
    cuda_o = os.path.join(bdir, "rd_cuda.o")
    cmds = [
        ["g++", "-O2", "-std=c++17", "-fPIC", "-fopenmp", "-Wall", "-I", INCLUDE, "-c",
         os.path.join(CSRC, "rd_host.cpp"), "-o", host_o],
        [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp", "-Xptxas", "-v",
         "-I", INCLUDE, "-c", os.path.join(CSRC, "rd_cuda.cu"), "-o", cuda_o],
        [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", host_o, cuda_o, "-o", LIB + ".tmp",
         "-lgomp", "-lpthread"],
    ]
    for c in cmds:
        r = subprocess.run(c, capture_output=True, text=True)
        if verbose or r.returncode != 0:
            sys.stderr.write(" ".join(c) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(c[:2])}")
        if "ptxas" in " ".join(r.stderr.splitlines()[:0]) or (c[0] == NVCC and "-c" in c):
            with open(os.path.join(bdir, "ptxas.log"), "w") as f:
                f.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
