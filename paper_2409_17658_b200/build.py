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

CUDA_UNITS = ["rd_cuda.cu", "rd_gemm_pm_stats.cu", "rd_gemm_pm_stats_tma.cu", "rd_gemm_pm_part.cu",
              "rd_gemm_row_rp.cu", "rd_gemm32.cu", "rd_gemm_pm_sk.cu", "rd_small.cu",
              "rd_gemm_pm64.cu"]
SOURCES = ["rd_host.cpp"] + CUDA_UNITS
HEADERS = ["rd_internal.h", "rd_gemm.cuh", "rd_gemm_kernels.cuh", os.path.join(INCLUDE, "rd.h")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compiles the host unit and the CUDA units in parallel (the GEMM instances live in
    separate units), then links librd.so; ptxas -v output goes to build/ptxas.log."""
    from concurrent.futures import ThreadPoolExecutor
    if not force and not _stale():
        return LIB
    bdir = os.path.join(PKG, "build")
    os.makedirs(bdir, exist_ok=True)
    objs = [os.path.join(bdir, os.path.splitext(u)[0] + ".o") for u in SOURCES]
    cmds = [["g++", "-O2", "-std=c++17", "-fPIC", "-fopenmp", "-Wall", "-I", INCLUDE, "-c",
             os.path.join(CSRC, "rd_host.cpp"), "-o", objs[0]]]
    for u, o in zip(CUDA_UNITS, objs[1:]):
        cmds.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp", "-Xptxas", "-v",
                     "-I", INCLUDE, "-c", os.path.join(CSRC, u), "-o", o])

    def run(c):
        return c, subprocess.run(c, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 4)) as ex:
        results = list(ex.map(run, cmds))
    log = []
    for c, r in results:
        if verbose or r.returncode != 0:
            sys.stderr.write(" ".join(c) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(c[:2])} {c[-3]}")
        if c[0] == NVCC:
            log.append(f"==== {c[-3]}\n" + r.stderr)
    with open(os.path.join(bdir, "ptxas.log"), "w") as f:
        f.write("".join(log))
    link = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", LIB + ".tmp", "-lgomp", "-lpthread"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(link) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
