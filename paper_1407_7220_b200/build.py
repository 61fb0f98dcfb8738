"""Builds libcvxreg_b200.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_1407_7220_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "cvxreg_b200")
LIB = os.path.join(PKG, "libcvxreg_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     *os.environ.get("CRB_NVCC_EXTRA", "").split(),
                     "-Xcompiler", "-ffp-contract=off", "-I" + os.path.join(ROOT, "include")]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
             "-I" + os.path.join(ROOT, "include")]
CU_SOURCES = ["sweep_mma.cu", "kernels.cu", "small.cu", "power.cu", "metrics.cu", "capi.cu",
              "alcc.cu", "general.cu", "balcc.cu"]
CXX_SOURCES = ["host.cpp"]
HEADERS = ["device.cuh", "kernels.cuh", "host.hpp", "pipeline.cuh", "iteration.cuh", "small.cuh",
           "handle.cuh", "balcc.cuh", "mma_geo.cuh"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _cxx():
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "cvxreg_b200.h")]
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([_nvcc(), *NVCC_FLAGS, "-c", s, "-o", o])
    for src in CXX_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([_cxx(), *CXX_FLAGS, "-c", s, "-o", o])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r

    with cf.ThreadPoolExecutor(max_workers=4) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(LIB, objs):
        run([_nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lnccl", "-lcudart_static", "-lrt",
             "-lpthread", "-ldl"])
    # C++ drop-in demo (include/cvxreg_b200/papg.hpp over the C ABI), used by the GPU tests
    demo_src = os.path.join(ROOT, "tests", "cpp", "dropin_demo.cpp")
    demo = os.path.join(PKG, "cxx_dropin_demo")
    hpp = os.path.join(ROOT, "include", "cvxreg_b200", "papg.hpp")
    if os.path.exists(demo_src) and (force or _stale(demo, [demo_src, hpp, LIB])):
        run([_cxx(), "-O2", "-std=c++17", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
             demo_src, "-o", demo, "-L" + PKG, "-lcvxreg_b200", "-Wl,-rpath,$ORIGIN"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
