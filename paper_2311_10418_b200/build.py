"""In-tree build of the B200 planner library (no JIT cache, no pip install).

Produces ``paper_2311_10418_b200/libpipeplan_b200.so`` containing
  * the sm_100a kernels and the C-ABI (csrc/*.cu, include/pipeplan_b200.h)
  * the drop-in C++ API of the reference planner (csrc/host/*.cpp,
    include/pipeplan/*.h)
Everything is compiled for ``-gencode arch=compute_100a,code=sm_100a`` with
``--fmad=false`` (and ``-ffp-contract=off`` on the host) because the planner
must be bit-exact with the FP64 reference.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libpipeplan_b200.so")
# Development variant: PP_TRACE=1 builds build/trace/libpipeplan_b200_trace.so
# with clock64 stamps in the DP kernel (tools/dp_trace.py); never shipped.
TRACE = os.environ.get("PP_TRACE") == "1"
if TRACE:
    BUILD = os.path.join(ROOT, "build", "trace")
    LIB = os.path.join(BUILD, "libpipeplan_b200_trace.so")

CU = ["sort.cu", "cost.cu", "dp.cu", "dp_coop.cu", "opcost.cu", "sched.cu", "ingest.cu", "report.cu", "slots.cu", "gtab.cu", "capi.cu", "calib.cu"]
CPP = ["host/workload.cpp", "host/cost_model.cpp", "host/microbatch.cpp", "host/order_search.cpp", "host/padding_report.cpp", "host/capi_host.cpp", "host/plan_file.cpp", "host/epoch.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++17", "-O3", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
           "-I" + INC] + ARCH + (["-DPP_DP_TRACE"] if TRACE else [])
CXXFLAGS = ["-std=c++20", "-O3", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall", "-Wextra",
            "-I" + INC, "-I/usr/local/cuda/include"]


def _headers():
    out = []
    for d in (CSRC, INC, os.path.join(INC, "pipeplan")):
        for f in os.listdir(d):
            if f.endswith((".h", ".cuh")):
                out.append(os.path.join(d, f))
    return out


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd[:3]) + " ...")
    return r


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = _headers()
    objs = []
    for f in CU:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f.replace("/", "_") + ".o")
        if force or _stale(obj, [src] + hdrs):
            _run([NVCC] + NVFLAGS + ["-c", src, "-o", obj], verbose)
        objs.append(obj)
    for f in CPP:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f.replace("/", "_") + ".o")
        if force or _stale(obj, [src] + hdrs):
            _run([CXX] + CXXFLAGS + ["-c", src, "-o", obj], verbose)
        objs.append(obj)
    if force or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"], verbose)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
    print(LIB)
