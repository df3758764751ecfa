"""Build libbingo.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libbingo.so")
TOOLS_SRC = [os.path.join(ROOT, "tools", "gather_bench.cu"), os.path.join(ROOT, "tools", "unit_kernels.cu")]
TOOLS_LIB = os.path.join(HERE, "libbingo_tools.so")
# in-process hardware counters for bench.py's roofline (CUPTI range profiler; measurement only)
METER_SRC = os.path.join(ROOT, "tools", "dram_meter.cpp")
METER_LIB = os.path.join(HERE, "libbingo_meter.so")
OBJDIR = os.path.join(ROOT, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(INCLUDE, "bingo.h"))
    return hs


def build(force: bool = False, verbose: bool = False, jobs: int = 8) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    hmax = max(os.path.getmtime(h) for h in headers())
    objs, procs = [], []
    for src in sources():
        obj = os.path.join(OBJDIR, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), hmax):
            cmd = [NVCC, *ARCH, *FLAGS, "-Xptxas", "-v", "-c", src, "-o", obj]
            procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
            if len(procs) >= jobs:
                _drain(procs, verbose)
    _drain(procs, verbose)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + f".{os.getpid()}.tmp"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    tmax = max(max(os.path.getmtime(t) for t in TOOLS_SRC), hmax)
    if force or not os.path.exists(TOOLS_LIB) or os.path.getmtime(TOOLS_LIB) < tmax:
        tmp = TOOLS_LIB + f".{os.getpid()}.tmp"
        subprocess.check_call([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                               "-I", INCLUDE, "-I", CSRC, "-o", tmp, *TOOLS_SRC, "-lcudart"])
        os.replace(tmp, TOOLS_LIB)
    if force or not os.path.exists(METER_LIB) or os.path.getmtime(METER_LIB) < os.path.getmtime(METER_SRC):
        tmp = METER_LIB + f".{os.getpid()}.tmp"
        cuda = os.path.dirname(os.path.dirname(NVCC))
        subprocess.check_call([NVCC, "-O2", "-std=c++17", "-Wno-deprecated-gpu-targets", "-Xcompiler", "-fPIC", "-shared",
                               "-I", os.path.join(cuda, "include"), "-o", tmp, METER_SRC,
                               "-L", os.path.join(cuda, "lib64"), "-lcupti", "-lnvperf_host", "-lcuda",
                               "-Xlinker", "-rpath=" + os.path.join(cuda, "lib64")])
        os.replace(tmp, METER_LIB)
    return LIB


def _drain(procs, verbose):
    while procs:
        cmd, p = procs.pop(0)
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        if verbose:
            sys.stderr.write(out)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
