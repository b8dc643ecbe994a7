"""Build libgc.so in-tree (nvcc for sm_100a + g++ for the host encoder)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libgc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES_CU = ["gc_kernels.cu"]
SOURCES_CPP = ["gc_encoder.cpp"]
HEADERS = ["gc_codecs.cuh", "gc_device.cuh"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES_CU + SOURCES_CPP + HEADERS]
    deps.append(os.path.join(INC, "gc.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for f in SOURCES_CU:
        o = os.path.join(BUILD, f + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v" if verbose else "-O3", "-I", INC, "-I", CSRC, "-c",
               os.path.join(CSRC, f), "-o", o]
        subprocess.check_call(cmd)
        objs.append(o)
    for f in SOURCES_CPP:
        o = os.path.join(BUILD, f + ".o")
        cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-Wall", "-I", INC, "-c",
               os.path.join(CSRC, f), "-o", o]
        subprocess.check_call(cmd)
        objs.append(o)
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lpthread"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
