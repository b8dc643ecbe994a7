"""Build libgc.so in-tree (nvcc for sm_100a + g++ for the host encoder)."""
from __future__ import annotations

import fcntl
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

SOURCES_CU = ["gc_kernels.cu", "gc_encode_gpu.cu"]
SOURCES_CPP = ["gc_encoder.cpp"]
HEADERS = ["gc_codecs.cuh", "gc_device.cuh", "gc_decode.cuh", "gc_skip.cuh"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES_CU + SOURCES_CPP + HEADERS]
    deps.append(os.path.join(INC, "gc.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, lib: str = LIB, defines=()) -> str:
    """Build `lib` (default: the product libgc.so).  A build with `defines` (ablations,
    timing) must name its own output: it never replaces the product library.  Concurrent
    callers (one per bench rank) serialise on a file lock; objects go to per-process names."""
    if defines and os.path.abspath(lib) == os.path.abspath(LIB):
        raise ValueError("a -D build needs its own output (--out=...), not the product libgc.so")
    if not force and lib == LIB and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    with open(os.path.join(BUILD, ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and lib == LIB and not _stale():   # another process built it meanwhile
            return LIB
        return _build_locked(verbose, lib, defines)


def _build_locked(verbose: bool, lib: str, defines) -> str:
    objs = []
    tag = f".{os.getpid()}"
    for f in SOURCES_CU:
        o = os.path.join(BUILD, f + "".join(d.replace("=", "") for d in defines) + tag + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "186",
               *[f"-D{d}" for d in defines],
               "-Xptxas", "-v" if verbose else "-O3", "-I", INC, "-I", CSRC, "-c",
               os.path.join(CSRC, f), "-o", o]
        subprocess.check_call(cmd)
        objs.append(o)
    for f in SOURCES_CPP:
        o = os.path.join(BUILD, f + tag + ".o")
        cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-Wall", "-I", INC, "-c",
               os.path.join(CSRC, f), "-o", o]
        subprocess.check_call(cmd)
        objs.append(o)
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lpthread"])
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    out = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    if defs and not out:
        sys.exit("a -D build needs --out=PATH (the product libgc.so is never an ablation build)")
    print(build(force="--force" in sys.argv or bool(defs), verbose="-v" in sys.argv,
                lib=out[0] if out else LIB, defines=defs))
