"""Build the in-tree CUDA library ``paper_1904_12754_b200/_lib/libexpmc_b200.so`` for sm_100a.

Plain nvcc (no torch JIT): the .so is built in-tree so it travels to the GPU box with the
gpurun snapshot.  ``python -m paper_1904_12754_b200.build`` or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libexpmc_b200.so")
SOURCES = ["kernels.cu", "context.cu", "driver.cpp", "gen.cpp", "io.cpp", "mc.cpp"]
HEADERS = ["internal.hpp", "walker.cuh", "ed_walker.cuh", "fem_walker.cuh", "fastmath.cuh", "log_table.inc"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-fopenmp", "-Xptxas", "-v", "-lgomp",
         "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [
        os.path.join(ROOT, "include", "expmc_b200.h"), os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile the library (to `out`, default the in-tree _lib/libexpmc_b200.so)."""
    lib = out or LIB
    if out is None and not force and not _stale():
        return LIB
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    # the image exports CC/CXX pointing at a gcc wrapper; nvcc's host compiler is explicit
    ccbin = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [NVCC, *ARCH, *FLAGS, "-ccbin", ccbin, "-shared", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *[f"-D{d}" for d in defines], *[os.path.join(CSRC, s) for s in SOURCES], "-ldl", "-o", lib + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = lib + ".build.log"
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(lib + ".tmp", lib)
    if verbose:
        sys.stdout.write(r.stderr)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
