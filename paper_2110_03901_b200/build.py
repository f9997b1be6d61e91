"""Build the sm_100a extension in-tree: paper_2110_03901_b200/libimconv.so.

Plain nvcc (no torch JIT cache): the shared object lives next to the package
so it travels to the GPU box with the repo snapshot.  cudart is linked
statically and libcuda is resolved at run time through
cudaGetDriverEntryPoint, so the library loads (and exports every symbol of
include/imconv.h) on a machine without a GPU.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libimconv.so")
LIB_INSTR = os.path.join(PKG, "libimconv_instr.so")  # same sources, -DIMCONV_INSTRUMENT=1 (tools only)
LIB_DEBUG = os.path.join(PKG, "libimconv_debug.so")  # same sources, -DIMCONV_DEBUG=1: invariant checks
SOURCES = [os.path.join(CSRC, f) for f in ("imconv_api.cu", "lru.cpp")]
# every header the sources can include: a stale .so must never survive an edit to one of them
HEADERS = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) + [
    os.path.join(ROOT, "include", "imconv.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-cudart", "static"]


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, instrument: bool = False, debug: bool = False) -> str:
    lib = LIB_INSTR if instrument else LIB_DEBUG if debug else LIB
    if not force and not _stale(lib):
        return lib
    cmd = [NVCC] + ARCH + FLAGS + ["-I", os.path.join(ROOT, "include"), "-shared", "-o", lib] + SOURCES
    if instrument:
        cmd.insert(1, "-DIMCONV_INSTRUMENT=1")
    if debug:
        cmd.insert(1, "-DIMCONV_DEBUG=1")
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv, instrument="--instrument" in sys.argv,
                debug="--debug" in sys.argv))
