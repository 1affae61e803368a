"""Build libdsssp.so (the C-ABI CUDA library) in-tree for sm_100a.

    python -m paper_1911_06895_b200.build

The shared library is plain nvcc output -- no torch extension machinery --
so any FFI (ctypes, cffi, cgo, JNI) can bind include/dsssp.h directly.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libdsssp.so")
# variant with the pull (vxm) relaxations compiled in (opt-in)
LIB_PULL = os.path.join(LIB_DIR, "libdsssp_pull.so")
VARIANTS = {LIB: [], LIB_PULL: ["-DDS_PULL_LIGHT=1", "-DDS_PULL_HEAVY=1"]}
SOURCES = ["dsssp.cu", "gen.cu", "shard.cu", "ingest.cpp"]
HEADERS = ["common.cuh", "sssp_kernel.cuh"]

NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
    "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libdsssp.so")


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(REPO, "include", "dsssp.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIB_DIR, exist_ok=True)
    only_main = os.environ.get("DS_BUILD_MAIN_ONLY") == "1"  # quick iteration builds
    for lib, extra in VARIANTS.items():
        if only_main and lib != LIB:
            continue
        if not force and not _stale(lib):
            continue
        tmp = lib + ".tmp"
        cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES]]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(tmp, lib)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
