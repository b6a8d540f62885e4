"""Build libvtgs.so (the sm_100a kernels + C ABI) in-tree with nvcc.

`python -m paper_2506_02741_b200.build` or `__graft_entry__.build()`.  The library links the
CUDA runtime statically, so it loads (and reports VTGS_ERR_NO_DEVICE) on a machine without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["instantiate.cu", "forward.cu", "composite_fwd.cu", "backward.cu", "ssim.cu", "abi.cu", "peaks.cu"]
HEADERS = ["vtgs_internal.cuh", "composite_common.cuh"]
LIB = os.path.join(HERE, "libvtgs.so")
LIB_CHECKED = os.path.join(HERE, "libvtgs_checked.so")   # -DVTGS_CHECKED: in-kernel bounds / invariant checks
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared",
         "-cudart", "static", "-Xptxas", "-warn-spills"]


def _inputs():
    return ([os.path.join(CSRC, s) for s in SOURCES + HEADERS]
            + [os.path.join(ROOT, "include", "vtgs.h"), os.path.abspath(__file__)])


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in _inputs())


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    lib = LIB_CHECKED if checked else LIB
    if not force and not stale(lib):
        return lib
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, *FLAGS, *(["-DVTGS_CHECKED"] if checked else []),
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", tmp]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
