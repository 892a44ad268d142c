"""Build libcjm.so (the C-ABI CUDA library) in-tree with nvcc for sm_100a.

    python -m paper_1705_00103_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcjm.so")
SOURCES = [os.path.join(CSRC, f) for f in ("cjm.cu", "schedule.cpp", "pool.cpp", "mask_bounds.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("sweep.cuh", "sweep_v4.cuh", "resident.cuh", "mask.cuh", "internal.h")] + \
    [os.path.join(ROOT, "include", "cjm.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[str, str]:
    import nvidia  # torch's bundled NCCL (the one torch.distributed loads)
    base = os.path.join(list(nvidia.__path__)[0], "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: str | None = None) -> str:
    """Build the library; `defines`/`out` build a measurement variant (e.g.
    ("CJM_V4_RELEASE=2",)) at another path -- never the product library."""
    target = out or LIB
    if not force and os.path.exists(target) and \
            os.path.getmtime(target) >= max(os.path.getmtime(d) for d in DEPS):
        return target
    inc, lib = nccl_dirs()
    tmp = target + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared",
           "-Xcompiler", "-fPIC,-ffp-contract=off", "-fmad=false",
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", inc,
           *[f"-D{d}" for d in defines], *SOURCES, "-o", tmp,
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
