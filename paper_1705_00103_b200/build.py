"""Build libcjm.so (the C-ABI CUDA library) in-tree with nvcc for sm_100a.

    python -m paper_1705_00103_b200.build
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcjm.so")
SOURCES = [os.path.join(CSRC, f) for f in (
    "cjm.cu", "kernels_v3.cu", "kernels_v4_5.cu", "kernels_v4_9.cu", "kernels_v4_17.cu",
    "schedule.cpp", "pool.cpp", "mask_bounds.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in (
    "sweep.cuh", "sweep_v4.cuh", "kernels.h", "kernels_v4.cuh", "resident.cuh", "mask.cuh",
    "internal.h")] + [os.path.join(ROOT, "include", "cjm.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
PTXAS_OPT = "-O3"
# ptxas -O1 for the warp-tiled sweep kernels: its less aggressive scheduling
# keeps the rotating register rings in place (steady 9-point period 14.5 vs
# 16.4 instructions per update, 3x fewer register moves, no spills; 17-point
# 245 registers, no spills) and measured 22.1 vs 22.8 us per sweep at 4096^2,
# 278 vs 280 at 16384^2, equal for the 17-point (profiles/r02_kernel_ab.jsonl)
PTXAS_PER_SOURCE = {"kernels_v4_5.cu": "-O1", "kernels_v4_9.cu": "-O1", "kernels_v4_17.cu": "-O1"}


def nccl_dirs() -> tuple[str, str]:
    import nvidia  # torch's bundled NCCL (the one torch.distributed loads)
    base = os.path.join(list(nvidia.__path__)[0], "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: str | None = None,
          src: str | None = None, ptxas: str = PTXAS_OPT) -> str:
    """Build the library; `defines` / `out` / `src` (a patched copy of csrc/)
    build a measurement variant at another path -- never the product library."""
    target = out or LIB
    if (defines or src or ptxas != PTXAS_OPT) and not out:
        raise ValueError("measurement builds need their own output path")
    if not force and os.path.exists(target) and \
            os.path.getmtime(target) >= max(os.path.getmtime(d) for d in DEPS):
        return target
    sources = [os.path.join(src, os.path.basename(f)) for f in SOURCES] if src else SOURCES
    inc, lib = nccl_dirs()
    tmp = target + f".tmp{os.getpid()}"
    objdir = tempfile.mkdtemp(prefix="cjm_build_")
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-ffp-contract=off", "-fmad=false",
              "-Xptxas", "__PTXAS__",
              "-I", os.path.join(ROOT, "include"), "-I", inc, *[f"-D{d}" for d in defines]]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        opt = PTXAS_PER_SOURCE.get(os.path.basename(src), ptxas) if ptxas == PTXAS_OPT else ptxas
        cmd = [opt + (",-v" if verbose else "") if c == "__PTXAS__" else c for c in common]
        r = subprocess.run([*cmd, "-c", src, "-o", obj], capture_output=True, text=True)
        return src, obj, r

    try:
        # one nvcc per translation unit, in parallel (the sweep-kernel
        # instantiations are spread over kernels_*.cu)
        with ThreadPoolExecutor(max_workers=len(sources)) as ex:
            results = list(ex.map(compile_one, sources))
        for src, _, r in results:
            if verbose or r.returncode:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode:
                raise subprocess.CalledProcessError(r.returncode, f"nvcc -c {src}")
        subprocess.check_call([nvcc(), *ARCH, "-shared", *[o for _, o, _ in results], "-o", tmp,
                               "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"])
    finally:
        shutil.rmtree(objdir, ignore_errors=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
