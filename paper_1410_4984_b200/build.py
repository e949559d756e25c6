"""In-tree build of libsgpx.so for sm_100a (nvcc; no JIT cache, the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsgpx.so")
SOURCES = [os.path.join(CSRC, f) for f in ("psi_kernels.cu", "psi_direct.cu", "psi1_kernels.cu", "psi1_tile.cu", "psi1_tc.cu", "psi_rowtile.cu", "sgpx_api.cu",
                                            "synth.cu", "dla.cu", "dcoord.cu", "fit.cu", "syrk.cu",
                                            "coordinator.cpp")]
HEADERS = [os.path.join(CSRC, f) for f in ("fp16_pieces.cuh", "psi_kernels.cuh", "psi_common.cuh", "tc_util.cuh", "coordinator.hpp", "dla.cuh", "dcoord.cuh")] + [
    os.path.join(ROOT, "include", "sgpx.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_LIB = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs, cmds = [], []
    for src in SOURCES:
        obj = os.path.join(CSRC, os.path.basename(src) + ".o")
        cmd = [NVCC, "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-O3,-march=x86-64-v3", "-x",
               "cu" if src.endswith(".cu") else "c++", "-c", src, "-o", obj]
        cmd[1:1] = os.environ.get("SGPX_NVCC_DEFS", "").split()  # experiment builds (-DNAME=value)
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        cmds.append(cmd)
        objs.append(obj)
    # one nvcc per translation unit, in parallel (the row-tile unit dominates the build time)
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        list(ex.map(subprocess.check_call, cmds))
    # cuBLAS (the SYRK path's plain GEMMs): libcublas.so.12 of this CUDA install, or the one torch has loaded
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-L" + CUDA_LIB, "-lcublas",
                           "-Xlinker", "-rpath=" + CUDA_LIB])
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
