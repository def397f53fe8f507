"""In-tree build of libvmsplat_b200.so (sm_100a) with nvcc.

Exactness-critical translation units (visibility raster and FP64
preprocessing) are compiled with ``-fmad=false`` so the compiler never fuses a
multiply-add the reference evaluates as two roundings; the blend, sort and ABI
units keep contraction on.  The built library lands next to this file (it is
git-ignored but travels to the GPU box with the gpurun snapshot).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvmsplat_b200.so")
BUILD = os.path.join(HERE, "csrc", "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
UNITS = {
    "vis.cu": ["-fmad=false"],
    "preprocess.cu": ["-fmad=false"],
    "prims.cu": [],
    "blend.cu": [],
    "abi.cu": [],
    "session.cu": [],
    "bvh.cu": ["-fmad=false"],
    "lod.cu": ["-fmad=false"],
    "dpt.cu": [],
}
HOST_UNITS = {"pagetable.cpp": ["-O2", "-std=c++17", "-fPIC"]}
HEADERS = ["common.cuh", "prims.h", "render.h", "vis.h"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA extension cannot be built")


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src, os.path.join(HERE, "..", "include", "vmsplat_b200.h")]
    deps += [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, extra: list | None = None) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    nv = nvcc()
    changed = force or not os.path.exists(LIB)
    for unit, flags in UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(BUILD, unit + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            cmd = [nv, *ARCH, *COMMON, *flags, *(extra or []), "-c", src, "-o", obj]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)
            changed = True
    for unit, flags in HOST_UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(BUILD, unit + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            subprocess.check_call(["g++", *flags, "-c", src, "-o", obj])
            changed = True
    if changed:
        cuda_lib = os.path.join(os.path.dirname(os.path.dirname(nv)), "lib64")
        subprocess.check_call([nv, *ARCH, "-shared", "-o", LIB, *objs,
                               f"-L{cuda_lib}", "-lcudart"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
