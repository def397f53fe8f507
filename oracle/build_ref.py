"""ORACLE — TEST INFRASTRUCTURE ONLY.

Recipe that compiles the reference's OWN native hot loops
(/root/reference/pkg/src/vmsplat/kernels/_core.pyx, built upstream by
pkg/setup.py:14-24 with ``-O3 -ffp-contract=off``) straight from where they lie
into ``oracle/_ref/`` (git-ignored, travels to the GPU box with the snapshot).
Nothing is copied into the repo: Cython writes its C translation into
oracle/_ref/ and gcc links the extension there.

The result is the CPU baseline of kind "reference" for bench.py (the
reference's Cython kernels driven by the NumPy restatement in oracle/core.py)
and a second checker for the C restatement in oracle/kernels.c.
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
SRC = "/root/reference/pkg/src/vmsplat/kernels/_core.pyx"


def target():
    suffix = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
    return os.path.join(OUT, "_core" + suffix)


def build(force=False) -> str | None:
    so = target()
    if os.path.exists(so) and not force:
        return so
    if not os.path.exists(SRC):
        return None  # GPU box: /root/reference is absent; use the prebuilt file
    import numpy

    os.makedirs(OUT, exist_ok=True)
    c_file = os.path.join(OUT, "_core.c")
    subprocess.check_call([sys.executable, "-m", "cython", "-3", "-o", c_file, SRC])
    inc = [sysconfig.get_paths()["include"], numpy.get_include()]
    cmd = ["gcc", "-O3", "-ffp-contract=off", "-fPIC", "-shared",
           "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION"]
    cmd += [f"-I{d}" for d in inc] + ["-o", so, c_file, "-lm"]
    subprocess.check_call(cmd)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
