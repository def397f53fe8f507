"""The reference package's import names (``vmsplat.render``, ``vmsplat.runtime``,
``vmsplat.kernels``, ...) mapped onto this package, so the hot-path tests of
the reference suite (pkg/tests/) read with the reference's imports
(tests/test_reference_suite.py).  ``install()`` registers the aliases in
sys.modules; ``scene(name)`` opens a fixture built by the reference's own
preprocessing pipeline (tests/golden/make_reference_scenes.py).
"""

from __future__ import annotations

import gzip
import json
import os
import shutil
import sys
import tempfile
import types

HERE = os.path.dirname(os.path.abspath(__file__))
SCENES = os.path.join(HERE, "golden", "ref_scenes")


def install():
    if "vmsplat" in sys.modules and getattr(sys.modules["vmsplat"], "IS_ALIAS", False):
        return sys.modules["vmsplat"]
    from paper_2506_19415_b200 import (camera_path, errors, gaussians, harness, kernels, lod,
                                       render, runtime, scene_io)

    pkg = types.ModuleType("vmsplat")
    pkg.__path__ = []
    pkg.IS_ALIAS = True
    mesh = types.ModuleType("vmsplat.mesh")
    mesh.ProxyMesh = runtime.ProxyMesh
    from oracle import core as _metrics_restatement  # test-side metrics (metrics.py)

    metrics = types.ModuleType("vmsplat.metrics")
    metrics.psnr = _metrics_restatement.psnr
    metrics.ssim = _metrics_restatement.ssim
    mods = {"render": render, "runtime": runtime, "kernels": kernels, "scene_io": scene_io,
            "errors": errors, "gaussians": gaussians, "camera_path": camera_path,
            "harness": harness, "mesh": mesh, "metrics": metrics, "lod": lod}
    sys.modules["vmsplat"] = pkg
    for name, mod in mods.items():
        setattr(pkg, name, mod)
        sys.modules[f"vmsplat.{name}"] = mod
    return pkg


_tmp = None


def scene_path(name: str) -> str:
    """Decompressed path of a reference-built scene fixture."""
    global _tmp
    if _tmp is None:
        _tmp = tempfile.mkdtemp(prefix="vmsplat_refsuite_")
    out = os.path.join(_tmp, f"{name}.vms")
    if not os.path.exists(out):
        with gzip.open(os.path.join(SCENES, f"{name}.vms.gz"), "rb") as fi, open(out, "wb") as fo:
            shutil.copyfileobj(fi, fo)
    return out


def scene(name: str):
    from paper_2506_19415_b200.scene_io import read_scene

    return read_scene(scene_path(name), mmap_gaussians=True)


def layout(name: str) -> dict:
    with open(os.path.join(SCENES, "layouts.json")) as fh:
        return json.load(fh)[name]
