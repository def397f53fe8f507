"""ORACLE — TEST INFRASTRUCTURE ONLY.

Loads the reference's own Cython hot loops compiled by ``oracle/build_ref.py``
into ``oracle/_ref/`` and exposes them with the reference wrapper coercions
(pkg/src/vmsplat/kernels/__init__.py:24-51).  ``available()`` is False when
the extension was not built.
"""

from __future__ import annotations

import importlib.util
import os

import numpy as np

from oracle import build_ref

_mod = None


def _load():
    global _mod
    if _mod is None:
        so = build_ref.target()
        if not os.path.exists(so):
            raise ImportError("oracle/_ref/_core not built")
        spec = importlib.util.spec_from_file_location("_core", so)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _mod = mod
    return _mod


def available() -> bool:
    try:
        _load()
        return True
    except ImportError:
        return False


def composite_splats(centers, conics, colors, alphas, bounds, image):
    _load().composite_splats(
        np.ascontiguousarray(centers, dtype=np.float32),
        np.ascontiguousarray(conics, dtype=np.float32),
        np.ascontiguousarray(colors, dtype=np.float32),
        np.ascontiguousarray(alphas, dtype=np.float32),
        np.ascontiguousarray(bounds, dtype=np.int32),
        image,
    )


def rasterize_triangles(tris, ids, id_image, invz_image):
    _load().rasterize_triangles(
        np.ascontiguousarray(tris, dtype=np.float64),
        np.ascontiguousarray(ids, dtype=np.uint32),
        id_image,
        invz_image,
    )


def radix_sort_pairs(keys, values):
    return _load().radix_sort_pairs(
        np.ascontiguousarray(keys, dtype=np.uint32),
        np.ascontiguousarray(values, dtype=np.int64),
    )
