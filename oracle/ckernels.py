"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of ``oracle/liboracle.so`` (the C restatement in
``oracle/kernels.c``) with the argument coercion of the reference wrappers
(pkg/src/vmsplat/kernels/__init__.py:24-51).  ``build()`` compiles it with
gcc ``-O3 -ffp-contract=off`` exactly as the reference builds its core
(pkg/setup.py:14-24).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_lib = None


def build(force=False):
    src = os.path.join(HERE, "kernels.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", LIB, src, "-lm"])
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        lib.oracle_composite_splats.argtypes = [P, P, P, P, P, I, P, I, I]
        lib.oracle_rasterize_triangles.argtypes = [P, P, I, P, P, I, I]
        lib.oracle_radix_sort_pairs.argtypes = [P, P, I]
        lib.oracle_nearest_faces.argtypes = [P, I, P, I, P, P]
        for f in (lib.oracle_composite_splats, lib.oracle_rasterize_triangles,
                  lib.oracle_radix_sort_pairs, lib.oracle_nearest_faces):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def composite_splats(centers, conics, colors, alphas, bounds, image):
    lib = _load()
    c = np.ascontiguousarray(centers, dtype=np.float32).reshape(-1, 2)
    q = np.ascontiguousarray(conics, dtype=np.float32).reshape(-1, 3)
    col = np.ascontiguousarray(colors, dtype=np.float32).reshape(-1, 3)
    al = np.ascontiguousarray(alphas, dtype=np.float32).reshape(-1)
    bd = np.ascontiguousarray(bounds, dtype=np.int32).reshape(-1, 4)
    assert image.dtype == np.float32 and image.flags.c_contiguous
    if lib.oracle_composite_splats(_p(c), _p(q), _p(col), _p(al), _p(bd), len(c),
                                   _p(image), image.shape[0], image.shape[1]) != 0:
        raise MemoryError("oracle composite")


def rasterize_triangles(tris, ids, id_image, invz_image):
    lib = _load()
    t = np.ascontiguousarray(tris, dtype=np.float64).reshape(-1, 3, 3)
    i = np.ascontiguousarray(ids, dtype=np.uint32).reshape(-1)
    assert id_image.dtype == np.uint32 and invz_image.dtype == np.float64
    lib.oracle_rasterize_triangles(_p(t), _p(i), len(t), _p(id_image), _p(invz_image),
                                   id_image.shape[0], id_image.shape[1])


def radix_sort_pairs(keys, values):
    lib = _load()
    k = np.array(keys, dtype=np.uint32, copy=True).reshape(-1)
    v = np.array(values, dtype=np.int64, copy=True).reshape(-1)
    if lib.oracle_radix_sort_pairs(_p(k), _p(v), len(k)) != 0:
        raise MemoryError("oracle radix")
    return k, v


def nearest_faces(points, tri_verts):
    """(faces int64, distances float64) per point: the answer of
    bvh_nearest_points (kernels/_core.pyx:279-334) by brute force."""
    lib = _load()
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    tv = np.ascontiguousarray(tri_verts, dtype=np.float64).reshape(-1, 3, 3)
    face = np.empty(len(pts), np.int64)
    dist = np.empty(len(pts), np.float64)
    lib.oracle_nearest_faces(_p(pts), len(pts), _p(tv), len(tv), _p(face), _p(dist))
    return face, dist
