"""Kernel-level drop-in for ``vmsplat.kernels`` (pkg/src/vmsplat/kernels/__init__.py).

Same names, argument meaning and in-place/return conventions as the
reference wrappers, backed only by the sm_100a kernels in
libvmsplat_b200.so — there is no NumPy or CPU backend to fall back to
(``BACKEND`` is always "cuda").  Inputs may be NumPy arrays (copied to the
device and back, in place for the image arguments) or CUDA tensors (used in
place, no host round trip).
"""

from __future__ import annotations

import numpy as np

from paper_2506_19415_b200 import _device, _lib

BACKEND = "cuda"


def _instances(bounds, h, w) -> int:
    """Tile instances of the clamped half-open boxes (workspace sizing)."""
    if _device.is_torch(bounds):
        b = bounds.reshape(-1, 4).to("cpu").numpy()
    else:
        b = np.asarray(bounds).reshape(-1, 4)
    if len(b) == 0:
        return 0
    b = b.astype(np.int64)
    TILE = int(_lib.load().vms_tile_size())
    x0 = np.maximum(b[:, 0], 0)
    x1 = np.minimum(b[:, 1], w)
    y0 = np.maximum(b[:, 2], 0)
    y1 = np.minimum(b[:, 3], h)
    ok = (x1 > x0) & (y1 > y0)
    tx = np.where(ok, (x1 - 1) // TILE - x0 // TILE + 1, 0)
    ty = np.where(ok, (y1 - 1) // TILE - y0 // TILE + 1, 0)
    return int((tx * ty).sum())


def composite_splats(centers, conics, colors, alphas, bounds, image, exact: bool = True):
    """Blend caller-ordered splats into float32 ``image`` (h, w, 3) in place
    (kernels/__init__.py:24-33; contract _ref.py:16-54)."""
    t = _device.require_cuda()
    on_dev = _device.is_torch(image) and image.is_cuda
    if not on_dev:
        if image.dtype != np.float32 or not image.flags.c_contiguous or image.ndim != 3:
            raise ValueError("image must be a C-contiguous float32 (h, w, 3) array")
    h, w = int(image.shape[0]), int(image.shape[1])
    c = _device.to_dev(centers, np.float32).reshape(-1, 2)
    n = int(c.shape[0])
    q = _device.to_dev(conics, np.float32).reshape(-1, 3)
    col = _device.to_dev(colors, np.float32).reshape(-1, 3)
    al = _device.to_dev(alphas, np.float32).reshape(-1)
    bd = _device.to_dev(bounds, np.int32).reshape(-1, 4)
    if not (len(q) == len(col) == len(al) == len(bd) == n):
        raise ValueError("composite_splats: per-splat arrays disagree in length")
    m = _instances(bounds, h, w)
    img = image if on_dev else t.from_numpy(image).cuda()
    lib = _lib.load()
    nbytes = lib.vms_composite_workspace_bytes(n, m, h, w)
    ws = _device.workspace("composite", nbytes)
    _lib.check(lib.vms_composite_splats(c.data_ptr(), q.data_ptr(), col.data_ptr(), al.data_ptr(),
                                        bd.data_ptr(), n, m, img.data_ptr(), h, w, int(exact),
                                        ws.data_ptr(), ws.numel(), _device.sptr()),
               "composite_splats")
    if not on_dev:
        image[...] = img.cpu().numpy()


def rasterize_triangles(tris, ids, id_image, invz_image):
    """Depth-tested ID rasterization into ``id_image`` / ``invz_image`` in place
    (kernels/__init__.py:36-43; contract _ref.py:57-96)."""
    t = _device.require_cuda()
    on_dev = _device.is_torch(id_image) and id_image.is_cuda
    h, w = int(id_image.shape[0]), int(id_image.shape[1])
    tr = _device.to_dev(tris, np.float64).reshape(-1, 3, 3)
    n = int(tr.shape[0])
    ii = _device.to_dev(ids, np.uint32).reshape(-1)
    if len(ii) != n:
        raise ValueError("rasterize_triangles: ids length mismatch")
    if on_dev:
        idi, zi = id_image, invz_image
    else:
        if id_image.dtype != np.uint32 or invz_image.dtype != np.float64:
            raise ValueError("id_image must be uint32 and invz_image float64")
        idi = _device.to_dev(id_image, np.uint32)
        zi = _device.to_dev(invz_image, np.float64)
    lib = _lib.load()
    ws = _device.workspace("raster", lib.vms_rasterize_workspace_bytes(n))
    _lib.check(lib.vms_rasterize_triangles(tr.data_ptr(), ii.data_ptr(), n, idi.data_ptr(),
                                           zi.data_ptr(), h, w, ws.data_ptr(), ws.numel(),
                                           _device.sptr()), "rasterize_triangles")
    if not on_dev:
        id_image[...] = idi.cpu().numpy()
        invz_image[...] = zi.cpu().numpy()


def radix_sort_pairs(keys, values):
    """Stable ascending sort of uint32 keys with an int64 payload; returns
    sorted copies (kernels/__init__.py:46-51; contract _ref.py:99-112)."""
    t = _device.require_cuda()
    on_dev = _device.is_torch(keys) and keys.is_cuda
    k = _device.to_dev(keys, np.uint32).reshape(-1).clone()
    v = _device.to_dev(values, np.int64).reshape(-1).clone()
    n = int(k.shape[0])
    if len(v) != n:
        raise ValueError("radix_sort_pairs: keys/values length mismatch")
    lib = _lib.load()
    ws = _device.workspace("radix", lib.vms_radix_workspace_bytes(n))
    _lib.check(lib.vms_radix_sort_pairs(k.data_ptr(), v.data_ptr(), n, ws.data_ptr(), ws.numel(),
                                        _device.sptr()), "radix_sort_pairs")
    if on_dev:
        return k, v
    return k.cpu().numpy(), v.cpu().numpy()


def bvh_nearest_points(points, bounds, children, ranges, tri_order, tri_verts):
    """Nearest mesh face (int64, lowest index on ties) and its distance
    (float64) for each query point, over the flat BVH arrays of
    ``geometry.FaceBvh`` (kernels/__init__.py:54-63, _core.pyx:279-334).
    Raises RuntimeError when a query overflows the 128-entry traversal
    stack, as the reference does."""
    t = _device.require_cuda()
    on_dev = _device.is_torch(points) and points.is_cuda
    pts = _device.to_dev(points, np.float64).reshape(-1, 3)
    bnd = _device.to_dev(bounds, np.float64).reshape(-1, 6)
    ch = _device.to_dev(children, np.int32).reshape(-1, 2)
    rg = _device.to_dev(ranges, np.int32).reshape(-1, 2)
    order = _device.to_dev(tri_order, np.int32).reshape(-1)
    tv = _device.to_dev(tri_verts, np.float64).reshape(-1, 3, 3)
    if len(bnd) != len(ch) or len(bnd) != len(rg) or len(bnd) == 0 or len(tv) == 0:
        raise ValueError("bvh_nearest_points: inconsistent BVH arrays")
    n = int(pts.shape[0])
    face = t.empty(n, dtype=t.int64, device=pts.device)
    dist = t.empty(n, dtype=t.float64, device=pts.device)
    flag = t.zeros(1, dtype=t.int32, device=pts.device)
    lib = _lib.load()
    _lib.check(lib.vms_bvh_nearest_points(pts.data_ptr(), n, bnd.data_ptr(), ch.data_ptr(),
                                          rg.data_ptr(), len(bnd), order.data_ptr(),
                                          tv.data_ptr(), len(tv), face.data_ptr(),
                                          dist.data_ptr(), flag.data_ptr(), _device.sptr()),
               "bvh_nearest_points")
    if int(flag.item()):
        raise RuntimeError("BVH traversal stack overflow")
    if on_dev:
        return face, dist
    return face.cpu().numpy(), dist.cpu().numpy()


__all__ = ["BACKEND", "composite_splats", "rasterize_triangles", "radix_sort_pairs",
           "bvh_nearest_points"]
