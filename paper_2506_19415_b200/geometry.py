"""Nearest-face queries on the proxy mesh (pkg/src/vmsplat/mesh/geometry.py:86-158).

``FaceBvh`` builds the reference's flat median-split BVH on the host (the
same node numbering, boxes, leaf spans and face order) and answers
``nearest`` with the sm_100a kernel behind ``kernels.bvh_nearest_points``;
the page builder's link sampling (paging.py:336) and record assignment
(paging.py:68) are its callers.  Results do not depend on the tree shape:
equal-distance boxes are never pruned and ties go to the lowest face index.
"""

from __future__ import annotations

import numpy as np

from paper_2506_19415_b200 import kernels
from paper_2506_19415_b200.errors import InvariantViolation


class FaceBvh:
    """Flat arrays: ``bounds`` (n, 6) lo|hi per node, ``children`` (n, 2)
    with (-1, -1) on leaves, ``ranges`` (n, 2) half-open spans of ``order``
    (the face permutation), ``tri_verts`` (F, 3, 3)."""

    LEAF_SIZE = 8

    def __init__(self, tri_verts: np.ndarray):
        tv = np.ascontiguousarray(tri_verts, dtype=np.float64).reshape(-1, 3, 3)
        if len(tv) == 0:
            raise InvariantViolation("cannot build a BVH over an empty mesh")
        self.tri_verts = tv
        lo, hi, mid = tv.min(axis=1), tv.max(axis=1), tv.mean(axis=1)
        order = np.arange(len(tv), dtype=np.int32)
        box, kids, span = [None], [(-1, -1)], [(0, len(tv))]
        todo = [(0, 0, len(tv))]  # LIFO: the right half of a split is built first
        while todo:
            node, a, b = todo.pop()
            sel = order[a:b]
            box[node] = np.concatenate([lo[sel].min(axis=0), hi[sel].max(axis=0)])
            span[node] = (a, b)
            if b - a <= self.LEAF_SIZE:
                continue
            c = mid[sel]
            axis = int(np.argmax(c.max(axis=0) - c.min(axis=0)))  # widest centroid extent
            order[a:b] = sel[np.argsort(c[:, axis], kind="stable")]
            half = a + (b - a) // 2
            left = len(box)
            box += [None, None]
            kids += [(-1, -1), (-1, -1)]
            span += [(0, 0), (0, 0)]
            kids[node] = (left, left + 1)
            todo += [(left, a, half), (left + 1, half, b)]
        self.bounds = np.ascontiguousarray(np.stack(box), dtype=np.float64)
        self.children = np.ascontiguousarray(kids, dtype=np.int32)
        self.ranges = np.ascontiguousarray(span, dtype=np.int32)
        self.order = order

    @classmethod
    def from_mesh(cls, mesh) -> "FaceBvh":
        v = np.asarray(mesh.vertices, dtype=np.float64)
        f = np.asarray(mesh.faces, dtype=np.int64)
        return cls(v[f])

    def nearest(self, points: np.ndarray):
        """(faces int64, distances float64) per query point."""
        pts = np.ascontiguousarray(np.atleast_2d(points), dtype=np.float64)
        return kernels.bvh_nearest_points(pts, self.bounds, self.children, self.ranges,
                                          self.order, self.tri_verts)


def nearest_faces(mesh, points: np.ndarray):
    """Build a BVH over the mesh and query it once (geometry.py:156-158)."""
    return FaceBvh.from_mesh(mesh).nearest(points)
