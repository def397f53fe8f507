"""Golden fixtures for the LOD pyramid from the LIVE
reference ``vmsplat.lod`` (pkg/src/vmsplat/lod.py).  Build container only:

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_lod_golden.py

Inputs are regenerated from seeds by tests/golden/inputs.py; outputs go to
tests/golden/lod.npz (the C2-size page only as SHA-256 digests).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from vmsplat import lod  # noqa: E402  (the reference)

from tests.golden import inputs  # noqa: E402


def main():
    out = {}
    # cluster_page (lod.py:83-131) + the Generator state it leaves behind
    walls = inputs.wall_scene(seed=6, count=120, extent=2.0, z=0.0)
    blobs = np.concatenate([inputs.wall_scene(seed=1, count=30, extent=0.5, z=0.0),
                            inputs.wall_scene(seed=2, count=30, extent=0.5, z=50.0)])
    dups = np.repeat(inputs.wall_scene(seed=9, count=40, extent=1.0, z=0.0), 3, axis=0)
    cases = [("w16", walls, 16, 3, 50), ("w10", walls, 10, 3, 50), ("blobs", blobs, 2, 1, 50),
             ("dups", dups, 70, 5, 50), ("w60i3", walls, 60, 8, 3)]
    for name, recs, k, seed, iters in cases:
        g = lod._page_rng(seed, 0)
        a = lod.cluster_page(recs, k, max_iters=iters, rng=g)
        out[f"cluster_{name}"] = a
        out[f"cluster_{name}_next"] = g.integers(0, 2**62, size=3)
    # merge_cluster (lod.py:134-154)
    rec = inputs.wall_scene(seed=7, count=1, extent=1.0, z=0.0)[0]
    flipped = rec.copy()
    flipped[3:7] *= -1.0
    merges = {"six": inputs.wall_scene(seed=7, count=6, extent=1.0, z=0.0),
              "hemi": np.stack([rec, flipped]), "one": rec[None],
              "many": inputs.box_scene(seed=4, count=300, extent=2.0, depth=5.0)}
    for name, m in merges.items():
        out[f"merge_{name}"] = lod.merge_cluster(m)
    # build_pyramid (lod.py:179-226)
    for name, counts, ps, levels, iters, seed, dup in inputs.LOD_PYRAMIDS:
        lv = lod.build_pyramid(inputs.padded_pages(counts, ps, dup=dup), ps, level_count=levels,
                               max_iters=iters, seed=seed)
        for k in range(1, levels):
            out[f"pyr_{name}_{k}"] = lv[k]
    name, counts, ps, levels, iters, seed, dup = inputs.LOD_BIG
    lv = lod.build_pyramid(inputs.padded_pages(counts, ps, dup=dup), ps, level_count=levels,
                           max_iters=iters, seed=seed)
    for k in range(1, levels):
        out[f"pyr_{name}_{k}_sha256"] = np.frombuffer(
            hashlib.sha256(np.ascontiguousarray(lv[k]).tobytes()).digest(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "lod.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
