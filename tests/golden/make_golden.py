"""Generate the golden fixtures under tests/golden/ from the LIVE reference.

Run in the build container only (needs /root/reference):

    cp -r /root/reference/pkg /tmp/refbuild
    (cd /tmp/refbuild && python setup.py build_ext --inplace)
    PYTHONPATH=/tmp/refbuild/src OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Every array stored here is an output of the reference package `vmsplat`
(kernels.BACKEND == "cython") on inputs that are either stored alongside or
regenerated from seeds by tests/golden/inputs.py.  The CPU test
tests/test_oracle_golden.py pins oracle/ against these files; the GPU tests
then compare the CUDA path with the pinned oracle.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from vmsplat import kernels as rk  # noqa: E402  (the reference)
from vmsplat import render as rr  # noqa: E402
from vmsplat import runtime as rt  # noqa: E402
from vmsplat.harness import BenchConfig, _stats_rows, run_benchmark  # noqa: E402
from vmsplat.mesh import ProxyMesh  # noqa: E402
from vmsplat.pipeline import preprocess  # noqa: E402
from vmsplat.scene_io import read_scene, write_scene  # noqa: E402
from vmsplat import synthetic  # noqa: E402

from tests.golden import inputs  # noqa: E402

assert rk.BACKEND == "cython", "build the reference's Cython core first"


def stats_text(stats):
    return "\n".join(",".join(r) for r in _stats_rows(stats)) + "\n"


def kernels_golden():
    out = {}
    for seed in (0, 1, 2):
        args = inputs.random_splats(seed, 400, 64, 48)
        img = np.zeros((48, 64, 3), np.float32)
        rk.composite_splats(*args, img)
        out[f"composite_{seed}"] = img
    for seed in (3, 4):
        tris, ids = inputs.random_tris(seed)
        idi = np.zeros((48, 64), np.uint32)
        zi = np.zeros((48, 64), np.float64)
        rk.rasterize_triangles(tris, ids, idi, zi)
        out[f"raster_ids_{seed}"] = idi
        out[f"raster_invz_{seed}"] = zi
    for seed in range(4):
        keys = inputs.random_keys(seed, 5000)
        sk, sv = rk.radix_sort_pairs(keys, np.arange(len(keys), dtype=np.int64))
        out[f"radix_vals_{seed}"] = sv
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)


def render_golden():
    out = {}
    recs = inputs.small_records(7, 3000)
    for i, cam in enumerate(inputs.small_cameras()):
        c = rr.Camera(**cam)
        out[f"image_{i}"] = rr.render_records(recs, c)
        keys, idx = rr.compute_keys(recs, c)
        out[f"keys_{i}"] = keys
        out[f"keyidx_{i}"] = idx
        centers, conics, colors, alphas, bounds, kept = rr.project_records(recs, c)
        out[f"centers_{i}"] = centers
        out[f"conics_{i}"] = conics
        out[f"colors_{i}"] = colors
        out[f"bounds_{i}"] = bounds
        out[f"kept_{i}"] = kept
    sh_c, sh_d = inputs.sh_inputs(11, 500)
    out["sh"] = rr.evaluate_sh(sh_c, sh_d)
    np.savez_compressed(os.path.join(HERE, "render.npz"), **out)


def city_golden():
    """Visibility, reduction and whole-session goldens on a small city."""
    from paper_2506_19415_b200 import scenegen

    lay = inputs.CITY_SMALL
    sc_mine = scenegen.city_scene(lay)
    path = "/tmp/golden_city.vms"
    from paper_2506_19415_b200.scene_io import write_scene as my_write

    my_write(sc_mine, path)
    scene = read_scene(path, mmap_gaussians=True)  # the reference reads our file
    out = {"gaus_sha256": np.frombuffer(
        hashlib.sha256(np.ascontiguousarray(scene.gaussians).tobytes()).digest(), np.uint8)}
    mesh = ProxyMesh(scene.vertices.astype(np.float64), scene.faces.astype(np.int32),
                     scene.face_page.copy())
    links = rt.links_table(scene)
    for i, cam in enumerate(inputs.city_cameras(lay)):
        c = rr.Camera(**cam)
        ids, depth = rr.render_visibility(mesh, c)
        req = rt.reduce_visibility(ids, depth, links)
        out[f"vis_ids_{i}"] = ids
        out[f"vis_depth_{i}"] = depth
        out[f"req_depths_{i}"] = req.depths
        out[f"req_direct_{i}"] = req.direct
    # whole sessions: stats.csv + required lists + plans + images
    from vmsplat import camera_path as ref_cp

    cam_path = inputs.city_path(lay, ref_cp)
    for name, kw in inputs.SESSION_VARIANTS.items():
        session = rt.VmSession(scene, **kw)
        stats = []
        for f in range(cam_path.frame_count):
            cam = cam_path.frame_camera(f)
            img, st = session.render_frame(cam, f)
            stats.append(st)
            out[f"{name}_image_{f}"] = img
            out[f"{name}_resident_{f}"] = np.array(sorted(session.table.resident), np.int64)
        out[f"{name}_stats"] = np.frombuffer(stats_text(
            [_fs(s) for s in stats]).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "city.npz"), **out)


def _fs(raw):
    from vmsplat.harness import FrameStats

    return FrameStats(frame=raw["frame"], required=raw["required_pages"],
                      missing=raw["missing_pages"], bytes_copied=raw["bytes_copied"],
                      usage=raw["usage"], resident_per_level=raw["resident_per_level"],
                      thresholds=raw["thresholds"],
                      durations={k: 0.0 for k in ("visibility", "reduce", "update", "copy",
                                                  "sort", "render")})


def pagetable_golden():
    """Randomised trace replay of update_page_table."""
    out = {}
    for trace in range(40):
        spec = inputs.table_trace(trace)
        table = rt.PageTable(spec["capacity"])
        ctl = rt.LodController(spec["thresholds"])
        plans, missing, resident = [], [], []
        for f, (depths, direct) in enumerate(spec["frames"]):
            req = rt.RequiredList(depths=depths, direct=direct)
            plan, miss = rt.update_page_table(table, req, ctl, f, spec["budget"])
            table.check()
            plans.append([(p.page_id, p.level, p.entry, p.slot) for p in plan])
            missing.append(miss)
            resident.append(sorted((k, v[0], v[1]) for k, v in table.resident.items()))
        out[f"t{trace}_plan_len"] = np.array([len(p) for p in plans], np.int64)
        out[f"t{trace}_plan"] = np.array([x for p in plans for x in p], np.int64).reshape(-1, 4)
        out[f"t{trace}_missing"] = np.array(missing, np.int64)
        out[f"t{trace}_res_len"] = np.array([len(r) for r in resident], np.int64)
        out[f"t{trace}_res"] = np.array([x for r in resident for x in r], np.int64).reshape(-1, 3)
    np.savez_compressed(os.path.join(HERE, "pagetable.npz"), **out)


def c1_golden():
    """BASELINE config 1 exactly as the survey built it: box_scene(seed=3,
    100k) -> reference preprocess(page_size=1920, grid=64, ...) -> 8-frame
    straight path at 256^2.  Stores the layout (mesh, links, record
    permutation) so the GPU box can rebuild the identical scene without the
    reference, plus the reference session outputs."""
    recs = synthetic.box_scene(seed=3, count=100_000, extent=20.0, depth=40.0)
    scene = preprocess(recs, page_size=1920, grid=64, close_radius=1, open_radius=1,
                       target_faces=600, level_count=1)
    g = np.asarray(scene.gaussians)
    # recover the permutation: row -> box_scene index (-1 = padding)
    lut = {recs[i].tobytes(): i for i in range(len(recs))}
    perm = np.array([lut.get(g[r].tobytes(), -1) for r in range(len(g))], np.int32)
    assert np.array_equal(np.where(perm[:, None] >= 0, recs[np.maximum(perm, 0)], 0), g)
    out = {
        "page_size": np.int64(scene.page_size),
        "center": scene.center, "half_extent": np.float64(scene.half_extent),
        "vertices": scene.vertices, "faces": scene.faces, "face_page": scene.face_page,
        "link_offsets": scene.link_offsets, "link_targets": scene.link_targets,
        "perm": perm,
        "gaus_sha256": np.frombuffer(hashlib.sha256(g.tobytes()).digest(), np.uint8),
    }
    from vmsplat import camera_path as ref_cp

    path = inputs.c1_path(ref_cp)
    stats_list = []
    imgs = {}

    def sink(i, img):
        imgs[i] = img

    stats_list = run_benchmark(scene, path, BenchConfig(), frame_sink=sink)
    out["stats"] = np.frombuffer(stats_text(stats_list).encode(), np.uint8)
    for i, img in imgs.items():
        out[f"image_sha_{i}"] = np.frombuffer(hashlib.sha256(img.tobytes()).digest(), np.uint8)
        out[f"image_rowsum_{i}"] = img.astype(np.float64).sum(axis=1)
    out["image_last"] = imgs[max(imgs)]
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **out)


def bvh_golden():
    """Nearest-face queries: the reference's BVH arrays and answers."""
    from vmsplat.mesh.geometry import FaceBvh

    out = {}
    for name, tv, pts in inputs.bvh_cases():
        bvh = FaceBvh(tv)
        faces, dist = bvh.nearest(pts)
        out[f"{name}_tri_verts"] = tv
        out[f"{name}_points"] = pts
        out[f"{name}_bounds"] = bvh.bounds
        out[f"{name}_children"] = bvh.children
        out[f"{name}_ranges"] = bvh.ranges
        out[f"{name}_order"] = bvh.order
        out[f"{name}_faces"] = faces
        out[f"{name}_dist"] = dist
    # the city proxy mesh, queried at the scene's record positions
    from paper_2506_19415_b200 import scenegen

    sc = scenegen.city_scene(inputs.CITY_SMALL)
    tv = np.asarray(sc.vertices, np.float64)[np.asarray(sc.faces, np.int64)]
    pts = np.asarray(sc.gaussians[::7, 0:3], np.float64)
    faces, dist = FaceBvh(tv).nearest(pts)
    out["city_tri_verts"] = tv
    out["city_points"] = pts
    out["city_faces"] = faces
    out["city_dist"] = dist
    np.savez_compressed(os.path.join(HERE, "bvh.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["kernels", "render", "pagetable", "city", "c1"]
    for w in which:
        globals()[f"{w}_golden"]()
        print("wrote", w)
