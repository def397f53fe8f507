"""Pin the CPU oracle (oracle/) to the live reference: every golden vector in
tests/golden/*.npz was produced by the reference package itself
(tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import ckernels, core
from tests.golden import inputs


def test_oracle_composite_matches_reference(golden):
    g = golden["kernels"]
    for seed in (0, 1, 2):
        img = np.zeros((48, 64, 3), np.float32)
        ckernels.composite_splats(*inputs.random_splats(seed, 400, 64, 48), img)
        assert np.array_equal(img, g[f"composite_{seed}"])


def test_oracle_rasterize_matches_reference(golden):
    g = golden["kernels"]
    for seed in (3, 4):
        tris, ids = inputs.random_tris(seed)
        idi = np.zeros((48, 64), np.uint32)
        zi = np.zeros((48, 64), np.float64)
        ckernels.rasterize_triangles(tris, ids, idi, zi)
        assert np.array_equal(idi, g[f"raster_ids_{seed}"])
        assert np.array_equal(zi.view(np.uint64), g[f"raster_invz_{seed}"].view(np.uint64))


def test_oracle_radix_matches_reference(golden):
    g = golden["kernels"]
    for seed in range(4):
        keys = inputs.random_keys(seed, 5000)
        sk, sv = ckernels.radix_sort_pairs(keys, np.arange(len(keys)))
        assert np.array_equal(sv, g[f"radix_vals_{seed}"])
        assert np.array_equal(sk, keys[sv])


def test_oracle_render_matches_reference(golden):
    g = golden["render"]
    recs = inputs.small_records(7, 3000)
    for i, cam in enumerate(inputs.small_cameras()):
        c = core.OCamera(**cam)
        assert np.array_equal(core.render_flat(recs, c), g[f"image_{i}"])
        k, idx = core.keys_of(recs, c)
        assert np.array_equal(k, g[f"keys_{i}"]) and np.array_equal(idx, g[f"keyidx_{i}"])
        centers, conics, colors, _, bounds, kept = core.project(recs, c)
        assert np.array_equal(centers, g[f"centers_{i}"])
        assert np.array_equal(conics, g[f"conics_{i}"])
        assert np.array_equal(colors, g[f"colors_{i}"])
        assert np.array_equal(bounds, g[f"bounds_{i}"])
        assert np.array_equal(kept, g[f"kept_{i}"])
    c, d = inputs.sh_inputs(11, 500)
    assert np.array_equal(core.sh_rgb(c, d), g["sh"])


def test_oracle_page_table_traces_match_reference(golden):
    g = golden["pagetable"]
    for trace in range(40):
        spec = inputs.table_trace(trace)
        table = core.OTable(spec["capacity"])
        ctl = core.OController(spec["thresholds"])
        plans, missing, res = [], [], []
        for f, (depths, direct) in enumerate(spec["frames"]):
            plan, miss = core.update_table(table, core.ORequired(depths, direct), ctl, f,
                                           spec["budget"])
            table.check()
            plans.extend(plan)
            missing.append(miss)
            res.extend(sorted((k, v[0], v[1]) for k, v in table.resident.items()))
        assert np.array_equal(np.array(plans, np.int64).reshape(-1, 4), g[f"t{trace}_plan"])
        assert np.array_equal(missing, g[f"t{trace}_missing"])
        assert np.array_equal(np.array(res, np.int64).reshape(-1, 3), g[f"t{trace}_res"])


def _city():
    from paper_2506_19415_b200 import scenegen

    return scenegen.city_scene(inputs.CITY_SMALL)


def test_oracle_visibility_matches_reference(golden):
    g = golden["city"]
    sc = _city()
    assert hashlib.sha256(sc.gaussians.tobytes()).digest() == g["gaus_sha256"].tobytes()
    links = core.link_lists(sc.link_offsets, sc.link_targets, sc.page_count)
    for i, cam in enumerate(inputs.city_cameras(inputs.CITY_SMALL)):
        c = core.OCamera(**cam)
        ids, depth = core.visibility(sc.vertices.astype(np.float64), sc.faces.astype(np.int32),
                                     sc.face_page, c)
        assert np.array_equal(ids, g[f"vis_ids_{i}"])
        assert np.array_equal(depth.view(np.uint64), g[f"vis_depth_{i}"].view(np.uint64))
        req = core.reduce_pages(ids, depth, links)
        assert np.array_equal(req.depths, g[f"req_depths_{i}"])
        assert np.array_equal(req.direct, g[f"req_direct_{i}"])


@pytest.mark.parametrize("variant", sorted(inputs.SESSION_VARIANTS))
def test_oracle_session_matches_reference(golden, variant):
    g = golden["city"]
    sc = _city()
    path = inputs.city_path(inputs.CITY_SMALL)
    s = core.OSession(sc, **inputs.SESSION_VARIANTS[variant])
    stats = []
    for f in range(path.frame_count):
        img, st = s.render_frame(path.frame_camera(f), f)
        stats.append(st)
        assert np.array_equal(img, g[f"{variant}_image_{f}"]), f
        assert np.array_equal(np.array(sorted(s.table.resident), np.int64),
                              g[f"{variant}_resident_{f}"])
    assert core.stats_csv(stats).encode() == g[f"{variant}_stats"].tobytes()


def test_oracle_c1_session_matches_reference(golden):
    """BASELINE config 1, the whole 8-frame path, default session knobs."""
    g = golden["c1"]
    sc, _ = inputs.c1_scene()
    path = inputs.c1_path()
    s = core.OSession(sc)
    stats = []
    for f in range(path.frame_count):
        img, st = s.render_frame(path.frame_camera(f), f)
        stats.append(st)
        assert hashlib.sha256(img.tobytes()).digest() == g[f"image_sha_{f}"].tobytes(), f
    assert core.stats_csv(stats).encode() == g["stats"].tobytes()


# -- nearest-face queries -----------------------------------
@pytest.mark.parametrize("case", ["random", "grid", "city"])
def test_oracle_nearest_faces_match_reference(golden, case):
    """kernels/_core.pyx:279-334 by brute force: faces (ties -> lowest index,
    the grid case has many) and distances bit for bit."""
    from oracle import ckernels

    g = golden["bvh"]
    faces, dist = ckernels.nearest_faces(g[f"{case}_points"], g[f"{case}_tri_verts"])
    assert np.array_equal(faces, g[f"{case}_faces"])
    assert np.array_equal(dist.view(np.uint64), g[f"{case}_dist"].view(np.uint64))


@pytest.mark.parametrize("case", ["random", "grid"])
def test_face_bvh_arrays_match_reference(golden, case):
    """geometry.FaceBvh builds mesh/geometry.py:86-142's flat BVH exactly
    (node numbering, boxes, spans, face order) - host code, no GPU."""
    from paper_2506_19415_b200.geometry import FaceBvh

    g = golden["bvh"]
    b = FaceBvh(g[f"{case}_tri_verts"])
    assert np.array_equal(b.bounds, g[f"{case}_bounds"])
    assert np.array_equal(b.children, g[f"{case}_children"])
    assert np.array_equal(b.ranges, g[f"{case}_ranges"])
    assert np.array_equal(b.order, g[f"{case}_order"])


def test_oracle_clipped_triangles_match_per_face_loop():
    """The vectorised clip/project (faces wholly beyond the near plane in
    one pass) emits the per-face loop's triangles bit for bit, in (face, fan)
    order, including faces crossing the plane and faces behind it."""
    rng = np.random.default_rng(3)
    verts = rng.uniform(-10, 10, size=(300, 3))
    verts[:, 2] = rng.uniform(-2, 12, size=300)
    faces = rng.integers(0, 300, size=(500, 3)).astype(np.int32)
    fpage = rng.integers(1, 60, size=500).astype(np.uint32)
    cam = core.OCamera((0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0), np.pi / 2, 64, 48, near=0.5)
    tris, ids = core.clipped_triangles(verts, faces, fpage, cam)
    view = cam.to_view(verts)
    ref_t, ref_i = [], []
    for fi in range(len(faces)):
        for cl in core.clip_near(view[faces[fi]], cam.near):
            ref_t.append(cam.to_pixels(cl))
            ref_i.append(fpage[fi])
    assert len(ref_t) == len(tris) and len(tris) > 400
    assert np.array_equal(np.stack(ref_t).view(np.uint64), tris.view(np.uint64))
    assert np.array_equal(np.asarray(ref_i, np.uint32), ids)


@pytest.mark.parametrize("window", [(0, 64, 0, 48), (10, 30, 5, 21), (50, 64, 40, 48)])
def test_oracle_render_window_equals_full_render(golden, window):
    """the windowed render reproduces the full render's
    window bit for bit (the C4 image-parity oracle)."""
    recs = inputs.small_records(7, 3000)
    for cam in inputs.small_cameras():
        c = core.OCamera(**cam)
        full = core.render_flat(recs, c)
        x0, x1, y0, y1 = window
        x1, y1 = min(x1, c.width), min(y1, c.height)
        win, n = core.render_window(recs, c, (x0, x1, y0, y1), chunk=700)
        assert np.array_equal(win, full[y0:y1, x0:x1])
