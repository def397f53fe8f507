"""Deterministic inputs shared by tests/golden/make_golden.py (run against the
reference) and the tests (run against oracle/ and the CUDA path).  Nothing
here imports the reference; generators that restate the reference's own test
inputs cite them."""

from __future__ import annotations

import math

import numpy as np

RECORD_SIZE = 59
SH_C0 = 0.28209479177387814


def random_splats(seed, n, w, h):
    """pkg/tests/test_kernels.py:21-34."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-5, max(w, h) + 5, size=(n, 2)).astype(np.float32)
    ell = rng.uniform(0.2, 1.5, size=(n, 2, 2))
    cov = ell @ ell.transpose(0, 2, 1) + 0.3 * np.eye(2)
    inv = np.linalg.inv(cov)
    conics = np.stack([inv[:, 0, 0], inv[:, 0, 1], inv[:, 1, 1]], axis=1).astype(np.float32)
    colors = rng.uniform(0, 1, size=(n, 3)).astype(np.float32)
    alphas = rng.uniform(0.05, 1.0, size=n).astype(np.float32)
    r = rng.integers(1, 12, size=n)
    x0 = np.floor(centers[:, 0] - r).astype(np.int32)
    y0 = np.floor(centers[:, 1] - r).astype(np.int32)
    bounds = np.stack([x0, x0 + 2 * r, y0, y0 + 2 * r], axis=1).astype(np.int32)
    return centers, conics, colors, alphas, bounds


def random_tris(seed, t=120):
    """pkg/tests/test_kernels.py:80-87."""
    rng = np.random.default_rng(seed)
    tris = np.empty((t, 3, 3), dtype=np.float64)
    tris[:, :, 0] = rng.uniform(-10, 74, size=(t, 3))
    tris[:, :, 1] = rng.uniform(-10, 58, size=(t, 3))
    tris[:, :, 2] = rng.uniform(0.01, 2.0, size=(t, 3))
    ids = rng.integers(1, 500, size=t).astype(np.uint32)
    return tris, ids


def bvh_cases():
    """Nearest-face query inputs (kernels/_core.pyx:279-334): (name, tri_verts
    (F, 3, 3) f64, points (Q, 3) f64)."""
    rng = np.random.default_rng(21)
    out = []
    # random triangles in a box, queries inside and around it
    a = rng.uniform(-5.0, 5.0, (600, 1, 3))
    tv = a + rng.normal(0.0, 0.6, (600, 3, 3))
    pts = rng.uniform(-7.0, 7.0, (3000, 3))
    out.append(("random", tv, pts))
    # a regular grid of quads (two triangles each): queries on shared
    # vertices and edges and above cell centres give exact distance ties
    n = 24
    g = np.stack(np.meshgrid(np.arange(n + 1.0), np.arange(n + 1.0), indexing="ij"), -1)
    v = np.concatenate([g.reshape(-1, 2), np.zeros(((n + 1) ** 2, 1))], 1)
    idx = np.arange((n + 1) ** 2).reshape(n + 1, n + 1)
    f = []
    for i in range(n):
        for j in range(n):
            f.append((idx[i, j], idx[i + 1, j], idx[i + 1, j + 1]))
            f.append((idx[i, j], idx[i + 1, j + 1], idx[i, j + 1]))
    tv = v[np.array(f)]
    q = rng.integers(0, n + 1, (1500, 2)).astype(np.float64)
    half = rng.integers(0, 2, (1500, 2)) * 0.5
    h = rng.choice([0.0, 0.25, -1.0, 3.0], 1500)[:, None]
    pts = np.concatenate([q + half, h], 1)
    out.append(("grid", tv, pts))
    return out


def random_keys(seed, n):
    rng = np.random.default_rng(seed)
    keys = rng.integers(0, 2 ** 32, size=n, dtype=np.uint64).astype(np.uint32)
    keys[: n // 4] = keys[n // 4: n // 2]  # plenty of duplicates: stability matters
    return keys


def small_records(seed, n):
    """Records in front of the origin, some padding, some behind the camera,
    all SH bands populated, random orientations."""
    rng = np.random.default_rng(seed)
    rec = np.zeros((n, RECORD_SIZE), np.float32)
    rec[:, 0] = rng.uniform(-4, 4, n)
    rec[:, 1] = rng.uniform(-4, 4, n)
    rec[:, 2] = rng.uniform(-2, 12, n)
    q = rng.normal(size=(n, 4))
    rec[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    rec[:, 7:10] = np.exp(rng.normal(np.log(0.12), 0.4, size=(n, 3)))
    rec[:, 10] = rng.uniform(0.3, 0.98, n)
    col = rng.uniform(0.05, 0.95, size=(n, 3))
    rec[:, 11:14] = (col - 0.5) / SH_C0
    rec[:, 14:59] = rng.normal(scale=0.05, size=(n, 45))
    rec[rng.choice(n, n // 20, replace=False)] = 0.0  # padding rows
    return rec


def _yaw_pitch(yaw, pitch):
    cy, sy = math.cos(yaw / 2), math.sin(yaw / 2)
    cp, sp = math.cos(pitch / 2), math.sin(pitch / 2)
    # q = q_yaw (about Y) * q_pitch (about X)
    w = cy * cp
    x = cy * sp
    y = sy * cp
    z = -sy * sp
    n = math.sqrt(w * w + x * x + y * y + z * z)
    return (w / n, x / n, y / n, z / n)


def small_cameras():
    return [
        dict(position=(0.0, 0.0, -3.0), orientation=(1.0, 0.0, 0.0, 0.0), fov_y=math.pi / 2,
             width=64, height=64),
        dict(position=(0.3, -0.2, -2.0), orientation=_yaw_pitch(0.21, -0.13), fov_y=1.2,
             width=80, height=56),
        dict(position=(1.1, 0.4, -5.0), orientation=_yaw_pitch(-0.37, 0.08), fov_y=0.9,
             width=48, height=72, near=0.2),
    ]


def sh_inputs(seed, n):
    rng = np.random.default_rng(seed)
    c = rng.normal(scale=0.4, size=(n, 16, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return c, d


def table_trace(trace):
    """A random update_page_table trace (SURVEY Appendix A.4 harness)."""
    rng = np.random.default_rng(1000 + trace)
    capacity = int(rng.integers(1, 30))
    pages = int(rng.integers(1, 90))
    levels = int(rng.integers(1, 5))
    thresholds = np.sort(rng.uniform(1.0, 60.0, size=levels - 1))
    thresholds = np.unique(thresholds)
    budget = float(rng.choice([0.25, 0.5, 1.0, 2.0, 3.0, 5.0, 10.0, np.inf]))
    frames = []
    for _ in range(int(rng.integers(5, 40))):
        depths = np.zeros(pages + 1, np.uint32)
        direct = np.zeros(pages + 1, bool)
        k = int(rng.integers(0, pages + 1))
        ids = rng.choice(np.arange(1, pages + 1), size=k, replace=False)
        d = rng.uniform(0.5, 80.0, size=k).astype(np.float32)
        d[rng.random(k) < 0.2] = np.float32(7.5)  # ties
        depths[ids] = np.uint32(0xFFFFFFFF) - d.view(np.uint32)
        direct[ids] = rng.random(k) < 0.7
        frames.append((depths, direct))
    return dict(capacity=capacity, thresholds=thresholds, budget=budget, frames=frames)


# a small city: 40 pages, 3 LOD levels (page_size 256 -> 256/128/64 records)
def _city_small():
    from paper_2506_19415_b200.scenegen import CityLayout

    return CityLayout(n_pages=40, page_size=256, levels=3, seed=5, scale=0.12)


CITY_SMALL = None
try:  # the package is importable in both contexts (no CUDA needed here)
    CITY_SMALL = _city_small()
except Exception:  # pragma: no cover
    CITY_SMALL = None


def city_cameras(lay):
    sx = lay.width + 0.5 * lay.street
    return [
        dict(position=(sx, -3.0, -6.0), orientation=(1.0, 0.0, 0.0, 0.0), fov_y=math.pi / 2,
             width=96, height=64),
        dict(position=(sx - 2.0, -6.0, 4.0), orientation=_yaw_pitch(0.6, 0.2), fov_y=1.3,
             width=80, height=80),
        dict(position=(-3.0, -4.0, -3.0), orientation=_yaw_pitch(0.8, 0.05), fov_y=1.0,
             width=72, height=48),
        dict(position=(sx, -2.0, 5.0), orientation=_yaw_pitch(math.pi, 0.0), fov_y=1.5,
             width=64, height=64, near=0.5),
    ]


def city_path(lay, cp_module=None):
    if cp_module is None:
        from paper_2506_19415_b200 import camera_path as cp_module
    sx = lay.width + 0.5 * lay.street
    cps = (cp_module.Checkpoint((sx, -3.0, -8.0), (1.0, 0.0, 0.0, 0.0)),
           cp_module.Checkpoint((sx, -3.0, 8.0), _yaw_pitch(0.0, 0.1)),
           cp_module.Checkpoint((sx + 5.0, -5.0, 14.0), _yaw_pitch(1.2, 0.1)))
    return cp_module.CameraPath(cps, speed=3.0, fps=1.0, fov_deg=80.0, width=64, height=48)


SESSION_VARIANTS = {
    "default": dict(buffer_pages=16, staging_pages=6.0, vis_scale=0.5),
    "nolod": dict(buffer_pages=12, staging_pages=4.0, vis_scale=0.5, lod_enabled=False),
    "nolinks": dict(buffer_pages=20, staging_pages=3.5, vis_scale=0.25, links_enabled=False),
}


def _synthetic_records(rng, pos, scale, opacity_range=(0.55, 0.95)):
    """Restates pkg/src/vmsplat/synthetic.py:20-35 (same RNG call order)."""
    n = len(pos)
    out = np.zeros((n, RECORD_SIZE), dtype=np.float32)
    out[:, 0:3] = pos
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    out[:, 3:7] = q
    out[:, 7:10] = scale
    out[:, 10] = rng.uniform(*opacity_range, size=n)
    colors = 0.5 + 0.35 * np.sin(pos * np.array([0.7, 1.1, 0.4]) + np.array([0.0, 2.1, 4.2]))
    colors += rng.normal(scale=0.03, size=(n, 3))
    out[:, 11:14] = (np.clip(colors, 0.05, 0.95) - 0.5) / SH_C0
    out[:, 14:17] = rng.normal(scale=0.02, size=(n, 3))
    return out


def box_scene(seed=3, count=30000, extent=20.0, depth=40.0):
    """Restates pkg/src/vmsplat/synthetic.py:116-128."""
    rng = np.random.default_rng(seed)
    pos = np.column_stack([rng.uniform(-extent, extent, count),
                           rng.uniform(-extent, extent, count),
                           rng.uniform(2.0, depth, count)])
    s = np.exp(rng.normal(np.log(0.18), 0.25, size=(count, 3))).astype(np.float32)
    return _synthetic_records(rng, pos, s)


def c1_scene(golden_dir=None):
    """Rebuild BASELINE config 1 (the reference-preprocessed box scene) from
    tests/golden/c1.npz without the reference: box_scene records gathered
    by the stored page permutation, mesh and links from the fixture."""
    import os

    from paper_2506_19415_b200.scene_io import SceneFile

    d = golden_dir or os.path.dirname(os.path.abspath(__file__))
    z = np.load(os.path.join(d, "c1.npz"))
    recs = box_scene(seed=3, count=100_000, extent=20.0, depth=40.0)
    perm = z["perm"]
    g = np.zeros((len(perm), RECORD_SIZE), np.float32)
    live = perm >= 0
    g[live] = recs[perm[live]]
    ps = int(z["page_size"])
    return SceneFile(stage="paged", page_size=ps, lod_levels=1, page_counts=[len(perm) // ps],
                     center=z["center"], half_extent=float(z["half_extent"]),
                     vertices=z["vertices"], faces=z["faces"], face_page=z["face_page"],
                     link_offsets=z["link_offsets"], link_targets=z["link_targets"],
                     gaussians=g), z


def c1_path(cp_module=None):
    """BASELINE config 1: 8-view straight path z -2 -> -16 at 256^2
    (speed 2, fps 1 -> 8 frames)."""
    if cp_module is None:
        from paper_2506_19415_b200 import camera_path as cp_module
    cps = (cp_module.Checkpoint((0.0, 0.0, -2.0), (1.0, 0.0, 0.0, 0.0)),
           cp_module.Checkpoint((0.0, 0.0, -16.0), (1.0, 0.0, 0.0, 0.0)))
    return cp_module.CameraPath(cps, speed=2.0, fps=1.0, fov_deg=90.0, width=256, height=256)


def wall_scene(seed=2, count=12000, extent=8.0, z=10.0, thickness=0.3, scale=0.28):
    """Restates pkg/src/vmsplat/synthetic.py:36-50,110-113."""
    rng = np.random.default_rng(seed)
    pos = np.column_stack([rng.uniform(-extent, extent, count),
                           rng.uniform(-extent, extent, count),
                           rng.normal(z, thickness, count)])
    s = np.exp(rng.normal(np.log(scale), 0.25, size=(count, 3))).astype(np.float32)
    s[:, 2] *= 0.6
    return _synthetic_records(rng, pos, s)


def padded_pages(counts, page_size, seed0=10, dup=1):
    """Level-0 pages (lod tests): page i holds counts[i] box-scene records
    (each repeated `dup` times, so k-means sees coincident points), padded
    with zero rows to page_size."""
    rows = []
    for i, c in enumerate(counts):
        base = box_scene(seed=seed0 + i, count=-(-c // dup), extent=3.0, depth=8.0)
        r = np.repeat(base, dup, axis=0)[:c]
        pad = np.zeros((page_size - c, RECORD_SIZE), np.float32)
        rows.append(np.concatenate([r, pad]))
    return np.concatenate(rows)


# (name, counts, page_size, level_count, max_iters, seed, dup)
LOD_PYRAMIDS = [
    ("reftest", (64, 50, 7), 64, 3, 10, 7, 1),
    ("mixed", (256, 201, 130, 33, 1, 0, 255, 96), 256, 4, 50, 7, 1),
    ("dups", (120, 64), 128, 3, 50, 11, 3),
]
# the C2-size page (one page of 2048 records, 2 levels): hash only
LOD_BIG = ("big", (2048,), 2048, 2, 50, 7, 1)
