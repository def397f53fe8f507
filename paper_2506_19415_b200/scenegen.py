"""Direct synthetic paged-scene generator ("city blocks") for the benchmark
configurations.

The reference's offline preprocessing (mesh -> paging -> k-means LOD) cannot
build million-record scenes in reasonable time, so this module writes the
paged ``.vms`` format directly, with a known structure:

* a grid of box buildings; each vertical facade is split into
  ``cols x rows`` square patches and every patch is one page of
  ``page_size`` live records scattered on the patch plane;
* the proxy mesh is one quad (two triangles) per page exactly on its patch,
  plus a page-0 ground quad (occludes, carries no page), so visibility
  culling sees real building-on-building occlusion;
* page links join patches whose rectangles touch (same facade neighbours
  and facades meeting at a building corner), sorted per page as the
  reference stores them (pkg/src/vmsplat/pipeline.py:100-105);
* LOD level k+1 of a page merges consecutive record pairs of level k (records
  are Morton-ordered on the patch, so pairs are spatial neighbours) with the
  attribute merge rule of pkg/src/vmsplat/lod.py:134-154 (means, hemisphere
  aligned quaternion mean, scale x 2^(1/3)).

Records follow pkg/src/vmsplat/synthetic.py:20-35 (random unit quaternions,
lognormal scales, opacity U(0.55, 0.95), smooth colour field in the DC term)
with all 45 higher SH coefficients non-zero (N(0, 0.02)).  Everything is a
pure function of the arguments and the seed.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from paper_2506_19415_b200.camera_path import CameraPath, Checkpoint
from paper_2506_19415_b200.gaussians import RECORD_SIZE
from paper_2506_19415_b200.scene_io import SceneFile, SceneWriter

SH_C0 = 0.28209479177387814
SCALE_FACTOR = 2.0 ** (1.0 / 3.0)


@dataclass(frozen=True)
class CityLayout:
    n_pages: int
    page_size: int = 2048
    levels: int = 3
    cols: int = 2          # patches across a facade
    rows: int = 5          # patches up a facade
    patch: float = 5.0     # patch edge (scene units)
    street: float = 8.0    # gap between buildings
    scale: float = 0.07    # median Gaussian std-dev
    seed: int = 0

    @property
    def width(self) -> float:
        return self.cols * self.patch

    @property
    def height(self) -> float:
        return self.rows * self.patch

    @property
    def pages_per_building(self) -> int:
        return 4 * self.cols * self.rows

    @property
    def n_buildings(self) -> int:
        return -(-self.n_pages // self.pages_per_building)

    @property
    def grid(self) -> int:
        return int(math.ceil(math.sqrt(self.n_buildings)))

    @property
    def spacing(self) -> float:
        return self.width + self.street


def _patches(lay: CityLayout):
    """Per page: (origin, u axis, v axis, normal) of its patch, building id."""
    out = []
    W, P = lay.width, lay.patch
    for b in range(lay.n_buildings):
        gi, gj = b % lay.grid, b // lay.grid
        x0, z0 = gi * lay.spacing, gj * lay.spacing
        # facades: (corner, along-facade unit, outward normal); up is -Y
        facades = [
            (np.array([x0, 0.0, z0]), np.array([1.0, 0, 0]), np.array([0, 0, -1.0])),
            (np.array([x0 + W, 0.0, z0]), np.array([0, 0, 1.0]), np.array([1.0, 0, 0])),
            (np.array([x0 + W, 0.0, z0 + W]), np.array([-1.0, 0, 0]), np.array([0, 0, 1.0])),
            (np.array([x0, 0.0, z0 + W]), np.array([0, 0, -1.0]), np.array([-1.0, 0, 0])),
        ]
        for corner, along, normal in facades:
            for r in range(lay.rows):
                for c in range(lay.cols):
                    origin = corner + along * (c * P) + np.array([0.0, -(r * P), 0.0])
                    out.append((origin, along * P, np.array([0.0, -P, 0.0]), normal, b))
                    if len(out) == lay.n_pages:
                        return out
    return out


def _morton2(u, v):
    def spread(x):
        x = x.astype(np.uint64) & np.uint64(0xFFFF)
        x = (x | (x << np.uint64(8))) & np.uint64(0x00FF00FF)
        x = (x | (x << np.uint64(4))) & np.uint64(0x0F0F0F0F)
        x = (x | (x << np.uint64(2))) & np.uint64(0x33333333)
        x = (x | (x << np.uint64(1))) & np.uint64(0x55555555)
        return x
    return spread(u) | (spread(v) << np.uint64(1))


def _page_records(lay: CityLayout, page_index: int, patch) -> np.ndarray:
    origin, du, dv, normal, _ = patch
    n = lay.page_size
    rng = np.random.default_rng([lay.seed, page_index])
    u = rng.uniform(0.0, 1.0, n)
    v = rng.uniform(0.0, 1.0, n)
    order = np.argsort(_morton2(np.minimum(u * 65536, 65535), np.minimum(v * 65536, 65535)),
                       kind="stable")
    u, v = u[order], v[order]
    off = rng.normal(0.0, 0.04, n)
    pos = origin + u[:, None] * du + v[:, None] * dv + off[:, None] * normal
    rec = np.zeros((n, RECORD_SIZE), dtype=np.float32)
    rec[:, 0:3] = pos
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    rec[:, 3:7] = q
    rec[:, 7:10] = np.exp(rng.normal(np.log(lay.scale), 0.25, size=(n, 3)))
    rec[:, 10] = rng.uniform(0.55, 0.95, n)
    col = 0.5 + 0.35 * np.sin(pos * np.array([0.23, 0.37, 0.19]) + np.array([0.0, 2.1, 4.2]))
    col += rng.normal(scale=0.03, size=(n, 3))
    rec[:, 11:14] = (np.clip(col, 0.05, 0.95) - 0.5) / SH_C0
    rec[:, 14:59] = rng.normal(scale=0.02, size=(n, 45))
    return rec


def merge_pairs(rec: np.ndarray) -> np.ndarray:
    """Merge consecutive record pairs (lod.merge_cluster rule for 2 members)."""
    a = rec[0::2].astype(np.float64)
    b = rec[1::2].astype(np.float64)
    out = np.empty_like(a)
    out[:, 0:3] = 0.5 * (a[:, 0:3] + b[:, 0:3])
    qa, qb = a[:, 3:7], b[:, 3:7].copy()
    flip = np.einsum("ij,ij->i", qb, qa) < 0
    qb[flip] *= -1.0
    q = 0.5 * (qa + qb)
    nrm = np.linalg.norm(q, axis=1, keepdims=True)
    out[:, 3:7] = np.where(nrm < 1e-6, qa, q / np.where(nrm < 1e-6, 1.0, nrm))
    out[:, 7:10] = 0.5 * (a[:, 7:10] + b[:, 7:10]) * SCALE_FACTOR
    out[:, 10:] = 0.5 * (a[:, 10:] + b[:, 10:])
    return out.astype(np.float32)


def _mesh_and_links(lay: CityLayout, patches):
    n = len(patches)
    verts = np.zeros((4 * n + 4, 3), dtype=np.float32)
    faces = np.zeros((2 * n + 2, 3), dtype=np.uint32)
    face_page = np.zeros(2 * n + 2, dtype=np.uint32)
    lo = np.zeros((n, 3))
    hi = np.zeros((n, 3))
    for p, (o, du, dv, _, _) in enumerate(patches):
        corners = np.stack([o, o + du, o + du + dv, o + dv])
        verts[4 * p:4 * p + 4] = corners
        faces[2 * p] = (4 * p, 4 * p + 1, 4 * p + 2)
        faces[2 * p + 1] = (4 * p, 4 * p + 2, 4 * p + 3)
        face_page[2 * p:2 * p + 2] = p + 1
        lo[p] = corners.min(axis=0)
        hi[p] = corners.max(axis=0)
    # ground quad (page 0): occludes what lies below street level
    ext = lay.grid * lay.spacing
    g0 = 4 * n
    verts[g0:g0 + 4] = [[-lay.street, 0.0, -lay.street], [ext, 0.0, -lay.street],
                        [ext, 0.0, ext], [-lay.street, 0.0, ext]]
    faces[2 * n] = (g0, g0 + 2, g0 + 1)
    faces[2 * n + 1] = (g0, g0 + 3, g0 + 2)
    # links: patches of the same building whose boxes touch
    bid = np.array([pt[4] for pt in patches])
    offsets = np.zeros(n + 1, dtype=np.uint32)
    targets = []
    eps = 1e-3 * lay.patch
    for p in range(n):
        same = np.flatnonzero(bid == bid[p])
        touch = np.all((lo[same] <= hi[p] + eps) & (hi[same] >= lo[p] - eps), axis=1)
        t = [int(q) + 1 for q in same[touch] if q != p]
        targets.extend(sorted(t))
        offsets[p + 1] = offsets[p] + len(t)
    return verts, faces, face_page, offsets, np.asarray(targets, dtype=np.uint32)


def city_metadata(lay: CityLayout) -> SceneFile:
    """SceneFile with everything except the record array."""
    patches = _patches(lay)
    verts, faces, face_page, off, tgt = _mesh_and_links(lay, patches)
    ext = lay.grid * lay.spacing
    lo = np.array([0.0, -lay.height, 0.0])
    hi = np.array([ext - lay.street, 0.0, ext - lay.street])
    center = (0.5 * (lo + hi)).astype(np.float32)
    half = float(max((hi - lo).max() * 0.5, 1e-6))
    return SceneFile(stage="full" if lay.levels > 1 else "paged", page_size=lay.page_size,
                     lod_levels=lay.levels, page_counts=[len(patches)] * lay.levels,
                     center=center, half_extent=half, vertices=verts, faces=faces,
                     face_page=face_page, link_offsets=off, link_targets=tgt,
                     gaussians=np.zeros((0, RECORD_SIZE), dtype=np.float32))


def _level_blocks(lay: CityLayout, patches, first: int, last: int):
    """Records of pages [first, last) for every level: list per level."""
    per_level = [[] for _ in range(lay.levels)]
    for p in range(first, last):
        rec = _page_records(lay, p, patches[p])
        for k in range(lay.levels):
            per_level[k].append(rec)
            if k + 1 < lay.levels:
                rec = merge_pairs(rec)
    return [np.concatenate(x, axis=0) for x in per_level]


def city_scene(lay: CityLayout) -> SceneFile:
    """In-memory scene (small layouts: tests and smoke runs)."""
    sc = city_metadata(lay)
    patches = _patches(lay)
    blocks = _level_blocks(lay, patches, 0, len(patches))
    sc.gaussians = np.ascontiguousarray(np.concatenate(blocks, axis=0))
    sc.validate()
    return sc


def write_city(path, lay: CityLayout, pages_per_batch: int = 64) -> None:
    """Stream-write a city scene level block by level block (bounded RAM)."""
    sc = city_metadata(lay)
    patches = _patches(lay)
    n = len(patches)
    with SceneWriter(path, sc) as w:
        for k in range(lay.levels):
            for a in range(0, n, pages_per_batch):
                b = min(n, a + pages_per_batch)
                rows = []
                for p in range(a, b):
                    rec = _page_records(lay, p, patches[p])
                    for _ in range(k):
                        rec = merge_pairs(rec)
                    rows.append(rec)
                w.write_records(np.concatenate(rows, axis=0))


def street_path(lay: CityLayout, frames: int = 120, width: int = 1920, height: int = 1080,
                eye: float = 3.0, fov_deg: float = 90.0) -> CameraPath:
    """Fly down the first street between building columns 0 and 1, then turn
    90 degrees into the next cross street; ``frames`` frames in total."""
    sx = lay.width + 0.5 * lay.street           # centre of the first street
    z_end = min(lay.grid, 3) * lay.spacing - 0.5 * lay.street
    turn_x = sx + 2 * lay.spacing
    yaw = lambda a: (math.cos(a / 2), 0.0, math.sin(a / 2), 0.0)  # noqa: E731
    cps = (
        Checkpoint((sx, -eye, -lay.street), yaw(0.0)),
        Checkpoint((sx, -eye, z_end), yaw(0.0)),
        Checkpoint((sx + 0.5 * lay.street, -eye, z_end + 0.2), yaw(math.pi / 2)),
        Checkpoint((turn_x, -eye, z_end + 0.2), yaw(math.pi / 2)),
    )
    probe = CameraPath(cps, speed=1.0, fps=1.0, fov_deg=fov_deg, width=width, height=height)
    fps = (frames - 1) / probe.duration + 1e-9
    return CameraPath(cps, speed=1.0, fps=fps, fov_deg=fov_deg, width=width, height=height)


# Named configurations (BASELINE.json "configs").
C2 = CityLayout(n_pages=1000, page_size=2048, levels=3)      # 2.05M records, 3 LOD levels
C3 = CityLayout(n_pages=10000, page_size=2048, levels=4)     # 20.5M records, 4 LOD levels
