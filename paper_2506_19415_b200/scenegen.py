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
    return _patches_from(lay, 0, lay.n_pages)


def _patches_from(lay: CityLayout, first_building: int, last_page: int):
    """Patches of pages [first_building * pages_per_building, last_page)."""
    out = []
    W, P = lay.width, lay.patch
    cap = last_page - first_building * lay.pages_per_building
    for b in range(first_building, lay.n_buildings):
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
                    if len(out) == cap:
                        return out
    return out


def _patches_range(lay: CityLayout, first: int, last: int):
    """_patches(lay)[first:last] without building the whole list."""
    b0 = first // lay.pages_per_building
    return _patches_from(lay, b0, last)[first - b0 * lay.pages_per_building:]


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
    # links: patches of the same building whose boxes touch (a building's
    # pages are contiguous, so each building is one small dense block)
    bid = np.array([pt[4] for pt in patches])
    offsets = np.zeros(n + 1, dtype=np.uint32)
    targets = []
    eps = 1e-3 * lay.patch
    starts = np.flatnonzero(np.r_[True, bid[1:] != bid[:-1]])
    ends = np.r_[starts[1:], n]
    for a, b in zip(starts, ends):
        blo, bhi = lo[a:b], hi[a:b]
        touch = np.all((blo[None, :, :] <= bhi[:, None, :] + eps)
                       & (bhi[None, :, :] >= blo[:, None, :] - eps), axis=2)
        for i in range(b - a):
            t = np.flatnonzero(touch[i])
            t = t[t != i] + a + 1   # ascending page ids, self excluded
            targets.append(t)
            offsets[a + i + 1] = offsets[a + i] + len(t)
    targets = np.concatenate(targets).astype(np.uint32) if targets else np.zeros(0, np.uint32)
    return verts, faces, face_page, offsets, targets


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


def _write_pages(job):
    """Worker of write_city: every level of pages [first, last) straight into
    the file's record section (page offsets are pure arithmetic)."""
    path, gaus_off, lay, first, last = job
    patches = _patches_range(lay, first, last)
    level_start = 0
    mm = np.memmap(path, dtype="<f4", mode="r+", offset=gaus_off,
                   shape=(lay.n_pages * sum(lay.page_size >> k for k in range(lay.levels)),
                          RECORD_SIZE))
    recs = [_page_records(lay, p, patches[p - first]) for p in range(first, last)]
    for k in range(lay.levels):
        per = lay.page_size >> k
        mm[level_start + first * per: level_start + last * per] = np.concatenate(recs, axis=0)
        level_start += lay.n_pages * per
        if k + 1 < lay.levels:
            recs = [merge_pairs(r) for r in recs]
    mm.flush()
    del mm
    return last - first


def write_city(path, lay: CityLayout, workers: int | None = None,
               pages_per_job: int = 256) -> None:
    """Write a city scene: metadata first, then every page's records at all
    levels, generated in parallel by ``workers`` processes (default: the
    usable cores) that write disjoint row ranges of the preallocated record
    section.  The bytes are independent of ``workers`` (each page's records
    are a pure function of the layout, the seed and the page index)."""
    import os

    from paper_2506_19415_b200.scene_io import preallocate_scene

    sc = city_metadata(lay)
    gaus_off = preallocate_scene(path, sc)
    n = lay.n_pages
    jobs = [(str(path), gaus_off, lay, a, min(n, a + pages_per_job))
            for a in range(0, n, pages_per_job)]
    if workers is None:
        try:
            workers = len(os.sched_getaffinity(0))
        except AttributeError:  # pragma: no cover
            workers = os.cpu_count() or 1
    workers = max(1, min(workers, len(jobs)))
    if workers == 1:
        done = sum(_write_pages(j) for j in jobs)
    else:
        import multiprocessing as mp

        with mp.get_context("fork").Pool(workers) as pool:
            done = sum(pool.imap_unordered(_write_pages, jobs))
    assert done == n


def street_path(lay: CityLayout, frames: int = 120, width: int = 1920, height: int = 1080,
                eye: float = 3.0, fov_deg: float = 90.0, blocks: int = 3) -> CameraPath:
    """Fly down the first street between building columns 0 and 1 for
    ``blocks`` blocks, then turn 90 degrees into the next cross street;
    ``frames`` frames in total."""
    sx = lay.width + 0.5 * lay.street           # centre of the first street
    z_end = min(lay.grid, blocks) * lay.spacing - 0.5 * lay.street
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
# C4 on the GPU boxes of this project: 196 GB of host DRAM and 80 GB of free
# disk cannot hold the 800M-record (189 GB) scene of BASELINE configs[3], so
# the out-of-core configuration is the largest LOD city that fits host DRAM
# with headroom: 170,000 pages x 2048 records at level 0 (348.2M) plus LOD
# levels 1-2 (174.1M + 87.0M) = 609.3M records, 143.8 GB, written to tmpfs
# and paged from there.
C4 = CityLayout(n_pages=170000, page_size=2048, levels=3)
