"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference per-frame path (`VmSession.render_frame`,
pkg/src/vmsplat/runtime.py:436-489) in NumPy, with the three hot loops in the
C restatement ``oracle/kernels.c`` (or, when built, the reference's own
Cython core compiled into ``oracle/_ref``).

Parity of this restatement is PINNED against the live reference: the script
``tests/golden/make_golden.py`` imports the reference package in the build
container and records its outputs into ``tests/golden/*.npz``; the CPU test
``tests/test_oracle_golden.py`` checks this module against them.

Who may import this module: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` — only as the
checker or the CPU baseline, never as a product path.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from oracle import ckernels

# -- constants (pkg/src/vmsplat/render.py:23-44, kernels/_core.pyx:20-21) ----
LOW_PASS = 0.3
MIN_DET = 1e-12
EXTENT_SIGMA = 3.0
SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
         -1.0925484305920792, 0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
         0.3731763325901154, -0.4570457994644658, 1.445305721320277,
         -0.5900435899266435)
RECORD_SIZE = 59
U32_MAX = 0xFFFFFFFF


class OracleInvariant(Exception):
    """Mirror of vmsplat.errors.InvariantViolation (errors.py:24-25)."""


# -- gaussians.quat_to_matrix (pkg/src/vmsplat/gaussians.py:76-96) ----------
def quat_rot(q):
    q = np.asarray(q, dtype=np.float64)
    one = q.ndim == 1
    q = q.reshape(-1, 4)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    m = np.empty((len(q), 3, 3))
    m[:, 0, 0] = 1 - 2 * (y * y + z * z)
    m[:, 0, 1] = 2 * (x * y - w * z)
    m[:, 0, 2] = 2 * (x * z + w * y)
    m[:, 1, 0] = 2 * (x * y + w * z)
    m[:, 1, 1] = 1 - 2 * (x * x + z * z)
    m[:, 1, 2] = 2 * (y * z - w * x)
    m[:, 2, 0] = 2 * (x * z - w * y)
    m[:, 2, 1] = 2 * (y * z + w * x)
    m[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return m[0] if one else m


# -- render.Camera (pkg/src/vmsplat/render.py:47-101) -----------------------
@dataclass(frozen=True)
class OCamera:
    position: tuple
    orientation: tuple
    fov_y: float
    width: int
    height: int
    near: float = 0.05

    @property
    def focal(self):
        return (self.height / 2.0) / np.tan(self.fov_y / 2.0)

    def rot(self):
        return quat_rot(np.asarray(self.orientation, dtype=np.float64))

    def to_view(self, pts):
        p = np.atleast_2d(np.asarray(pts, dtype=np.float64))
        return (p - np.asarray(self.position, dtype=np.float64)) @ self.rot()

    def to_pixels(self, view):
        f = self.focal
        out = np.empty_like(view)
        out[:, 0] = f * view[:, 0] / view[:, 2] + self.width / 2.0
        out[:, 1] = f * view[:, 1] / view[:, 2] + self.height / 2.0
        out[:, 2] = 1.0 / view[:, 2]
        return out

    def scaled(self, s):
        return OCamera(self.position, self.orientation, self.fov_y,
                       max(1, int(round(self.width * s))),
                       max(1, int(round(self.height * s))), self.near)


def as_ocam(cam) -> OCamera:
    return OCamera(tuple(cam.position), tuple(cam.orientation), float(cam.fov_y),
                   int(cam.width), int(cam.height), float(cam.near))


# -- render.evaluate_sh (pkg/src/vmsplat/render.py:104-135) -----------------
def sh_rgb(coeffs, dirs):
    c = np.asarray(coeffs, dtype=np.float64).reshape(-1, 16, 3)
    d = np.asarray(dirs, dtype=np.float64).reshape(-1, 3)
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    xx, yy, zz = x * x, y * y, z * z
    xy, yz, xz = x * y, y * z, x * z
    b = np.empty((len(d), 16))
    b[:, 0] = SH_C0
    b[:, 1] = -SH_C1 * y
    b[:, 2] = SH_C1 * z
    b[:, 3] = -SH_C1 * x
    b[:, 4] = SH_C2[0] * xy
    b[:, 5] = SH_C2[1] * yz
    b[:, 6] = SH_C2[2] * (2.0 * zz - xx - yy)
    b[:, 7] = SH_C2[3] * xz
    b[:, 8] = SH_C2[4] * (xx - yy)
    b[:, 9] = SH_C3[0] * y * (3.0 * xx - yy)
    b[:, 10] = SH_C3[1] * xy * z
    b[:, 11] = SH_C3[2] * y * (4.0 * zz - xx - yy)
    b[:, 12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy)
    b[:, 13] = SH_C3[4] * x * (4.0 * zz - xx - yy)
    b[:, 14] = SH_C3[5] * z * (xx - yy)
    b[:, 15] = SH_C3[6] * x * (xx - 3.0 * yy)
    return np.maximum(0.5 + np.einsum("nk,nkc->nc", b, c), 0.0)


# -- render.compute_keys / depth_order (render.py:138-152, 235-239) ---------
def keys_of(records, cam):
    records = np.asarray(records, dtype=np.float32)
    if len(records) == 0:
        return np.zeros(0, np.uint32), np.zeros(0, np.int64)
    view = cam.to_view(records[:, 0:3].astype(np.float64))
    live = (records[:, 10] > 0.0) & (view[:, 2] > cam.near)
    idx = np.flatnonzero(live).astype(np.int64)
    return view[idx, 2].astype(np.float32).view(np.uint32), idx


def order_of(records, cam, kern=None):
    kern = kern or ckernels
    k, idx = keys_of(records, cam)
    _, order = kern.radix_sort_pairs(k, idx)
    return order


# -- render.project_records (render.py:155-220) -----------------------------
def project(records, cam):
    records = np.asarray(records, dtype=np.float32)
    m = len(records)
    if m == 0:
        z = np.zeros
        return (z((0, 2)), z((0, 3)), z((0, 3), np.float32), z(0, np.float32),
                z((0, 4), np.int32), z(0, bool))
    mu = records[:, 0:3].astype(np.float64)
    rot = quat_rot(records[:, 3:7].astype(np.float64))
    scale = records[:, 7:10].astype(np.float64)
    alphas = records[:, 10]
    sh = records[:, 11:].reshape(m, 16, 3)
    crot = cam.rot()
    pos = np.asarray(cam.position, dtype=np.float64)
    view = (mu - pos) @ crot
    tx, ty, tz = view[:, 0], view[:, 1], view[:, 2]
    f = cam.focal
    ms = rot * scale[:, None, :]
    cov3 = ms @ ms.transpose(0, 2, 1)
    j = np.zeros((m, 2, 3))
    j[:, 0, 0] = f / tz
    j[:, 0, 2] = -f * tx / (tz * tz)
    j[:, 1, 1] = f / tz
    j[:, 1, 2] = -f * ty / (tz * tz)
    jw = j @ crot.T
    cov2 = jw @ cov3 @ jw.transpose(0, 2, 1)
    a = cov2[:, 0, 0] + LOW_PASS
    b = cov2[:, 0, 1]
    c = cov2[:, 1, 1] + LOW_PASS
    det = a * c - b * b
    kept = det >= MIN_DET
    with np.errstate(divide="ignore", invalid="ignore"):
        conics = np.column_stack((c / det, -b / det, a / det))
    mid = 0.5 * (a + c)
    lam = mid + np.sqrt(np.maximum(0.25 * (a - c) ** 2 + b * b, 0.0))
    rad = EXTENT_SIGMA * np.sqrt(np.maximum(lam, 0.0))
    cx = f * tx / tz + cam.width / 2.0
    cy = f * ty / tz + cam.height / 2.0
    x0 = np.maximum(np.floor(cx - rad - 0.5), 0.0)
    x1 = np.minimum(np.ceil(cx + rad + 0.5), cam.width)
    y0 = np.maximum(np.floor(cy - rad - 0.5), 0.0)
    y1 = np.minimum(np.ceil(cy + rad + 0.5), cam.height)
    kept &= (x1 > x0) & (y1 > y0)
    vd = mu - pos
    nrm = np.linalg.norm(vd, axis=1, keepdims=True)
    vd = vd / np.where(nrm > 0, nrm, 1.0)
    colors = sh_rgb(sh, vd).astype(np.float32)
    centers = np.column_stack((cx, cy))
    bounds = np.column_stack((x0, x1, y0, y1)).astype(np.int32)
    k = np.flatnonzero(kept)
    return centers[k], conics[k], colors[k], alphas[k].astype(np.float32), bounds[k], kept


def composite_in_order(records, order, cam, kern=None):
    """render.composite_ordered (render.py:242-248)."""
    kern = kern or ckernels
    srt = np.asarray(records, dtype=np.float32)[order]
    centers, conics, colors, alphas, bounds, _ = project(srt, cam)
    img = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
    kern.composite_splats(centers, conics, colors, alphas, bounds, img)
    return img


def render_flat(records, cam, kern=None):
    """render.render_records (render.py:251-253)."""
    return composite_in_order(records, order_of(records, cam, kern), cam, kern)


def render_window(records, cam, window, kern=None, chunk=1 << 20):
    """Pixels [x0, x1) x [y0, y1) of render_records(records, cam)
    (render.py:251-253) without projecting every record: SURVEY 8(c)(ii).

    Order: keys and the stable sort over ALL records, exactly as
    render_records.  Selection: a record can only touch the window if its
    projected bbox does; its bbox radius is 3*sqrt(lambda_max(cov2 + 0.3 I))
    with lambda_max(cov2) <= ||J||_F^2 * max(scale)^2 (the camera rotation
    and the record's rotation are orthogonal), so records whose centre lies
    farther than that bound (+2 px) from the window are dropped before the
    projection.  The survivors are projected (in sorted order) and the ones
    whose exact bounds meet the window are composited into a window-sized
    image with centres shifted by the window origin (an exact f64 shift of an
    f32 centre) and bounds clipped to the window.  Each window pixel then sees
    exactly the splats, in exactly the order, that render_records gives it."""
    kern = kern or ckernels
    records = np.asarray(records, dtype=np.float32)
    x0, x1, y0, y1 = (int(v) for v in window)
    order = order_of(records, cam, kern)
    if not len(order):
        return np.zeros((y1 - y0, x1 - x0, 3), np.float32), 0
    f = cam.focal
    pos = np.asarray(cam.position, dtype=np.float64)
    crot = cam.rot()
    keep = []
    for a in range(0, len(order), chunk):
        idx = order[a:a + chunk]
        r = records[idx]
        v = (r[:, 0:3].astype(np.float64) - pos) @ crot
        z = v[:, 2]
        cx = f * v[:, 0] / z + cam.width / 2.0
        cy = f * v[:, 1] / z + cam.height / 2.0
        smax = np.max(r[:, 7:10].astype(np.float64), axis=1)
        jf2 = 2.0 * f * f / (z * z) + f * f * (v[:, 0] ** 2 + v[:, 1] ** 2) / (z ** 4)
        rad = 3.0 * np.sqrt(jf2 * smax * smax * 1.0001 + LOW_PASS) + 2.0
        near = ((cx + rad >= x0) & (cx - rad <= x1) & (cy + rad >= y0) & (cy - rad <= y1))
        keep.append(idx[near])
    sel = np.concatenate(keep)
    centers, conics, colors, alphas, bounds, _ = project(records[sel], cam)
    b = bounds
    hit = (b[:, 0] < x1) & (b[:, 1] > x0) & (b[:, 2] < y1) & (b[:, 3] > y0)
    bb = b[hit].copy()
    bb[:, 0] = np.maximum(bb[:, 0], x0)
    bb[:, 1] = np.minimum(bb[:, 1], x1)
    bb[:, 2] = np.maximum(bb[:, 2], y0)
    bb[:, 3] = np.minimum(bb[:, 3], y1)
    full = np.zeros((cam.height, cam.width, 3), np.float32)
    kern.composite_splats(centers[hit], conics[hit], colors[hit], alphas[hit], bb, full)
    img = np.ascontiguousarray(full[y0:y1, x0:x1])
    return img, int(hit.sum())


# -- render._clip_near / render_visibility (render.py:256-307) --------------
def clip_near(tv, near):
    inside = tv[:, 2] > near
    n_in = int(inside.sum())
    if n_in == 0:
        return []
    if n_in == 3:
        return [tv]
    poly = []
    for i in range(3):
        a, b = tv[i], tv[(i + 1) % 3]
        if inside[i]:
            poly.append(a)
        if inside[i] != inside[(i + 1) % 3]:
            t = (near - a[2]) / (b[2] - a[2])
            poly.append(a + t * (b - a))
    return [np.stack([poly[0], poly[i], poly[i + 1]]) for i in range(1, len(poly) - 1)]


def clipped_triangles(vertices, faces, face_page, cam):
    """Per-face clip + project, emitted in (face, fan) order
    (render.py:288-304).  Faces entirely beyond the near plane are projected
    in one vectorised pass (elementwise, the same operations per vertex as
    the per-face loop); only faces crossing the plane take the clip loop."""
    faces = np.asarray(faces)
    if not len(faces):
        return np.zeros((0, 3, 3)), np.zeros(0, np.uint32)
    view = cam.to_view(np.asarray(vertices, dtype=np.float64))
    tv = view[faces]                                   # (F, 3, 3)
    n_in = (tv[:, :, 2] > cam.near).sum(axis=1)
    full = n_in == 3
    part = np.flatnonzero((n_in > 0) & ~full)
    pieces = {}
    for fi in part:
        pieces[int(fi)] = [cam.to_pixels(cl) for cl in clip_near(tv[fi], cam.near)]
    counts = full.astype(np.int64)
    for fi, lst in pieces.items():
        counts[fi] = len(lst)
    total = int(counts.sum())
    if total == 0:
        return np.zeros((0, 3, 3)), np.zeros(0, np.uint32)
    start = np.cumsum(counts) - counts
    tris = np.empty((total, 3, 3))
    ids = np.empty(total, np.uint32)
    fidx = np.flatnonzero(full)
    if len(fidx):
        tris[start[fidx]] = cam.to_pixels(tv[fidx].reshape(-1, 3)).reshape(-1, 3, 3)
        ids[start[fidx]] = np.asarray(face_page)[fidx]
    for fi, lst in pieces.items():
        for k, t in enumerate(lst):
            tris[start[fi] + k] = t
            ids[start[fi] + k] = face_page[fi]
    return np.ascontiguousarray(tris), ids


def visibility(vertices, faces, face_page, cam, kern=None):
    kern = kern or ckernels
    idimg = np.zeros((cam.height, cam.width), dtype=np.uint32)
    invz = np.zeros((cam.height, cam.width), dtype=np.float64)
    tris, ids = clipped_triangles(vertices, faces, face_page, cam)
    if len(tris):
        kern.rasterize_triangles(tris, ids, idimg, invz)
    with np.errstate(divide="ignore"):
        depth = np.where(invz > 0.0, 1.0 / np.where(invz > 0.0, invz, 1.0), np.inf)
    return idimg, depth.astype(np.float64)


# -- runtime depth codec, reduce, LOD (runtime.py:26-158) -------------------
def enc_depth(d):
    return U32_MAX - int(np.float32(d).view(np.uint32))


def dec_depth(e):
    return float(np.uint32(U32_MAX - int(e)).view(np.float32))


def enc_depth_arr(d):
    return np.uint32(U32_MAX) - np.asarray(d, dtype=np.float32).view(np.uint32)


@dataclass
class ORequired:
    depths: np.ndarray
    direct: np.ndarray

    def ids(self):
        return np.flatnonzero(self.depths).astype(np.int64)


def link_lists(link_offsets, link_targets, page_count, enabled=True):
    out = [np.zeros(0, np.uint32)]
    for p in range(1, page_count + 1):
        if enabled:
            out.append(np.asarray(link_targets[link_offsets[p - 1]:link_offsets[p]], np.uint32))
        else:
            out.append(np.zeros(0, np.uint32))
    return out


def reduce_pages(page_img, depth_img, links):
    n = len(links) - 1
    flat = np.asarray(page_img).ravel().astype(np.int64)
    if flat.size and flat.max() > n:
        raise OracleInvariant(f"visibility page id {int(flat.max())} out of range (page count {n})")
    depths = np.zeros(n + 1, np.uint32)
    direct = np.zeros(n + 1, bool)
    live = flat != 0
    if live.any():
        np.maximum.at(depths, flat[live], enc_depth_arr(np.asarray(depth_img).ravel()[live]))
        direct[np.unique(flat[live])] = True
        base = depths.copy()
        for p in np.flatnonzero(direct):
            for q in links[p]:
                q = int(q)
                if q != p and base[p] > depths[q]:
                    depths[q] = base[p]
    return ORequired(depths, direct)


@dataclass
class OController:
    thresholds: np.ndarray
    step: float = 0.05
    band_low: float = 0.5
    band_high: float = 0.8
    step_min: float = 0.005
    step_max: float = 0.5
    window: int = 30
    last_dir: int = 0
    last_frame: int = -(10 ** 9)

    def __post_init__(self):
        self.thresholds = np.asarray(self.thresholds, dtype=np.float64)
        if np.any(np.diff(self.thresholds) <= 0):
            raise OracleInvariant("thresholds must be strictly increasing")


def init_thresholds(radius, levels):
    k = levels - 1
    return radius * np.power(2.0, np.arange(k) - (k - 1), dtype=np.float64)


def lod_of(enc, ctl):
    return int(np.count_nonzero(ctl.thresholds < dec_depth(enc)))


def adapt(ctl, usage, frame):
    if usage > ctl.band_high:
        direction = -1
    elif usage < ctl.band_low:
        direction = +1
    else:
        return
    if ctl.thresholds.size == 0:
        return
    if frame - ctl.last_frame <= ctl.window:
        factor = 1.01 if direction == ctl.last_dir else 0.99
        ctl.step = float(np.clip(ctl.step * factor, ctl.step_min, ctl.step_max))
    ctl.thresholds = ctl.thresholds * (1.0 + direction * ctl.step)
    ctl.last_dir = direction
    ctl.last_frame = frame


# -- runtime.PageTable / update_page_table (runtime.py:161-346) -------------
class OEntry:
    __slots__ = ("level", "last", "slots")

    def __init__(self):
        self.level, self.last, self.slots = -1, -1, []


class OTable:
    def __init__(self, capacity):
        if capacity < 1:
            raise OracleInvariant("page table needs at least one entry")
        self.entries = [OEntry() for _ in range(capacity)]
        self.resident = {}

    @property
    def capacity(self):
        return len(self.entries)

    def occupied(self):
        return sum(1 for e in self.entries if e.level >= 0)

    def usage(self):
        return self.occupied() / self.capacity

    def counts(self, levels):
        c = [0] * levels
        for ei, _ in self.resident.values():
            c[self.entries[ei].level] += 1
        return tuple(c)

    def check(self):
        seen = {}
        for ei, e in enumerate(self.entries):
            if e.level < 0:
                if e.slots:
                    raise OracleInvariant(f"empty entry {ei} has slots")
                continue
            if len(e.slots) != (1 << e.level):
                raise OracleInvariant(f"entry {ei} slot count mismatch")
            for si, pid in enumerate(e.slots):
                if pid:
                    if pid in seen:
                        raise OracleInvariant(f"page {pid} resident twice")
                    seen[pid] = (ei, si)
        if seen != self.resident:
            raise OracleInvariant("residency map out of sync with entries")

    def alloc(self, level, protected):
        for ei, e in enumerate(self.entries):
            if e.level == level:
                for si, pid in enumerate(e.slots):
                    if pid == 0:
                        return ei, si
        for ei, e in enumerate(self.entries):
            if e.level < 0:
                e.level, e.slots = level, [0] * (1 << level)
                return ei, 0
        best = None
        for ei, e in enumerate(self.entries):
            if ei in protected:
                continue
            key = (e.last, ei)
            if best is None or key < best:
                best = key
        if best is None:
            return None
        ei = best[1]
        e = self.entries[ei]
        for pid in e.slots:
            if pid:
                del self.resident[pid]
        e.level, e.slots = level, [0] * (1 << level)
        return ei, 0

    def place(self, pid, ei, si, frame):
        old = self.resident.get(pid)
        e = self.entries[ei]
        e.slots[si] = pid
        e.last = frame
        self.resident[pid] = (ei, si)
        if old is not None and old != (ei, si):
            oe = self.entries[old[0]]
            oe.slots[old[1]] = 0
            if not any(oe.slots):
                oe.level, oe.slots = -1, []


def update_table(table, req, ctl, frame, budget):
    """Returns (plan [(pid, level, entry, slot)], missing)."""
    ids = req.ids()
    protected = set()
    work = []
    for pid in ids:
        pid = int(pid)
        enc = int(req.depths[pid])
        level = lod_of(enc, ctl)
        loc = table.resident.get(pid)
        if loc is not None:
            table.entries[loc[0]].last = frame
            protected.add(loc[0])
            if table.entries[loc[0]].level != level:
                work.append((2, -enc, pid, level))
        else:
            work.append((0 if req.direct[pid] else 1, -enc, pid, level))
    work.sort()
    plan = []
    spent = 0.0
    for _, _, pid, level in work:
        cost = 1.0 / (1 << level)
        if spent + cost > budget:
            break
        got = table.alloc(level, protected)
        if got is None:
            continue
        ei, si = got
        table.place(pid, ei, si, frame)
        protected.add(ei)
        plan.append((pid, level, ei, si))
        spent += cost
    missing = sum(1 for pid in ids if int(pid) not in table.resident)
    return plan, missing


# -- scene page arithmetic (scene_io.py:144-161) ----------------------------
def page_rows(page_size, page_counts, level, pid):
    per = page_size >> level
    start = sum(page_counts[k] * (page_size >> k) for k in range(level))
    start += (pid - 1) * per
    return start, start + per


class OSession:
    """VmSession (runtime.py:393-489) over plain arrays.

    ``scene`` must expose page_size, lod_levels, page_counts, half_extent,
    vertices, faces, face_page, link_offsets, link_targets, gaussians.
    """

    def __init__(self, scene, buffer_pages=500, staging_pages=40, vis_scale=0.25,
                 band=(0.5, 0.8), step=0.05, lod_enabled=True, links_enabled=True,
                 kern=None):
        if scene.page_count == 0:
            raise OracleInvariant("scene has no pages; run paging first")
        self.kern = kern or ckernels
        self.scene = scene
        self.vertices = np.asarray(scene.vertices).astype(np.float64)
        self.faces = np.asarray(scene.faces).astype(np.int32)
        self.face_page = np.asarray(scene.face_page).astype(np.uint32)
        self.links = link_lists(scene.link_offsets, scene.link_targets,
                                scene.page_count, links_enabled)
        levels = scene.lod_levels if lod_enabled else 1
        radius = scene.half_extent * np.sqrt(3.0)
        self.controller = OController(init_thresholds(radius, levels), step=step,
                                      band_low=band[0], band_high=band[1])
        self.lod_enabled = lod_enabled and levels > 1
        self.table = OTable(buffer_pages)
        self.page_size = scene.page_size
        self.buffer = np.zeros((buffer_pages * scene.page_size, RECORD_SIZE), np.float32)
        self.staging_pages = staging_pages
        self.vis_scale = vis_scale
        self.last_required = None
        self.last_plan = None

    def _slot_rows(self, ei, si, level):
        per = self.page_size >> level
        a = ei * self.page_size + si * per
        return a, a + per

    def resident_records(self):
        parts = []
        for pid in sorted(self.table.resident):
            ei, si = self.table.resident[pid]
            a, b = self._slot_rows(ei, si, self.table.entries[ei].level)
            parts.append(self.buffer[a:b])
        if not parts:
            return np.zeros((0, RECORD_SIZE), np.float32)
        return np.concatenate(parts, axis=0)

    def render_frame(self, camera, frame_index, want_image=True):
        cam = as_ocam(camera)
        sc = self.scene
        t0 = time.perf_counter()
        pimg, dimg = visibility(self.vertices, self.faces, self.face_page,
                                cam.scaled(self.vis_scale), self.kern)
        t1 = time.perf_counter()
        req = reduce_pages(pimg, dimg, self.links)
        t2 = time.perf_counter()
        plan, missing = update_table(self.table, req, self.controller, frame_index,
                                     self.staging_pages)
        t3 = time.perf_counter()
        copied = 0
        for pid, level, ei, si in plan:
            a, b = page_rows(sc.page_size, sc.page_counts, level, pid)
            rows = sc.gaussians[a:b]
            c, d = self._slot_rows(ei, si, level)
            self.buffer[c:d] = rows
            copied += rows.nbytes
        t4 = time.perf_counter()
        usage = self.table.usage()
        if self.lod_enabled:
            adapt(self.controller, usage, frame_index)
        records = self.resident_records()
        t5 = time.perf_counter()
        image = None
        order = order_of(records, cam, self.kern) if want_image else None
        t6 = time.perf_counter()
        if want_image:
            image = composite_in_order(records, order, cam, self.kern)
        t7 = time.perf_counter()
        self.last_required = req
        self.last_plan = plan
        stats = {
            "frame": frame_index,
            "required_pages": int(len(req.ids())),
            "resident_pages": int(len(self.table.resident)),
            "resident_per_level": self.table.counts(sc.lod_levels),
            "planned_copies": len(plan),
            "missing_pages": int(missing),
            "bytes_copied": int(copied),
            "usage": usage,
            "lod_step": self.controller.step,
            "thresholds": tuple(float(t) for t in self.controller.thresholds),
            "time_visibility": t1 - t0,
            "time_reduce": t2 - t1,
            "time_update": t3 - t2,
            "time_copy": (t4 - t3) + (t5 - t4),
            "time_sort": t6 - t5,
            "time_render": t7 - t6,
        }
        return image, stats


def stats_csv(stats_list):
    """harness._stats_rows byte format (pkg/src/vmsplat/harness.py:335-348)."""
    levels = len(stats_list[0]["resident_per_level"])
    lines = [",".join(["frame", "required", "missing", "bytes_copied", "usage"]
                      + [f"resident_l{k}" for k in range(levels)] + ["thresholds"])]
    for s in stats_list:
        row = [str(s["frame"]), str(s["required_pages"]), str(s["missing_pages"]),
               str(s["bytes_copied"]), repr(float(s["usage"]))]
        row += [str(c) for c in s["resident_per_level"]]
        row.append(";".join(repr(float(t)) for t in s["thresholds"]))
        lines.append(",".join(row))
    return "\n".join(lines) + "\n"


def ssim(a, b):
    """metrics.ssim (pkg/src/vmsplat/metrics.py:33-75): 11x11 Gaussian window
    (sigma 1.5), reflected borders, mean over interior pixels per channel,
    then over channels; K1 = 0.01, K2 = 0.03."""
    from scipy.ndimage import correlate

    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim == 2:
        a, b = a[:, :, None], b[:, :, None]
    r = np.arange(11, dtype=np.float64) - 5.0
    g = np.exp(-(r * r) / (2.0 * 1.5 * 1.5))
    k = np.outer(g, g)
    k /= k.sum()
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    h, w = a.shape[:2]
    vals = []
    for ch in range(a.shape[2]):
        x, y = a[:, :, ch], b[:, :, ch]
        mx, my = correlate(x, k, mode="reflect"), correlate(y, k, mode="reflect")
        xx = correlate(x * x, k, mode="reflect") - mx * mx
        yy = correlate(y * y, k, mode="reflect") - my * my
        xy = correlate(x * y, k, mode="reflect") - mx * my
        s = ((2.0 * mx * my + c1) * (2.0 * xy + c2)) / ((mx * mx + my * my + c1) * (xx + yy + c2))
        vals.append(float(np.mean(s[5:h - 5, 5:w - 5])))
    return float(np.mean(vals))


def psnr(a, b):
    d = np.asarray(a, np.float64) - np.asarray(b, np.float64)
    mse = float(np.mean(d * d))
    return math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)
