"""Renderer API of the reference (pkg/src/vmsplat/render.py), GPU-backed.

Camera convention (render.py:1-11): +Z forward, +X right, +Y down, principal
point at the image centre, f = (h/2)/tan(fov_y/2), pixel (x, y) samples at
(x + 0.5, y + 0.5).  ``Camera`` is host-side pose bookkeeping exactly as in
the reference; every per-record / per-pixel stage runs in libvmsplat_b200.so:

  evaluate_sh, compute_keys, project_records  -> vms_project_records / vms_evaluate_sh
  depth_order                                 -> + vms_radix_sort_pairs
  composite_ordered                           -> + vms_composite_splats
  render_records                              -> vms_render (the session's
                                                 preprocess/sort/tile/blend path)
  render_visibility                           -> vms_visibility
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from paper_2506_19415_b200 import _device, _lib, kernels
from paper_2506_19415_b200.errors import InvariantViolation
from paper_2506_19415_b200.gaussians import RECORD_SIZE, quat_to_matrix

LOW_PASS = 0.3
MIN_DET = 1e-12
EXTENT_SIGMA = 3.0
SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
         -1.0925484305920792, 0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
         -0.4570457994644658, 1.445305721320277, -0.5900435899266435)
TILE = 16


@dataclass(frozen=True)
class Camera:
    """Pinhole camera (render.py:47-101)."""

    position: tuple
    orientation: tuple  # unit quaternion (w, x, y, z)
    fov_y: float
    width: int
    height: int
    near: float = 0.05

    def __post_init__(self):
        if not (0.0 < self.fov_y < np.pi):
            raise InvariantViolation("fov_y must lie in (0, pi)")
        if self.width < 1 or self.height < 1:
            raise InvariantViolation("resolution must be at least 1x1")
        if self.near <= 0:
            raise InvariantViolation("near plane must be positive")
        pos = np.asarray(self.position, dtype=np.float64)
        q = np.asarray(self.orientation, dtype=np.float64)
        if not (np.isfinite(pos).all() and np.isfinite(q).all()):
            raise InvariantViolation("camera pose must be finite")
        if abs(np.linalg.norm(q) - 1.0) > 1e-6:
            raise InvariantViolation("camera orientation must be a unit quaternion")

    @property
    def focal(self) -> float:
        return (self.height / 2.0) / np.tan(self.fov_y / 2.0)

    def rotation(self) -> np.ndarray:
        """Camera-to-world rotation (columns are the camera axes)."""
        return quat_to_matrix(np.asarray(self.orientation, dtype=np.float64))

    def world_to_view(self, points) -> np.ndarray:
        p = np.atleast_2d(np.asarray(points, dtype=np.float64))
        return (p - np.asarray(self.position, dtype=np.float64)) @ self.rotation()

    def view_to_pixels(self, view) -> np.ndarray:
        f = self.focal
        out = np.empty_like(view)
        out[:, 0] = f * view[:, 0] / view[:, 2] + self.width / 2.0
        out[:, 1] = f * view[:, 1] / view[:, 2] + self.height / 2.0
        out[:, 2] = 1.0 / view[:, 2]
        return out

    def scaled(self, factor: float) -> "Camera":
        return Camera(self.position, self.orientation, self.fov_y,
                      max(1, int(round(self.width * factor))),
                      max(1, int(round(self.height * factor))), self.near)

    def struct(self, dot_mode: int | None = None) -> _lib.Camera:
        """The kernel-argument form (vms_camera)."""
        if dot_mode is None:
            dot_mode = _device.probe_dot_mode()[0]
        return _device.camera_struct(self.position, self.rotation(), self.focal, self.width,
                                     self.height, self.near, dot_mode)


def evaluate_sh(coeffs, dirs) -> np.ndarray:
    """Degree-3 SH -> RGB, max(0, 0.5 + sum) (render.py:104-135)."""
    c = _device.to_dev(np.asarray(coeffs, dtype=np.float64).reshape(-1, 16, 3), np.float64)
    d = _device.to_dev(np.asarray(dirs, dtype=np.float64).reshape(-1, 3), np.float64)
    n = int(d.shape[0])
    out = _device.torch().empty((n, 3), dtype=_device.torch().float64, device=d.device)
    _lib.check(_lib.load().vms_evaluate_sh(c.data_ptr(), d.data_ptr(), n, out.data_ptr(),
                                           _device.sptr()), "evaluate_sh")
    return out.cpu().numpy()


def _project(records, camera, geometry: bool):
    t = _device.require_cuda()
    rec = _device.to_dev(records, np.float32).reshape(-1, RECORD_SIZE)
    n = int(rec.shape[0])
    dev = rec.device
    keys = t.empty(n, dtype=t.uint32, device=dev)
    cam = camera.struct()
    outs = None
    if geometry:
        outs = (t.empty((n, 2), dtype=t.float64, device=dev),
                t.empty((n, 3), dtype=t.float64, device=dev),
                t.empty((n, 3), dtype=t.float32, device=dev),
                t.empty((n, 4), dtype=t.int32, device=dev),
                t.zeros(n, dtype=t.uint8, device=dev))
    ptrs = [o.data_ptr() for o in outs] if outs else [None] * 5
    _lib.check(_lib.load().vms_project_records(rec.data_ptr(), n, ctypes.byref(cam), *ptrs,
                                               keys.data_ptr(), _device.sptr()),
               "project_records")
    return rec, keys, outs


def compute_keys(records, camera: Camera):
    """(keys uint32, indices int64) of the live records (render.py:138-152)."""
    if len(records) == 0:
        return np.zeros(0, np.uint32), np.zeros(0, np.int64)
    _, keys, _ = _project(records, camera, False)
    k = keys.cpu().numpy()
    idx = np.flatnonzero(k != 0xFFFFFFFF).astype(np.int64)
    return k[idx], idx


def project_records(records, camera: Camera):
    """EWA projection (render.py:155-220): (centers f64, conics f64, colors
    f32, alphas f32, bounds i32 half-open, kept mask)."""
    records = np.asarray(records, dtype=np.float32).reshape(-1, RECORD_SIZE)
    m = len(records)
    if m == 0:
        z = np.zeros
        return (z((0, 2)), z((0, 3)), z((0, 3), np.float32), z(0, np.float32),
                z((0, 4), np.int32), z(0, bool))
    _, _, outs = _project(records, camera, True)
    centers, conics, colors, bounds, kept = (o.cpu().numpy() for o in outs)
    kept = kept.astype(bool)
    k = np.flatnonzero(kept)
    return (centers[k], conics[k], colors[k], records[k, 10].astype(np.float32), bounds[k],
            kept)


def depth_order(records, camera: Camera) -> np.ndarray:
    """Front-to-back order of the live records (render.py:235-239)."""
    keys, idx = compute_keys(records, camera)
    _, order = kernels.radix_sort_pairs(keys, idx)
    return order


def composite_ordered(records, order, camera: Camera, exact: bool = True) -> np.ndarray:
    """Project records in the given order and composite (render.py:242-248)."""
    sorted_records = np.asarray(records, dtype=np.float32)[np.asarray(order)]
    centers, conics, colors, alphas, bounds, _ = project_records(sorted_records, camera)
    image = np.zeros((camera.height, camera.width, 3), dtype=np.float32)
    kernels.composite_splats(centers, conics, colors, alphas, bounds, image, exact=exact)
    return image


class FlatRenderer:
    """Device state for rendering a contiguous record array through the
    session's render path (vms_render): pool = the records themselves, one
    chunk table entry per 128 rows, gather index = row."""

    def __init__(self, m_cap: int = 0):
        self.m_cap = m_cap
        self._ws = None
        self._ws_key = None

    def render(self, records, camera: Camera, exact: bool = True, out=None,
               dot_mode: int | None = None):
        t = _device.require_cuda()
        rec = _device.to_dev(records, np.float32).reshape(-1, RECORD_SIZE)
        n = int(rec.shape[0])
        chunks = np.zeros((max(1, -(-n // 128)), 4), dtype=np.uint32)
        starts = np.arange(0, n, 128, dtype=np.int64)
        chunks[:len(starts), 0] = starts
        chunks[:len(starts), 1] = starts
        chunks[:len(starts), 2] = np.minimum(128, n - starts)
        dchunks = _device.to_dev(chunks, np.uint32)
        image = out if out is not None else t.empty(
            (camera.height, camera.width, 3), dtype=t.float32, device=rec.device)
        cam = camera.struct(dot_mode)
        lib = _lib.load()
        m_cap = max(self.m_cap, 16 * max(n, 1024))
        nbytes = lib.vms_render_workspace_bytes(max(n, 1), m_cap, camera.width, camera.height)
        ws = _device.workspace("flat_render", nbytes)
        ctr = t.zeros(4, dtype=t.int32).pin_memory()
        a = _lib.RenderArgs()
        a.cam = cam
        a.pool = rec.data_ptr()
        a.chunks = dchunks.data_ptr()
        a.n_chunks = len(starts)
        a.n_splats = n
        a.n_cap = max(n, 1)
        a.m_cap = m_cap
        a.image = image.data_ptr()
        a.accumulate = 0
        a.exact = int(exact)
        a.counters_out = ctr.data_ptr()
        a.workspace = ws.data_ptr()
        _lib.check(lib.vms_render(ctypes.byref(a), _device.sptr()), "render")
        t.cuda.current_stream().synchronize()
        if int(ctr[2]):
            # the frame was blended from the depth-sorted list (correct, slow);
            # size the tile-instance buffer for the next call
            m_cap = int(ctr[3]) + int(ctr[3]) // 4 + 1024
        self.m_cap = m_cap
        return image


_flat = None


def render_records(records, camera: Camera, exact: bool = True) -> np.ndarray:
    """Cull, sort front to back, project, composite (render.py:251-253).
    Returns float32 (h, w, 3)."""
    global _flat
    if _flat is None:
        _flat = FlatRenderer()
    if len(records) == 0:
        return np.zeros((camera.height, camera.width, 3), dtype=np.float32)
    return _flat.render(records, camera, exact=exact).cpu().numpy()


class VisibilityBuffers:
    """Device copies of a proxy mesh + links, reused across frames."""

    def __init__(self, vertices, faces, face_page, page_count, link_offsets=None,
                 link_targets=None):
        t = _device.require_cuda()
        self.n_faces = int(len(faces))
        self.page_count = int(page_count)
        self.verts = _device.to_dev(np.asarray(vertices, dtype=np.float64).reshape(-1, 3),
                                    np.float64)
        self.faces = _device.to_dev(np.asarray(faces, dtype=np.int32).reshape(-1, 3), np.int32)
        self.face_page = _device.to_dev(np.asarray(face_page, dtype=np.uint32).reshape(-1),
                                        np.uint32)
        if link_offsets is None:
            link_offsets = np.zeros(self.page_count + 1, dtype=np.uint32)
            link_targets = np.zeros(0, dtype=np.uint32)
        self.link_off = _device.to_dev(np.asarray(link_offsets, dtype=np.uint32), np.uint32)
        tg = np.asarray(link_targets, dtype=np.uint32)
        self.link_tgt = _device.to_dev(tg if len(tg) else np.zeros(1, np.uint32), np.uint32)
        lib = _lib.load()
        self.ws = t.empty(lib.vms_visibility_workspace_bytes(self.n_faces, self.page_count),
                          dtype=t.uint8, device=self.verts.device)
        P = self.page_count + 1
        self.req_pid = t.zeros(P, dtype=t.uint32).pin_memory()
        self.req_enc = t.zeros(P, dtype=t.uint32).pin_memory()
        self.req_direct = t.zeros(P, dtype=t.uint8).pin_memory()
        self.req_level = t.zeros(P, dtype=t.uint8).pin_memory()
        self.req_meta = t.zeros(4, dtype=t.uint32).pin_memory()

    def launch(self, vis_cam: Camera, thresholds=(), dot_mode: int = 0, id_image=None,
               invz_image=None, depth_out=None, direct_out=None):
        a = _lib.VisArgs()
        a.cam = vis_cam.struct(dot_mode)
        a.verts = self.verts.data_ptr()
        a.faces = self.faces.data_ptr()
        a.face_page = self.face_page.data_ptr()
        a.n_faces = self.n_faces
        a.page_count = self.page_count
        a.link_off = self.link_off.data_ptr()
        a.link_tgt = self.link_tgt.data_ptr()
        th = list(thresholds)
        if len(th) > 8:
            raise InvariantViolation("at most 9 LOD levels are supported")
        for i, v in enumerate(th):
            a.lod.thresholds[i] = float(v)
        a.lod.count = len(th)
        a.id_image = _lib.ptr(id_image)
        a.invz_image = _lib.ptr(invz_image)
        a.depth_out = _lib.ptr(depth_out)
        a.direct_out = _lib.ptr(direct_out)
        a.out.pid = self.req_pid.data_ptr()
        a.out.enc = self.req_enc.data_ptr()
        a.out.direct = self.req_direct.data_ptr()
        a.out.level = self.req_level.data_ptr()
        a.out.meta = self.req_meta.data_ptr()
        a.workspace = self.ws.data_ptr()
        _lib.check(_lib.load().vms_visibility(ctypes.byref(a), _device.sptr()), "visibility")

    def required(self):
        """Host view of the last compacted required list (after a sync)."""
        n = int(self.req_meta[1])
        bad = int(self.req_meta[2])
        if bad:
            raise InvariantViolation(
                f"visibility page id {bad} out of range (page count {self.page_count})")
        return (self.req_pid[:n].numpy(), self.req_enc[:n].numpy(),
                self.req_direct[:n].numpy(), self.req_level[:n].numpy())


def render_visibility(mesh, camera: Camera):
    """Page-ID image (u32) + view depth (f64, +inf background) of the proxy
    mesh (render.py:279-307).  Page-0 faces occlude but carry no page."""
    t = _device.require_cuda()
    faces = np.asarray(mesh.faces)
    fp = np.asarray(mesh.face_page, dtype=np.uint32)
    pc = int(fp.max()) if len(fp) else 0
    vb = VisibilityBuffers(mesh.vertices, faces, fp, pc)
    idi = t.zeros((camera.height, camera.width), dtype=t.uint32, device=vb.verts.device)
    zi = t.zeros((camera.height, camera.width), dtype=t.float64, device=vb.verts.device)
    vb.launch(camera, (), _device.probe_dot_mode()[0], id_image=idi, invz_image=zi)
    t.cuda.current_stream().synchronize()
    invz = zi.cpu().numpy()
    with np.errstate(divide="ignore"):
        depth = np.where(invz > 0.0, 1.0 / np.where(invz > 0.0, invz, 1.0), np.inf)
    return idi.cpu().numpy(), depth.astype(np.float64)
