"""Page-table runtime and the per-frame path (pkg/src/vmsplat/runtime.py).

Frame pipeline of ``VmSession.render_frame`` (runtime.py:436-489), B200 form:

  [1]+[2] vms_visibility      page-ID raster of the proxy mesh, fused depth
                              reduce, one-hop links, per-page LOD, ordered
                              compaction straight into mapped pinned memory
          (one event sync: the only device->host dependency of a frame)
  [3]     vms_pt_update       host C++ page table (exact update_page_table)
          vms_upload_pages    planned pages, pinned host scene -> device pool,
                              on a side stream
          adapt_thresholds    host FP64 controller (exact)
  [4-6]   vms_render          preprocess of every resident record straight
                              from the pool (no gather copy), depth sort,
                              tile duplication + tile sort, per-tile blend

Host-side value types (RequiredList, LodController, PlannedCopy) and the
depth codec keep the reference names and semantics.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from paper_2506_19415_b200 import _device, _lib
from paper_2506_19415_b200.errors import InvariantViolation
from paper_2506_19415_b200.gaussians import RECORD_BYTES, RECORD_SIZE

MAX_U32 = 0xFFFFFFFF
CHUNK = 128


# -- depth codec (runtime.py:26-43) ------------------------------------------
def encode_depth(d) -> int:
    """Monotone u32 depth, strictly decreasing in distance, 0 reserved."""
    return MAX_U32 - int(np.float32(d).view(np.uint32))


def decode_depth(e: int) -> float:
    return float(np.uint32(MAX_U32 - int(e)).view(np.float32))


def encode_depth_array(d) -> np.ndarray:
    return np.uint32(MAX_U32) - np.asarray(d, dtype=np.float32).view(np.uint32)


@dataclass
class RequiredList:
    """Per page id (1-based; 0 unused): encoded nearest depth (0 = not
    needed) and whether the page was seen directly (runtime.py:46-60)."""

    depths: np.ndarray
    direct: np.ndarray

    @property
    def page_count(self) -> int:
        return len(self.depths) - 1

    def required_ids(self) -> np.ndarray:
        return np.flatnonzero(self.depths).astype(np.int64)


def links_table(scene) -> list:
    """Per-page link target arrays, index = page id (runtime.py:63-67)."""
    return [np.zeros(0, dtype=np.uint32)] + [
        np.asarray(scene.links_for_page(p), dtype=np.uint32)
        for p in range(1, scene.page_count + 1)]


def _links_csr(links_by_page):
    n = len(links_by_page) - 1
    off = np.zeros(n + 1, dtype=np.uint32)
    parts = []
    for p in range(1, n + 1):
        tg = np.asarray(links_by_page[p], dtype=np.uint32)
        parts.append(tg)
        off[p] = off[p - 1] + len(tg)
    tgt = np.concatenate(parts) if parts else np.zeros(0, np.uint32)
    return off, tgt


def reduce_visibility(page_image, depth_image, links_by_page) -> RequiredList:
    """Fold a visibility frame into the required-page list on the GPU
    (runtime.py:70-96): nearest encoded depth per painted page, links pull
    the source's pre-propagation depth, one hop only."""
    t = _device.require_cuda()
    n = len(links_by_page) - 1
    ids = _device.to_dev(np.asarray(page_image).reshape(-1), np.uint32)
    dep = _device.to_dev(np.asarray(depth_image, dtype=np.float64).reshape(-1), np.float64)
    off, tgt = _links_csr(links_by_page)
    doff = _device.to_dev(off, np.uint32)
    dtgt = _device.to_dev(tgt if len(tgt) else np.zeros(1, np.uint32), np.uint32)
    depths = t.zeros(n + 1, dtype=t.uint32, device=ids.device)
    direct = t.zeros(n + 1, dtype=t.uint8, device=ids.device)
    bad = t.zeros(1, dtype=t.uint32, device=ids.device)
    ws = _device.workspace("reduce", 4 * (n + 1))
    lib = _lib.load()
    _lib.check(lib.vms_reduce_visibility(ids.data_ptr(), dep.data_ptr(), int(ids.numel()), n,
                                         doff.data_ptr(), dtgt.data_ptr(), depths.data_ptr(),
                                         direct.data_ptr(), bad.data_ptr(), ws.data_ptr(),
                                         ws.numel(), _device.sptr()), "reduce_visibility")
    b = int(bad.cpu().numpy()[0])
    if b:
        raise InvariantViolation(f"visibility page id {b} out of range (page count {n})")
    return RequiredList(depths=depths.cpu().numpy(), direct=direct.cpu().numpy().astype(bool))


# -- LOD controller (runtime.py:99-158), host FP64 ----------------------------
@dataclass
class LodController:
    thresholds: np.ndarray
    step: float = 0.05
    band_low: float = 0.5
    band_high: float = 0.8
    step_min: float = 0.005
    step_max: float = 0.5
    window: int = 30
    last_move_direction: int = 0
    last_move_frame: int = -(10 ** 9)

    def __post_init__(self):
        self.thresholds = np.asarray(self.thresholds, dtype=np.float64)
        if np.any(np.diff(self.thresholds) <= 0):
            raise InvariantViolation("thresholds must be strictly increasing")

    @property
    def level_count(self) -> int:
        return len(self.thresholds) + 1


def initial_thresholds(scene_radius: float, level_count: int) -> np.ndarray:
    """Geometric spread ending at the scene radius, e.g. (r/4, r/2, r)."""
    k = level_count - 1
    return scene_radius * np.power(2.0, np.arange(k) - (k - 1), dtype=np.float64)


def select_lod(encoded_depth: int, controller: LodController) -> int:
    """Level = number of thresholds strictly below the decoded distance."""
    return int(np.count_nonzero(controller.thresholds < decode_depth(encoded_depth)))


def adapt_thresholds(controller: LodController, usage_ratio: float, frame: int) -> None:
    """Nudge thresholds toward the usage band, in place (runtime.py:135-158)."""
    if usage_ratio > controller.band_high:
        direction = -1
    elif usage_ratio < controller.band_low:
        direction = +1
    else:
        return
    if controller.thresholds.size == 0:
        return
    if frame - controller.last_move_frame <= controller.window:
        factor = 1.01 if direction == controller.last_move_direction else 0.99
        controller.step = float(
            np.clip(controller.step * factor, controller.step_min, controller.step_max))
    controller.thresholds = controller.thresholds * (1.0 + direction * controller.step)
    controller.last_move_direction = direction
    controller.last_move_frame = frame


# -- page table (runtime.py:161-291) on the C++ engine -------------------------
class PageTableEntry:
    """Snapshot of one physical entry: LOD level (-1 empty), LRU stamp, slots."""

    __slots__ = ("lod_level", "last_used_frame", "slots")

    def __init__(self, level=-1, last=-1, slots=()):
        self.lod_level = level
        self.last_used_frame = last
        self.slots = list(slots)

    @property
    def empty(self) -> bool:
        return self.lod_level < 0

    def occupied_slots(self) -> int:
        return sum(1 for s in self.slots if s)


@dataclass(frozen=True)
class PlannedCopy:
    page_id: int
    level: int
    entry: int
    slot: int


class PageTable:
    """Flat entry array + page-id -> (entry, slot) residency map, held by
    the host C++ page table (O(log n) allocation, exact LRU semantics)."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise InvariantViolation("page table needs at least one entry")
        self._lib = _lib.load()
        h = self._lib.vms_pt_create(int(capacity))
        if not h:
            raise InvariantViolation(self._lib.vms_last_error().decode())
        self._h = ctypes.c_void_p(h)
        self._cap = int(capacity)
        self._plan_cap = 0
        self._plan = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.vms_pt_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def capacity(self) -> int:
        return self._cap

    def occupied_entries(self) -> int:
        return int(self._lib.vms_pt_occupied(self._h))

    def usage_ratio(self) -> float:
        return self.occupied_entries() / self.capacity

    def resident_arrays(self):
        n = int(self._lib.vms_pt_resident_count(self._h))
        pid = np.zeros(n, np.uint32)
        ent = np.zeros(n, np.int32)
        slot = np.zeros(n, np.int32)
        _lib.check(self._lib.vms_pt_resident(self._h, pid.ctypes.data, ent.ctypes.data,
                                             slot.ctypes.data, n), "pt_resident")
        return pid, ent, slot

    @property
    def resident(self) -> dict:
        pid, ent, slot = self.resident_arrays()
        return {int(p): (int(e), int(s)) for p, e, s in zip(pid, ent, slot)}

    def resident_count(self) -> int:
        return int(self._lib.vms_pt_resident_count(self._h))

    @property
    def entries(self) -> list:
        level = np.zeros(self._cap, np.int32)
        last = np.zeros(self._cap, np.int64)
        ms = 1 << 8
        slots = np.zeros((self._cap, ms), np.uint32)
        _lib.check(self._lib.vms_pt_entries(self._h, level.ctypes.data, last.ctypes.data,
                                            slots.ctypes.data, ms), "pt_entries")
        out = []
        for i in range(self._cap):
            lv = int(level[i])
            s = slots[i, :(1 << lv)] if lv >= 0 else []
            out.append(PageTableEntry(lv, int(last[i]), [int(x) for x in s]))
        return out

    def resident_level(self, page_id: int):
        loc = self.resident.get(page_id)
        return None if loc is None else self.entries[loc[0]].lod_level

    def resident_counts(self, level_count: int) -> tuple:
        c = np.zeros(level_count, np.int64)
        _lib.check(self._lib.vms_pt_resident_counts(self._h, c.ctypes.data, level_count),
                   "resident_counts")
        return tuple(int(x) for x in c)

    def check(self) -> None:
        _lib.check(self._lib.vms_pt_check(self._h), "page table check")

    def update(self, pid, enc, direct, level, frame: int, budget: float):
        """Run update_page_table on compacted arrays; returns
        (plan_pid, plan_level, plan_entry, plan_slot, missing)."""
        n = len(pid)
        if self._plan_cap < max(n, 1):
            self._plan_cap = max(n, 1) * 2
            self._plan = (np.zeros(self._plan_cap, np.uint32), np.zeros(self._plan_cap, np.uint8),
                          np.zeros(self._plan_cap, np.int32), np.zeros(self._plan_cap, np.int32))
        pp, pl, pe, ps = self._plan
        n_plan = ctypes.c_int64(0)
        missing = ctypes.c_int64(0)
        pid = np.ascontiguousarray(pid, np.uint32)
        enc = np.ascontiguousarray(enc, np.uint32)
        direct = np.ascontiguousarray(direct, np.uint8)
        level = np.ascontiguousarray(level, np.uint8)
        _lib.check(self._lib.vms_pt_update(self._h, pid.ctypes.data, enc.ctypes.data,
                                           direct.ctypes.data, level.ctypes.data, n, int(frame),
                                           float(budget), pp.ctypes.data, pl.ctypes.data,
                                           pe.ctypes.data, ps.ctypes.data, self._plan_cap,
                                           ctypes.byref(n_plan), ctypes.byref(missing)),
                   "update_page_table")
        k = n_plan.value
        return pp[:k].copy(), pl[:k].copy(), pe[:k].copy(), ps[:k].copy(), int(missing.value)


def update_page_table(table: PageTable, required: RequiredList, controller: LodController,
                      frame: int, staging_budget_pages: float):
    """Two-pass table update (runtime.py:294-346).  Returns (plan, missing)."""
    ids = required.required_ids()
    enc = required.depths[ids].astype(np.uint32)
    direct = required.direct[ids].astype(np.uint8)
    level = np.array([select_lod(int(e), controller) for e in enc], dtype=np.uint8)
    pp, pl, pe, ps, missing = table.update(ids.astype(np.uint32), enc, direct, level, frame,
                                           staging_budget_pages)
    plan = [PlannedCopy(int(a), int(b), int(c), int(d)) for a, b, c, d in zip(pp, pl, pe, ps)]
    return plan, missing


# -- the session ----------------------------------------------------------------
class ProxyMesh:
    """Triangle mesh with one page id per face (mesh/geometry.py:13-45)."""

    def __init__(self, vertices, faces, face_page=None):
        self.vertices = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
        self.faces = np.asarray(faces, dtype=np.int32).reshape(-1, 3)
        if face_page is None:
            face_page = np.zeros(len(self.faces), dtype=np.uint32)
        self.face_page = np.asarray(face_page, dtype=np.uint32).reshape(-1)

    @property
    def vertex_count(self) -> int:
        return self.vertices.shape[0]

    @property
    def face_count(self) -> int:
        return self.faces.shape[0]


class VmSession:
    """Owns the page table, the device page pool and the controller across
    frames (runtime.py:393-434).

    Extra (non-reference) knobs: ``exact`` blends in FP64 with the
    reference's arithmetic; ``upload_mode`` 1 uploads a frame's pages with a
    single gather kernel over mapped pinned memory, 0 with one
    cudaMemcpyAsync per page; ``device`` selects the GPU.
    """

    def __init__(self, scene, buffer_pages: int = 500, staging_pages: float = 40,
                 vis_scale: float = 0.25, band=(0.5, 0.8), step: float = 0.05,
                 lod_enabled: bool = True, links_enabled: bool = True, exact: bool = True,
                 upload_mode: int = 1, device=None):
        from paper_2506_19415_b200.render import VisibilityBuffers

        t = _device.require_cuda()
        if scene.page_count == 0:
            raise InvariantViolation("scene has no pages; run paging first")
        self.device = t.device("cuda", t.cuda.current_device()) if device is None else \
            t.device(device)
        self.scene = scene
        self.mesh = ProxyMesh(np.asarray(scene.vertices).astype(np.float64),
                              np.asarray(scene.faces).astype(np.int32),
                              np.asarray(scene.face_page).copy())
        self.links_enabled = links_enabled
        self._links = None
        level_count = scene.lod_levels if lod_enabled else 1
        radius = scene.half_extent * np.sqrt(3.0)
        self.controller = LodController(initial_thresholds(radius, level_count), step=step,
                                        band_low=band[0], band_high=band[1])
        self.lod_enabled = lod_enabled and level_count > 1
        self.table = PageTable(buffer_pages)
        self.staging_pages = staging_pages
        self.vis_scale = vis_scale
        self.exact = bool(exact)
        self.upload_mode = int(upload_mode)
        self.page_size = int(scene.page_size)
        self.dot_mode, self.dot_mode_exact = _device.probe_dot_mode()

        with t.cuda.device(self.device):
            if links_enabled:
                off = np.asarray(scene.link_offsets, np.uint32)
                tgt = np.asarray(scene.link_targets, np.uint32)
            else:
                off = np.zeros(scene.page_count + 1, np.uint32)
                tgt = np.zeros(0, np.uint32)
            self.vis = VisibilityBuffers(self.mesh.vertices, self.mesh.faces, self.mesh.face_page,
                                         scene.page_count, off, tgt)
            # device page pool: capacity entries of page_size records
            self.n_cap = buffer_pages * self.page_size
            self.pool = t.empty((self.n_cap, RECORD_SIZE), dtype=t.float32, device=self.device)
            # shared pinned host copy of every level's records (the streaming source)
            self.host = _pinned_records(scene)
            self.m_cap = max(16 * self.n_cap, 1 << 20)
            self._alloc_render_ws()
            max_chunks = buffer_pages * (-(-self.page_size // CHUNK) + (1 << max(0, scene.lod_levels - 1)))
            self.chunks_host = t.zeros((max_chunks, 4), dtype=t.int32).pin_memory()
            self.chunks_dev = t.zeros((max_chunks, 4), dtype=t.int32, device=self.device)
            self.copies_host = t.zeros((scene.page_count + 1, 3), dtype=t.int64).pin_memory()
            self.counters = t.zeros(4, dtype=t.int32).pin_memory()
            self.copy_stream = t.cuda.Stream(device=self.device)
            ev = lambda: t.cuda.Event(enable_timing=True)  # noqa: E731
            self.ev = {k: ev() for k in ("start", "vis", "req", "copy0", "copy1", "render0",
                                         "pre", "sorted", "blend0", "blend1", "end")}
            self.ev_copy_done = t.cuda.Event()
            for e in self.ev.values():  # torch creates CUDA events lazily
                e.record(t.cuda.current_stream())
        self._last_render = None  # args of the last render, for overflow recovery
        self.frame_log = []

    # reference attribute: per-page link arrays
    @property
    def links(self):
        if self._links is None:
            sc = self.scene
            self._links = (links_table(sc) if self.links_enabled else
                           [np.zeros(0, dtype=np.uint32) for _ in range(sc.page_count + 1)])
        return self._links

    @property
    def buffer(self):
        return self.pool

    def _alloc_render_ws(self):
        t = _device.torch()
        sc = self.scene
        self._ws_res = None
        self.render_ws = None
        self._ws_for = None

    def _ensure_render_ws(self, width, height):
        t = _device.torch()
        key = (width, height, self.m_cap)
        if self._ws_for != key:
            nbytes = _lib.load().vms_render_workspace_bytes(self.n_cap, self.m_cap, width, height)
            self.render_ws = None
            self.render_ws = t.empty(nbytes, dtype=t.uint8, device=self.device)
            self._ws_for = key

    # -- stages ------------------------------------------------------------
    def _visibility(self, camera):
        thr = self.controller.thresholds if self.controller.thresholds.size else ()
        self.vis.launch(camera.scaled(self.vis_scale), thr, self.dot_mode)

    def _launch_render(self, camera, image, n_chunks, n_res, record_events=True):
        self._ensure_render_ws(camera.width, camera.height)
        a = _lib.RenderArgs()
        a.cam = camera.struct(self.dot_mode)
        a.pool = self.pool.data_ptr()
        a.chunks = self.chunks_dev.data_ptr()
        a.n_chunks = n_chunks
        a.n_splats = n_res
        a.n_cap = self.n_cap
        a.m_cap = self.m_cap
        a.image = image.data_ptr()
        a.accumulate = 0
        a.exact = int(self.exact)
        a.counters_out = self.counters.data_ptr()
        a.workspace = self.render_ws.data_ptr()
        if record_events:
            for i, k in enumerate(("pre", "sorted", "blend0", "blend1")):
                a.events[i] = self.ev[k].cuda_event
        _lib.check(_lib.load().vms_render(ctypes.byref(a), _device.sptr()), "render")

    def _check_overflow(self, camera, image, n_chunks, n_res):
        """After a sync: if the tile-instance buffer overflowed, grow it and
        re-render (the pool and chunk table are unchanged)."""
        t = _device.torch()
        while int(self.counters[2]):
            need = int(self.counters[3])
            self.m_cap = need + need // 4 + (1 << 16)
            self._launch_render(camera, image, n_chunks, n_res, record_events=False)
            t.cuda.current_stream().synchronize()

    def render_frame(self, camera, frame_index: int, out=None):
        """Run one frame.  Returns (image, stats) with the reference's stats
        keys (runtime.py:471-488).  ``out``: None -> new numpy array;
        a pinned/regular numpy (h, w, 3) f32 array -> filled in place;
        "device" -> a CUDA tensor (no host copy)."""
        t = _device.torch()
        ev = self.ev
        stream = t.cuda.current_stream()
        sc = self.scene
        h0 = time.perf_counter()
        ev["start"].record(stream)
        self._visibility(camera)
        ev["vis"].record(stream)
        ev["req"].record(stream)
        ev["req"].synchronize()
        pid, enc, direct, level = self.vis.required()
        h1 = time.perf_counter()
        pp, pl, pe, ps, missing = self.table.update(pid, enc, direct, level, frame_index,
                                                    self.staging_pages)
        h2 = time.perf_counter()
        # uploads on the side stream
        bytes_copied = 0
        n_plan = len(pp)
        if n_plan:
            per = (self.page_size >> pl.astype(np.int64)).astype(np.int64)
            starts = np.zeros(len(sc.page_counts) + 1, np.int64)
            for k in range(sc.lod_levels):
                starts[k + 1] = starts[k] + sc.page_counts[k] * (self.page_size >> k)
            src_rows = starts[pl.astype(np.int64)] + (pp.astype(np.int64) - 1) * per
            dst_rows = pe.astype(np.int64) * self.page_size + ps.astype(np.int64) * per
            cp = self.copies_host.numpy()
            cp[:n_plan, 0] = src_rows * RECORD_BYTES
            cp[:n_plan, 1] = dst_rows * RECORD_BYTES
            cp[:n_plan, 2] = per * RECORD_BYTES
            bytes_copied = int((per * RECORD_BYTES).sum())
            self.copy_stream.wait_stream(stream)
            with t.cuda.stream(self.copy_stream):
                ev["copy0"].record(self.copy_stream)
                _lib.check(_lib.load().vms_upload_pages(
                    self.copies_host.data_ptr(), n_plan, self.host.data_ptr(),
                    self.pool.data_ptr(), self.upload_mode, self.copy_stream.cuda_stream),
                    "upload_pages")
                ev["copy1"].record(self.copy_stream)
            stream.wait_stream(self.copy_stream)
        h3 = time.perf_counter()
        usage = self.table.usage_ratio()
        if self.lod_enabled:
            adapt_thresholds(self.controller, usage, frame_index)
        # chunk table of every resident page, ascending page id
        n_rec = ctypes.c_int64(0)
        cap = self.chunks_host.shape[0]
        n_chunks = int(_lib.load().vms_pt_chunks(self.table.handle, self.page_size,
                                                 self.chunks_host.data_ptr(), cap,
                                                 ctypes.byref(n_rec)))
        if n_chunks > cap:
            raise InvariantViolation("chunk table overflow")
        n_res = int(n_rec.value)
        if n_chunks:
            self.chunks_dev[:n_chunks].copy_(self.chunks_host[:n_chunks], non_blocking=True)
        h4 = time.perf_counter()
        if out is None or isinstance(out, np.ndarray):
            image = self._frame_image(camera)
        elif isinstance(out, str) and out == "device":
            image = self._frame_image(camera)
        else:
            image = out
        ev["render0"].record(stream)
        self._launch_render(camera, image, n_chunks, n_res)
        ev["end"].record(stream)
        if out is None or isinstance(out, np.ndarray):
            ev["end"].synchronize()
            self._check_overflow(camera, image, n_chunks, n_res)
            if out is None:
                host_img = image.cpu().numpy()
            else:
                hv = t.from_numpy(out)
                hv.copy_(image, non_blocking=True)
                stream.synchronize()
                host_img = out
        else:
            ev["end"].synchronize()
            self._check_overflow(camera, image, n_chunks, n_res)
            host_img = image
        h5 = time.perf_counter()
        d = lambda a, b: ev[a].elapsed_time(ev[b]) / 1e3  # noqa: E731
        t_copy = d("copy0", "copy1") if n_plan else 0.0
        stats = {
            "frame": frame_index,
            "required_pages": int(len(pid)),
            "resident_pages": int(self.table.resident_count()),
            "resident_per_level": self.table.resident_counts(sc.lod_levels),
            "planned_copies": int(n_plan),
            "missing_pages": int(missing),
            "bytes_copied": int(bytes_copied),
            "usage": usage,
            "lod_step": self.controller.step,
            "thresholds": tuple(float(x) for x in self.controller.thresholds),
            "time_visibility": d("start", "vis"),
            "time_reduce": 0.0,
            "time_update": h2 - h1,
            "time_copy": t_copy + (h4 - h3),
            "time_sort": d("render0", "sorted"),
            "time_render": d("sorted", "end"),
            "time_frame_wall": h5 - h0,
            "time_preprocess": d("render0", "pre"),
            "time_tiles": d("sorted", "blend0"),
            "time_blend": d("blend0", "blend1"),
            "time_device_frame": d("start", "end"),
            "n_kept": int(self.counters[0]),
            "n_instances": int(self.counters[1]),
            "n_resident_records": n_res,
            "n_chunks": n_chunks,
        }
        return host_img, stats

    def _frame_image(self, camera):
        t = _device.torch()
        key = (camera.height, camera.width)
        imgs = getattr(self, "_images", None)
        if imgs is None or imgs[0] != key:
            imgs = (key, [t.empty((camera.height, camera.width, 3), dtype=t.float32,
                                  device=self.device) for _ in range(2)], 0)
        key, bufs, i = imgs
        self._images = (key, bufs, i ^ 1)
        return bufs[i]


def _pinned_records(scene):
    """Copy the scene's record section into page-locked host memory, in
    256 MB slices (works for np.memmap sources without a second copy)."""
    t = _device.torch()
    g = scene.gaussians
    n = len(g)
    host = t.empty((max(n, 1), RECORD_SIZE), dtype=t.float32).pin_memory()
    hv = host.numpy()
    step = max(1, (256 << 20) // RECORD_BYTES)
    for a in range(0, n, step):
        hv[a:a + step] = g[a:a + step]
    return host
