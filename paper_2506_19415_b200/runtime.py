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
        self._owner = None

    @classmethod
    def borrowed(cls, handle, capacity: int, owner):
        """A view of a page table owned by a C++ session (kept alive by owner)."""
        self = cls.__new__(cls)
        self._lib = _lib.load()
        self._h = ctypes.c_void_p(handle)
        self._cap = int(capacity)
        self._plan_cap = 0
        self._plan = None
        self._owner = owner
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and getattr(self, "_owner", None) is None:
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


DEVICE_TABLE_MAX_CAPACITY = 8192  # csrc/dpt.cu kMaxCap (entry metadata in shared memory)
DEVICE_TABLE_MAX_LEVELS = 6        # <= 32 slots per entry
# largest page count the device table's 30-bit page ids address
DEVICE_TABLE_MAX_PAGES = (1 << 30) - 1


class DevicePageTable:
    """The same table resident in device memory (SURVEY §8(f) F2,
    csrc/dpt.cu): ``update`` runs update_page_table's two passes on the GPU
    (one CTA; bit-identical plans, LRU stamps and residency to PageTable and
    the reference).  Queries take a device snapshot.  capacity <= 8192,
    levels <= 6; ``page_count`` bounds the page ids."""

    def __init__(self, capacity: int, page_count: int, levels: int = 1):
        if capacity < 1:
            raise InvariantViolation("page table needs at least one entry")
        self._lib = _lib.load()
        t = _device.require_cuda()
        h = self._lib.vms_dpt_create(int(capacity), int(page_count), int(levels))
        if not h:
            raise InvariantViolation(self._lib.vms_last_error().decode())
        self._h = ctypes.c_void_p(h)
        self._cap, self._pages, self._levels = int(capacity), int(page_count), int(levels)
        self._t = t
        dev = t.device("cuda", t.cuda.current_device())
        self._frame = t.zeros(16, dtype=t.uint8, device=dev)
        self._stats = t.zeros(ctypes.sizeof(_lib.DptStats), dtype=t.uint8, device=dev)
        self._n = t.zeros(1, dtype=t.int32, device=dev)
        self._last_stats = _lib.DptStats()
        self._owner = None

    @classmethod
    def borrowed(cls, handle, capacity: int, page_count: int, levels: int, owner):
        """A view of the device table owned by a session (kept alive by owner)."""
        self = cls.__new__(cls)
        self._lib = _lib.load()
        self._h = ctypes.c_void_p(handle)
        self._cap, self._pages, self._levels = int(capacity), int(page_count), int(levels)
        self._owner = owner
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and getattr(self, "_owner", None) is None:
            self._lib.vms_dpt_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def capacity(self) -> int:
        return self._cap

    def _state(self):
        ms = 1 << (self._levels - 1)
        level = np.zeros(self._cap, np.int32)
        last = np.zeros(self._cap, np.int64)
        slots = np.zeros((self._cap, ms), np.uint32)
        res = np.zeros(self._pages + 1, np.uint32)
        _lib.check(self._lib.vms_dpt_state(self._h, level.ctypes.data, last.ctypes.data,
                                           slots.ctypes.data, ms, res.ctypes.data,
                                           _device.sptr()), "dpt_state")
        return level, last, slots, res

    @property
    def entries(self) -> list:
        level, last, slots, _ = self._state()
        return [PageTableEntry(int(lv), int(la), [int(x) for x in sl[:(1 << lv)]] if lv >= 0 else [])
                for lv, la, sl in zip(level, last, slots)]

    @property
    def resident(self) -> dict:
        _, _, _, res = self._state()
        ids = np.flatnonzero(res != 0xFFFFFFFF)
        return {int(p): (int(res[p] >> 8), int(res[p] & 0xFF)) for p in ids}

    def resident_count(self) -> int:
        return len(self.resident)

    def occupied_entries(self) -> int:
        level, _, _, _ = self._state()
        return int((level >= 0).sum())

    def usage_ratio(self) -> float:
        return self.occupied_entries() / self.capacity

    def resident_level(self, page_id: int):
        loc = self.resident.get(page_id)
        return None if loc is None else self.entries[loc[0]].lod_level

    def resident_counts(self, level_count: int) -> tuple:
        counts = [0] * level_count
        level, _, _, res = self._state()
        for p in np.flatnonzero(res != 0xFFFFFFFF):
            counts[int(level[res[p] >> 8])] += 1
        return tuple(counts)

    def check(self) -> None:
        """Cross-check the residency map against the entries (runtime.py:218-234)."""
        level, _, slots, res = self._state()
        seen = {}
        for ei in range(self._cap):
            if level[ei] < 0:
                continue
            for si, pid in enumerate(slots[ei, :(1 << int(level[ei]))]):
                if pid:
                    if int(pid) in seen:
                        raise InvariantViolation(f"page {pid} resident twice")
                    seen[int(pid)] = (ei, si)
        mapped = {int(p): (int(res[p] >> 8), int(res[p] & 0xFF))
                  for p in np.flatnonzero(res != 0xFFFFFFFF)}
        if seen != mapped:
            raise InvariantViolation("residency map out of sync with entries")

    def update(self, pid, enc, direct, level, frame: int, budget: float):
        """update_page_table's two passes on the device (compacted required
        arrays, ascending page id); returns (plan_pid, plan_level,
        plan_entry, plan_slot, missing)."""
        t = self._t
        n = len(pid)
        dev = self._frame.device
        def arr(x, dt):  # at least one element (an empty list passes a dummy)
            x = np.ascontiguousarray(x, dt)
            return _device.to_dev(x if len(x) else np.zeros(1, dt), dt)

        pid_d, enc_d = arr(pid, np.uint32), arr(enc, np.uint32)
        dir_d, lvl_d = arr(direct, np.uint8), arr(level, np.uint8)
        fr = _lib.DptFrame(int(frame), float(budget))
        self._frame.copy_(t.frombuffer(bytearray(bytes(fr)), dtype=t.uint8))
        self._n.fill_(n)
        cap = max(n, 1)
        pp = t.zeros(cap, dtype=t.int32, device=dev)
        pl = t.zeros(cap, dtype=t.uint8, device=dev)
        pe = t.zeros(cap, dtype=t.int32, device=dev)
        ps = t.zeros(cap, dtype=t.int32, device=dev)
        _lib.check(self._lib.vms_dpt_update(self._h, _lib.ptr(pid_d), _lib.ptr(enc_d),
                                            _lib.ptr(dir_d), _lib.ptr(lvl_d), self._n.data_ptr(),
                                            self._frame.data_ptr(), pp.data_ptr(), pl.data_ptr(),
                                            pe.data_ptr(), ps.data_ptr(), cap,
                                            self._stats.data_ptr(), _device.sptr()),
                   "update_page_table (device)")
        raw = self._stats.cpu().numpy().tobytes()
        st = _lib.DptStats.from_buffer_copy(raw)
        self._last_stats = st
        if st.bad:
            raise InvariantViolation("required page id or LOD level out of range")
        k = int(st.n_plan)
        return (pp[:k].cpu().numpy().astype(np.uint32), pl[:k].cpu().numpy(),
                pe[:k].cpu().numpy(), ps[:k].cpu().numpy(), int(st.missing))


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
    frames (runtime.py:393-434).  Each ``render_frame`` is ONE call into the
    C++ session (csrc/session.cu): visibility -> event sync -> page table ->
    uploads (side stream) -> chunk table -> render; the FP64 LOD controller
    adapts on the host afterwards, exactly as the reference orders it.

    Extra (non-reference) knobs: ``exact`` (default) blends with the
    reference's FP64 arithmetic, False selects the FP32 blend;
    ``upload_mode`` 0 uploads a frame's pages from the page-locked host
    scene (``HostScene``) with one batched copy-engine call (no SM time,
    overlaps the render in flight), 1 with one gather kernel over mapped
    pinned memory, 2 streams them
    from the scene's memory-mapped rows (host threads gather each frame's
    pages into a page-locked bounce buffer; for scenes larger than the
    page-locked memory one wants to commit - out-of-core); the
    default (None) picks 0 when the scene can be page-locked, else 2; ``timing``
    records per-stage CUDA events (the stats' time_* keys; costs one sync per
    frame); ``device`` selects the GPU.
    """

    def __init__(self, scene, buffer_pages: int = 500, staging_pages: float = 40,
                 vis_scale: float = 0.25, band=(0.5, 0.8), step: float = 0.05,
                 lod_enabled: bool = True, links_enabled: bool = True, exact: bool = True,
                 upload_mode: int | None = None, timing: bool = True, device=None,
                 instance_capacity: int | None = None, device_table: bool | None = None):
        from paper_2506_19415_b200.render import VisibilityBuffers

        t = _device.require_cuda()
        if scene.page_count == 0:
            raise InvariantViolation("scene has no pages; run paging first")
        if scene.lod_levels > 16:
            raise InvariantViolation("at most 16 LOD levels are supported")
        if lod_enabled and scene.lod_levels > 9:
            # vms_lod carries 8 thresholds (levels 0-8)
            raise InvariantViolation("LOD selection supports at most 9 levels; "
                                     "pass lod_enabled=False for deeper scenes")
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
        self.staging_pages = staging_pages
        self.vis_scale = vis_scale
        self.exact = bool(exact)
        self.upload_mode = -1 if upload_mode is None else int(upload_mode)
        self.timing = bool(timing)
        self.page_size = int(scene.page_size)
        self.capacity = int(buffer_pages)
        if buffer_pages < 1:
            raise InvariantViolation("page table needs at least one entry")
        self.dot_mode, self.dot_mode_exact = _device.probe_dot_mode()
        self._lib = _lib.load()
        with t.cuda.device(self.device):
            if links_enabled:
                off = np.asarray(scene.link_offsets, np.uint32)
                tgt = np.asarray(scene.link_targets, np.uint32)
            else:
                off = np.zeros(scene.page_count + 1, np.uint32)
                tgt = np.zeros(0, np.uint32)
            self.vis = VisibilityBuffers(self.mesh.vertices, self.mesh.faces, self.mesh.face_page,
                                         scene.page_count, off, tgt)
            self.n_cap = self.capacity * self.page_size
            self.pool = t.empty((self.n_cap, RECORD_SIZE), dtype=t.float32, device=self.device)
            if self.upload_mode < 0:
                # auto: DMA from the page-locked scene when it can be
                # page-locked (a registered tmpfs file, or a private copy
                # that fits), else stream through the bounce buffer
                try:
                    HostScene.of(scene)
                    self.upload_mode = 0
                except (MemoryError, RuntimeError) as exc:
                    import warnings

                    warnings.warn(f"scene not page-lockable ({exc}); streaming pages from "
                                  "the mapping (upload_mode 2)", RuntimeWarning)
                    self.upload_mode = 2
            self._fd = None
            if self.upload_mode == 2:
                # streaming source: the scene's own (memory-mapped) rows; the
                # session gathers each frame's pages through a page-locked
                # bounce buffer, so the scene need not fit in pinned memory.
                # A file-backed scene is read with pread (host threads, no
                # page faults on the untouched mapping)
                self.host = np.ascontiguousarray(scene.gaussians, dtype=np.float32)
                host_ptr = self.host.ctypes.data
                if isinstance(scene.gaussians, np.memmap) and getattr(scene, "path", None):
                    import os

                    self._fd = os.open(scene.path, os.O_RDONLY)
            else:
                # page-locked, mapped into the device; shared by every
                # session of the process (and, for a memory-mapped file, by
                # every process mapping it)
                self.host = HostScene.of(scene)
                host_ptr = self.host.ptr
            d = _lib.SessionDesc()
            d.host_records = host_ptr
            d.host_rows = int(len(scene.gaussians))
            d.page_size = self.page_size
            d.lod_levels = int(scene.lod_levels)
            for k, c in enumerate(scene.page_counts):
                d.page_counts[k] = int(c)
            d.page_count = int(scene.page_count)
            d.n_faces = self.vis.n_faces
            d.verts = self.vis.verts.data_ptr()
            d.faces = self.vis.faces.data_ptr()
            d.face_page = self.vis.face_page.data_ptr()
            d.link_off = self.vis.link_off.data_ptr()
            d.link_tgt = self.vis.link_tgt.data_ptr()
            d.pool = self.pool.data_ptr()
            d.capacity = self.capacity
            d.vis_ws = self.vis.ws.data_ptr()
            d.exact = int(self.exact)
            d.upload_mode = self.upload_mode
            d.host_fd = -1 if self._fd is None else int(self._fd)
            d.host_fd_offset = int(getattr(scene, "gaus_offset", 0)) if self._fd is not None else 0
            # tile-instance capacity; the session regrows it on overflow
            # (64 M instances, 1 GB: frames with the camera inside dense
            # geometry need tens of millions; past it they blend through the
            # exact but slower spill path)
            d.m_cap = int(instance_capacity) if instance_capacity else 1 << 26
            # the page table on the device: the visibility
            # graph runs update_page_table too; the host only issues copies
            if device_table is None:
                # default: on the device whenever it fits its limits (measured:
                # +3-4 % device fps, +4-5 % e2e on C2/C3, equal on C4);
                # VMSPLAT_DEVICE_TABLE
                # = 0 / 1 forces the host C++ table / the device table
                import os

                env = os.environ.get("VMSPLAT_DEVICE_TABLE", "")
                device_table = env == "1" if env in ("0", "1") else (
                    self.capacity <= DEVICE_TABLE_MAX_CAPACITY and
                    int(scene.lod_levels) <= DEVICE_TABLE_MAX_LEVELS and
                    int(scene.page_count) <= DEVICE_TABLE_MAX_PAGES)
            d.device_table = int(bool(device_table))
            self.device_table = bool(device_table)
            self._desc = d
            self._h = None
            h = self._lib.vms_session_create(ctypes.byref(d))
            if not h:
                raise InvariantViolation(self._lib.vms_last_error().decode())
            self._h = ctypes.c_void_p(h)
            if self.device_table:
                self.table = DevicePageTable.borrowed(self._lib.vms_session_dpt(self._h),
                                                      self.capacity, scene.page_count,
                                                      scene.lod_levels, self)
            else:
                self.table = PageTable.borrowed(self._lib.vms_session_table(self._h),
                                                self.capacity, self)
        self._args = _lib.FrameArgs()
        self._stats = _lib.FrameStats()
        self._pinned_out = None

    def close(self):
        """Free the session's device and page-locked memory now.  The session
        and its page table refer to each other, so dropping the last
        reference leaves the teardown (a device synchronisation, GBs of
        frees) to Python's cycle collector - which may run it in the middle
        of another session's frames.  The table view is invalid afterwards."""
        tbl = self.__dict__.get("table")
        if tbl is not None:
            tbl._h = ctypes.c_void_p(0)
        self.__del__()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.vms_session_destroy(h)
            self._h = None
        fd = getattr(self, "_fd", None)
        if fd is not None:
            import os

            os.close(fd)
            self._fd = None

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

    def render_frame(self, camera, frame_index: int, out=None, wait: bool = True):
        """Run one frame.  Returns (image, stats) with the reference's stats
        keys (runtime.py:471-488) plus device counters.  ``out``: None -> a new
        (page-locked) numpy array; a float32 (h, w, 3) numpy array -> filled
        in place (by DMA when it is page-locked, else through a staging
        buffer); "device" -> a CUDA tensor, ordered on the current stream (the
        session alternates two such buffers), returned as soon as the frame
        is enqueued; a float32 (h, w, 3) CUDA tensor -> written in place, the
        same way.  ``wait=False`` with page-locked host output also
        returns as soon as the frame is enqueued (``slots`` frames in
        flight); the array is complete after ``wait(0)`` (or ``wait(k)`` once
        k more frames have been submitted, k < slots)."""
        t = _device.torch()
        lib = self._lib
        h0 = time.perf_counter()
        a = self._args
        fill_frame_cameras(a, camera, self.vis_scale, self.dot_mode)
        thr = self.controller.thresholds
        if thr.size > 8:
            raise InvariantViolation("at most 9 LOD levels are supported")
        for i, v in enumerate(thr):
            a.lod.thresholds[i] = float(v)
        a.lod.count = int(thr.size)
        a.frame = int(frame_index)
        a.budget = float(self.staging_pages)
        a.timing = int(self.timing)
        device_out = isinstance(out, str) and out == "device"
        a.host_image = None
        a.sync = 0
        host = None
        if isinstance(out, t.Tensor):
            # a caller-owned CUDA tensor (e.g. a slot of a frame stack): the
            # blend writes it directly, ordered on the current stream
            if out.device != self.device or out.dtype != t.float32 or \
                    tuple(out.shape) != (camera.height, camera.width, 3) or \
                    not out.is_contiguous():
                raise ValueError("out tensor must be a contiguous float32 (h, w, 3) tensor on "
                                 "the session's device")
            image = out
            device_out = True
        else:
            image = self._frame_image(camera)
        if not device_out:
            # host output: the blend writes the page-locked host array directly
            # (zero-copy, whole-row PCIe writes overlapped with the blend) - the
            # caller's array when it is page-locked, else a fresh page-locked
            # array (out=None) or a staging buffer copied into `out`.  Memory
            # the device cannot address takes a banded device->host copy.
            if out is None:
                target = self._fresh_output(camera)
                host = target
            else:
                if out.dtype != np.float32 or out.shape != (camera.height, camera.width, 3) \
                        or not out.flags.c_contiguous:
                    raise ValueError("out must be a C-contiguous float32 (h, w, 3) array")
                if self._zero_copy(out):
                    target = out
                else:
                    host = self._staging(camera)
                    target = host.numpy()
            staged = host is not None and out is not None  # copied into `out` below
            if (wait or staged) and self._zero_copy(target):
                image = target  # the blend writes the host array over PCIe
                a.sync = 1
            else:
                # device image + DMA copy; with wait=False the copy overlaps the
                # next frame's render and completes before wait()/recycling
                a.host_image = target.ctypes.data
                a.sync = 1 if (wait or staged) else 0
        a.image = image.ctypes.data if isinstance(image, np.ndarray) else image.data_ptr()
        stream = _device.sptr()
        st = self._stats
        # one call: visibility, page table, uploads, render graph, and for
        # host output the banded image copy (waits for the frame)
        _lib.check(lib.vms_session_frame(self._h, ctypes.byref(a), ctypes.byref(st), stream),
                   "render_frame")
        usage = st.occupied_entries / self.capacity
        if self.lod_enabled:
            adapt_thresholds(self.controller, usage, frame_index)
        h1 = time.perf_counter()
        levels = self.scene.lod_levels
        stats = {
            "frame": frame_index,
            "required_pages": int(st.required),
            "resident_pages": int(st.resident),
            "resident_per_level": tuple(int(st.resident_per_level[k]) for k in range(levels)),
            "planned_copies": int(st.planned),
            "missing_pages": int(st.missing),
            "bytes_copied": int(st.bytes_copied),
            "usage": usage,
            "lod_step": self.controller.step,
            "thresholds": tuple(float(x) for x in self.controller.thresholds),
            "time_visibility": st.ms_vis / 1e3,
            "time_reduce": 0.0,
            "time_update": st.host_update_s,
            "time_copy": st.ms_copy / 1e3,
            "time_sort": (st.ms_preprocess + st.ms_sort) / 1e3,
            "time_render": (st.ms_tiles + st.ms_blend) / 1e3,
            "time_preprocess": st.ms_preprocess / 1e3,
            "time_tiles": st.ms_tiles / 1e3,
            "time_blend": st.ms_blend / 1e3,
            "time_device_frame": st.ms_frame / 1e3,
            "time_host_gather": st.ms_host_gather / 1e3,
            "time_frame_wall": h1 - h0,
            "n_kept": int(st.n_kept),
            "n_instances": int(st.n_inst),
            "n_need": int(st.n_need),
            "overflow": int(st.overflow),
            "n_resident_records": int(st.n_res),
            "n_chunks": int(st.n_chunks),
            "n_tris": int(st.n_tris),
        }
        if device_out:
            return image, stats
        if out is None:
            return host, stats
        if host is not None:
            out[...] = host.numpy()
        return out, stats

    def _fresh_output(self, camera):
        """A page-locked (h, w, 3) array nobody else holds: the reference
        returns a new array per frame, so a buffer is reused only once every
        array handed out from it has been dropped by the caller (its
        reference count is back to the pool's own)."""
        import sys

        t = _device.torch()
        key = (camera.height, camera.width)
        pool = self.__dict__.setdefault("_out_pool", {}).setdefault(key, [])
        for i in range(len(pool)):
            # references: the pool's tuple and getrefcount's argument
            if sys.getrefcount(pool[i][1]) <= 2:
                return pool[i][1]
        # page-locking synchronises the device and takes milliseconds: grow
        # the pool to what a pipelined caller needs in one go (the frames in
        # flight, the one being handed over and the one being submitted)
        first = None
        for _ in range(max(1, self.slots + 2 - len(pool))):
            ten = t.empty((camera.height, camera.width, 3), dtype=t.float32, pin_memory=True)
            pool.append((ten, ten.numpy()))
            first = pool[-1][1] if first is None else first
        while len(pool) > 64:  # the caller keeps frames: stop tracking the oldest
            del pool[0]
        return first

    def _zero_copy(self, arr) -> bool:
        # asked every call (cudaPointerGetAttributes is cheap): a cached answer
        # keyed by address could outlive the buffer it was asked about
        return bool(self._lib.vms_host_accessible(arr.ctypes.data)) and bool(
            self._lib.vms_host_accessible(arr.ctypes.data + arr.nbytes - 1))

    def _staging(self, camera):
        t = _device.torch()
        key = (camera.height, camera.width)
        if self._pinned_out is None or self._pinned_out[0] != key:
            self._pinned_out = (key, t.empty((camera.height, camera.width, 3), dtype=t.float32)
                                .pin_memory())
        return self._pinned_out[1]

    @property
    def slots(self) -> int:
        """Frames the session keeps in flight: render_frame(i) waits for
        frame i - slots (VMSPLAT_SLOTS, default 4)."""
        return int(self._lib.vms_session_slots(self._h))

    def prepare(self, camera) -> None:
        """Allocate the render workspaces for the camera's resolution now
        (otherwise the first frame does it); the page cache stays cold."""
        _lib.check(self._lib.vms_session_prepare(self._h, int(camera.width), int(camera.height)),
                   "prepare")

    def wait(self, back: int = 0):
        """Block until the last submitted frame (back=0) or one before it
        (back < slots) is complete - for ``render_frame(..., wait=False)``."""
        _lib.check(self._lib.vms_session_wait(self._h, int(back)), "wait")

    def flush(self):
        """Wait for the last frame (device-output mode); returns its device
        counters (kept splats, tile instances, overflow, needed)."""
        cnt = (ctypes.c_uint32 * 4)()
        _lib.check(self._lib.vms_session_counters(self._h, cnt, _device.sptr()), "flush")
        return tuple(int(x) for x in cnt)

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



def fill_frame_cameras(args, camera, vis_scale: float, dot_mode: int) -> None:
    """args.cam / args.vis_cam = camera.struct(), camera.scaled(vis_scale)
    .struct() - the same numbers (quat_to_matrix's elementwise FP64
    arithmetic in the same order, the same focal and rounding), without
    building NumPy arrays and a second validated Camera each frame."""
    w, x, y, z = (float(v) for v in camera.orientation)
    rot = (1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
           2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
           2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y))
    pos = [float(v) for v in camera.position]
    t = float(np.tan(camera.fov_y / 2.0))
    vw = max(1, int(round(camera.width * vis_scale)))
    vh = max(1, int(round(camera.height * vis_scale)))
    for c, wd, ht in ((args.cam, camera.width, camera.height), (args.vis_cam, vw, vh)):
        c.pos[0], c.pos[1], c.pos[2] = pos
        for i in range(9):
            c.rot[i] = rot[i]
        c.focal = (ht / 2.0) / t
        c.half_w = wd / 2.0
        c.half_h = ht / 2.0
        c.near = float(camera.near)
        c.width = int(wd)
        c.height = int(ht)
        c.dot_mode = int(dot_mode)


def _mem_available() -> int:
    try:
        with open("/proc/meminfo") as fh:
            for ln in fh:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return 1 << 62


def _on_tmpfs(path) -> bool:
    """True if ``path`` lives on a tmpfs mount (its pages ARE host DRAM)."""
    import os

    try:
        real = os.path.realpath(path)
        best, kind = "", ""
        with open("/proc/mounts") as fh:
            for ln in fh:
                parts = ln.split()
                if len(parts) >= 3:
                    mnt = parts[1].replace("\\040", " ")
                    if (real == mnt or real.startswith(mnt.rstrip("/") + "/")) and \
                            len(mnt) > len(best):
                        best, kind = mnt, parts[2]
        return kind == "tmpfs"
    except OSError:
        return False


class HostScene:
    """The host-resident page source of a scene: its GAUS section (every LOD
    level) page-locked and mapped into the device address space, so page
    uploads are DMA from it (runtime.py:362-374 ``execute_copies`` reads the
    same rows through ``SceneFile.page_records``).

    A ``.vms`` file on tmpfs (host DRAM; e.g. /dev/shm) is page-locked IN
    PLACE: the record section is mapped shared (the driver cannot pin a
    read-only file mapping, so this mapping is read-write; it is registered
    with cudaHostRegisterReadOnly and never written) and registered - no copy
    is made, and every session, and every process (one per GPU) that maps
    the same file, streams from the same physical pages.  Any other source
    (a file on disk, an in-memory array) is copied once into page-locked
    memory per process; one HostScene per source is shared by all sessions
    of the process.
    """

    _live: dict = {}

    def __init__(self, scene):
        import os

        t = _device.torch()
        g = scene.gaussians
        self.rows = int(len(g))
        self._base = None
        self._tensor = None
        self._array = None
        path = getattr(scene, "path", None)
        if isinstance(g, np.memmap) and self.rows and path and _on_tmpfs(path) and \
                os.access(path, os.W_OK):
            lib = _lib.load()
            mm = np.memmap(path, dtype="<f4", mode="r+", offset=int(scene.gaus_offset),
                           shape=(self.rows, RECORD_SIZE))
            base = ctypes.c_void_p()
            st = lib.vms_host_register(mm.ctypes.data, mm.nbytes, 1, ctypes.byref(base))
            if st == _lib.VMS_OK:
                self._lib = lib
                self._base = base
                self._array = mm
                self.ptr = int(mm.ctypes.data)
                self.kind = "registered-tmpfs-mapping"
                return
            import warnings

            warnings.warn("cudaHostRegister of the scene mapping failed (%s)"
                          % lib.vms_last_error().decode(), RuntimeWarning)
        if g.nbytes > _mem_available() // 2:
            # a private copy would not fit next to the source
            raise MemoryError(f"the {g.nbytes >> 20} MB scene is neither a tmpfs file that "
                              "can be page-locked in place nor small enough for a private "
                              "page-locked copy; use upload_mode=2 (streaming from the mapping)")
        host = t.empty((max(self.rows, 1), RECORD_SIZE), dtype=t.float32).pin_memory()
        hv = host.numpy()
        step = max(1, (256 << 20) // RECORD_BYTES)
        for a in range(0, self.rows, step):
            hv[a:a + step] = g[a:a + step]
        self._tensor = host
        self.ptr = int(host.data_ptr())
        self.kind = "pinned-copy"

    def __del__(self):
        if getattr(self, "_base", None) is not None:
            self._lib.vms_host_unregister(self._base)
            self._base = None

    @classmethod
    def of(cls, scene) -> "HostScene":
        import weakref

        g = scene.gaussians
        if isinstance(g, np.memmap):
            key = ("mmap", getattr(g, "filename", None), int(g.offset), int(len(g)),
                   int(g.ctypes.data))
        else:
            key = ("array", id(g), int(g.ctypes.data), int(len(g)))
        ref = cls._live.get(key)
        hs = ref() if ref is not None else None
        if hs is None:
            hs = cls(scene)
            cls._live[key] = weakref.ref(hs)
        return hs
