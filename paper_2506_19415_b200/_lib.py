"""ctypes binding of libvmsplat_b200.so — the role the reference's Cython
module plays for `vmsplat.kernels` (pkg/src/vmsplat/kernels/__init__.py:13-21),
without a fallback: if the CUDA library is missing the import fails loudly.

Structs mirror include/vmsplat_b200.h field for field.
"""

from __future__ import annotations

import ctypes
import os

from paper_2506_19415_b200.errors import CudaError, InvariantViolation

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvmsplat_b200.so")

VMS_OK = 0
VMS_ERR_INVALID = 1
VMS_ERR_RANGE = 2
VMS_ERR_CUDA = 3
VMS_ERR_NOMEM = 4
VMS_ERR_INVARIANT = 5

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U32 = ctypes.c_uint32
SZ = ctypes.c_size_t
D = ctypes.c_double


class Camera(ctypes.Structure):
    _fields_ = [("pos", D * 3), ("rot", D * 9), ("focal", D), ("half_w", D), ("half_h", D),
                ("near", D), ("width", I32), ("height", I32), ("dot_mode", I32),
                ("pad_", I32)]


class Lod(ctypes.Structure):
    _fields_ = [("thresholds", D * 8), ("count", I32), ("pad_", I32)]


class RequiredOut(ctypes.Structure):
    _fields_ = [("pid", P), ("enc", P), ("direct", P), ("level", P), ("meta", P)]


class VisArgs(ctypes.Structure):
    _fields_ = [("cam", Camera), ("verts", P), ("faces", P), ("face_page", P),
                ("n_faces", U32), ("page_count", U32), ("link_off", P), ("link_tgt", P),
                ("lod", Lod), ("id_image", P), ("invz_image", P), ("depth_out", P),
                ("direct_out", P), ("out", RequiredOut), ("workspace", P)]


class Chunk(ctypes.Structure):
    _fields_ = [("row", U32), ("gather", U32), ("count", U32), ("pad_", U32)]


class RenderArgs(ctypes.Structure):
    _fields_ = [("cam", Camera), ("pool", P), ("chunks", P), ("n_chunks", U32),
                ("n_splats", U32), ("n_cap", U32), ("m_cap", U32), ("image", P),
                ("accumulate", I32), ("exact", I32), ("counters_out", P), ("workspace", P),
                ("events", P * 4)]


class Copy(ctypes.Structure):
    _fields_ = [("src_offset", ctypes.c_uint64), ("dst_offset", ctypes.c_uint64),
                ("nbytes", ctypes.c_uint64)]


class SessionDesc(ctypes.Structure):
    _fields_ = [("host_records", P), ("host_rows", ctypes.c_uint64), ("page_size", U32),
                ("lod_levels", U32), ("page_counts", U32 * 16), ("page_count", U32),
                ("n_faces", U32), ("verts", P), ("faces", P), ("face_page", P),
                ("link_off", P), ("link_tgt", P), ("pool", P), ("capacity", U32),
                ("m_cap", U32), ("vis_ws", P), ("render_ws", P),
                ("render_ws_bytes", ctypes.c_uint64), ("width", I32), ("height", I32),
                ("exact", I32), ("upload_mode", I32), ("host_fd", I32),
                ("host_fd_offset", ctypes.c_uint64), ("device_table", I32), ("pad_", I32)]


class FrameArgs(ctypes.Structure):
    _fields_ = [("cam", Camera), ("vis_cam", Camera), ("lod", Lod), ("frame", I64),
                ("budget", D), ("image", P), ("host_image", P), ("timing", I32),
                ("sync", I32)]


class FrameStats(ctypes.Structure):
    _fields_ = [("required", U32), ("resident", U32), ("planned", U32), ("missing", U32),
                ("bytes_copied", ctypes.c_uint64), ("occupied_entries", U32),
                ("capacity", U32), ("n_tris", U32), ("n_chunks", U32), ("n_res", U32),
                ("n_kept", U32), ("n_inst", U32), ("overflow", U32), ("n_need", U32),
                ("pad_", U32), ("resident_per_level", I64 * 16), ("ms_vis", ctypes.c_float),
                ("ms_copy", ctypes.c_float), ("ms_preprocess", ctypes.c_float),
                ("ms_sort", ctypes.c_float), ("ms_tiles", ctypes.c_float),
                ("ms_blend", ctypes.c_float), ("ms_frame", ctypes.c_float),
                ("ms_host_gather", ctypes.c_float), ("host_update_s", D)]


class Philox(ctypes.Structure):
    """NumPy Philox bit-generator state (include/vmsplat_b200.h vms_philox)."""
    _fields_ = [("counter", ctypes.c_uint64 * 4), ("key", ctypes.c_uint64 * 2),
                ("buffer", ctypes.c_uint64 * 4), ("buffer_pos", I32), ("has_uint32", I32),
                ("uinteger", U32), ("_pad", U32)]


class DptFrame(ctypes.Structure):
    _fields_ = [("frame", I64), ("budget", D)]


class DptStats(ctypes.Structure):
    _fields_ = [("n_req", U32), ("n_plan", U32), ("missing", U32), ("resident", U32),
                ("occupied", U32), ("bad", U32), ("plan_overflow", U32), ("n_chunks", U32),
                ("n_records", U32), ("pad_", U32), ("resident_per_level", U32 * 16)]


class LodParams(ctypes.Structure):
    _fields_ = [("weights", D * 5), ("scale_factor", D), ("max_iters", I32), ("k", I32)]


# name -> (restype, argtypes); every symbol include/vmsplat_b200.h declares
SIGNATURES = {
    "vms_last_error": (ctypes.c_char_p, []),
    "vms_abi_version": (I32, []),
    "vms_tile_size": (I32, []),
    "vms_profile_enable": (I32, [I32]),
    "vms_profile_report": (I64, [P, I64]),
    "vms_composite_workspace_bytes": (SZ, [I64, I64, I32, I32]),
    "vms_composite_splats": (I32, [P, P, P, P, P, I64, I64, P, I32, I32, I32, P, SZ, P]),
    "vms_rasterize_workspace_bytes": (SZ, [I64]),
    "vms_rasterize_triangles": (I32, [P, P, I64, P, P, I32, I32, P, SZ, P]),
    "vms_radix_workspace_bytes": (SZ, [I64]),
    "vms_radix_sort_pairs": (I32, [P, P, I64, P, SZ, P]),
    "vms_world_to_view": (I32, [P, I64, ctypes.POINTER(Camera), P, P]),
    "vms_project_records": (I32, [P, I64, ctypes.POINTER(Camera), P, P, P, P, P, P, P]),
    "vms_evaluate_sh": (I32, [P, P, I64, P, P]),
    "vms_visibility_workspace_bytes": (SZ, [U32, U32]),
    "vms_visibility": (I32, [ctypes.POINTER(VisArgs), P]),
    "vms_reduce_visibility": (I32, [P, P, I64, U32, P, P, P, P, P, P, SZ, P]),
    "vms_upload_pages": (I32, [P, I64, P, P, I32, P]),
    "vms_render_workspace_bytes": (SZ, [U32, U32, I32, I32]),
    "vms_render": (I32, [ctypes.POINTER(RenderArgs), P]),
    "vms_pt_create": (P, [I64]),
    "vms_pt_destroy": (None, [P]),
    "vms_pt_update": (I32, [P, P, P, P, P, I64, I64, D, P, P, P, P, I64,
                            ctypes.POINTER(I64), ctypes.POINTER(I64)]),
    "vms_pt_capacity": (I64, [P]),
    "vms_pt_occupied": (I64, [P]),
    "vms_pt_resident_count": (I64, [P]),
    "vms_pt_resident": (I32, [P, P, P, P, I64]),
    "vms_pt_entries": (I32, [P, P, P, P, I32]),
    "vms_pt_resident_counts": (I32, [P, P, I32]),
    "vms_pt_check": (I32, [P]),
    "vms_pt_chunks": (I64, [P, I64, P, I64, ctypes.POINTER(I64)]),
    "vms_session_render_ws_bytes": (SZ, [U32, U32, U32, I32, I32]),
    "vms_session_create": (P, [ctypes.POINTER(SessionDesc)]),
    "vms_session_destroy": (None, [P]),
    "vms_session_table": (P, [P]),
    "vms_session_dpt": (P, [P]),
    "vms_session_cert_count": (I32, [P, P]),
    "vms_debug_cert_all": (I32, [I32]),
    "vms_debug_lane_lists": (I32, [I32, I32]),
    "vms_session_set_render_ws": (I32, [P, P, ctypes.c_uint64, U32, I32, I32]),
    "vms_session_frame": (I32, [P, ctypes.POINTER(FrameArgs), ctypes.POINTER(FrameStats), P]),
    "vms_session_counters": (I32, [P, P, P]),
    "vms_session_wait": (I32, [P, I32]),
    "vms_session_slots": (I32, [P]),
    "vms_session_prepare": (I32, [P, I32, I32]),
    "vms_host_accessible": (I32, [P]),
    "vms_host_register": (I32, [P, ctypes.c_uint64, I32, ctypes.POINTER(P)]),
    "vms_host_unregister": (I32, [P]),
    "vms_debug_blend_trace": (I32, [P]),
    "vms_debug_exp": (I32, [P, I64, P, P]),
    "vms_bvh_nearest_points": (I32, [P, I64, P, P, P, I64, P, P, I64, P, P, P, P]),
    "vms_lod_workspace_bytes": (SZ, [U32, U32]),
    "vms_dpt_create": (P, [I32, I32, I32]),
    "vms_dpt_destroy": (None, [P]),
    "vms_dpt_smem_bytes": (SZ, [P]),
    "vms_dpt_update": (I32, [P, P, P, P, P, P, P, P, P, P, P, I64, P, P]),
    "vms_dpt_chunks": (I32, [P, U32, P, I64, P, P]),
    "vms_dpt_state": (I32, [P, P, P, P, I32, P, P]),
    "vms_lod_level": (I32, [P, U32, U32, P, U32, ctypes.POINTER(LodParams), P, P, P, P, SZ, P]),
}

_lib = None


def load():
    """Load (and if needed build) the CUDA library; raise if impossible."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from paper_2506_19415_b200 import build as _build

            _build.build()
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.vms_abi_version() != 1:
            raise RuntimeError("libvmsplat_b200.so ABI version mismatch")
        _lib = lib
    return _lib


def check(status: int, what: str = "") -> None:
    if status == VMS_OK:
        return
    msg = load().vms_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status in (VMS_ERR_RANGE, VMS_ERR_INVARIANT):
        raise InvariantViolation(text)
    if status == VMS_ERR_INVALID:
        raise ValueError(text)
    if status == VMS_ERR_NOMEM:
        raise MemoryError(text)
    raise CudaError(text)


def profile_report() -> str:
    lib = load()
    n = lib.vms_profile_report(None, 0)
    buf = ctypes.create_string_buffer(int(n) + 1)
    lib.vms_profile_report(buf, n + 1)
    return buf.value.decode()


def ptr(t) -> int | None:
    """Raw address of a torch tensor / numpy array (None for None)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    return stream.cuda_stream
