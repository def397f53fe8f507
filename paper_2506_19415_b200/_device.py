"""Device plumbing: CUDA availability, cached workspaces, host<->device
conversion and the BLAS dot-order probe.  PyTorch is used only for device
memory, pinned host memory and streams; all compute is in libvmsplat_b200.so.
"""

from __future__ import annotations

import ctypes

import numpy as np

from paper_2506_19415_b200 import _lib
from paper_2506_19415_b200.errors import CudaError

_torch = None
_ws = {}
_dot_mode = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise CudaError("a CUDA device is required: this package has no CPU fallback")
    _lib.load()
    return t


def workspace(name: str, nbytes: int, device=None):
    """A cached uint8 device buffer of at least ``nbytes`` (grown by 1.25x)."""
    t = require_cuda()
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    key = (name, str(dev))
    buf = _ws.get(key)
    if buf is None or buf.numel() < nbytes:
        size = max(int(nbytes * 1.25), 1 << 16)
        buf = t.empty(size, dtype=t.uint8, device=dev)
        _ws[key] = buf
    return buf


def release_workspaces():
    _ws.clear()


def is_torch(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor)


def to_dev(x, dtype, device=None):
    """numpy / torch -> contiguous CUDA tensor of ``dtype`` (numpy dtype)."""
    t = require_cuda()
    tdt = {np.float32: t.float32, np.float64: t.float64, np.int32: t.int32,
           np.uint32: t.uint32, np.int64: t.int64, np.uint8: t.uint8}[np.dtype(dtype).type]
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    if isinstance(x, t.Tensor):
        return x.to(device=dev, dtype=tdt).contiguous()
    a = np.ascontiguousarray(x, dtype=dtype)
    return t.from_numpy(a).to(dev, non_blocking=False)


def stream():
    return torch().cuda.current_stream()


def sptr():
    return _lib.stream_ptr(stream())


def camera_struct(position, rot, focal, width, height, near, dot_mode) -> _lib.Camera:
    c = _lib.Camera()
    for i in range(3):
        c.pos[i] = float(position[i])
    r = np.asarray(rot, dtype=np.float64).reshape(9)
    for i in range(9):
        c.rot[i] = float(r[i])
    c.focal = float(focal)
    c.half_w = width / 2.0
    c.half_h = height / 2.0
    c.near = float(near)
    c.width = int(width)
    c.height = int(height)
    c.dot_mode = int(dot_mode)
    return c


def probe_dot_mode() -> tuple[int, bool]:
    """Pick the FP64 dot order that reproduces this host's ``(p - pos) @ R``
    (NumPy -> BLAS) bit for bit.  Returns
    (mode, exact); exact is False when neither order matches."""
    global _dot_mode
    if _dot_mode is not None:
        return _dot_mode
    t = require_cuda()
    rng = np.random.default_rng(20250619)
    from paper_2506_19415_b200.gaussians import quat_to_matrix

    result = None
    for mode in (0, 1):
        ok = True
        for n in (7, 311, 20011):
            pts = rng.uniform(-50, 50, size=(n, 3)).astype(np.float32).astype(np.float64)
            q = rng.normal(size=4)
            q /= np.linalg.norm(q)
            pos = rng.uniform(-5, 5, size=3)
            rot = quat_to_matrix(q)
            host = (pts - pos) @ rot
            cam = camera_struct(pos, rot, 1.0, 1, 1, 0.05, mode)
            dp = t.from_numpy(pts).cuda()
            out = t.empty_like(dp)
            _lib.check(_lib.load().vms_world_to_view(dp.data_ptr(), n, ctypes.byref(cam),
                                                     out.data_ptr(), sptr()), "probe")
            if not np.array_equal(out.cpu().numpy().view(np.uint64), host.view(np.uint64)):
                ok = False
                break
        if ok:
            result = (mode, True)
            break
    if result is None:
        import warnings

        warnings.warn("neither FP64 dot order reproduces this host's BLAS (p - pos) @ R bit "
                      "for bit: visibility page sets and sort keys may differ from the "
                      "reference in rare ties (SURVEY Appendix A.1)", RuntimeWarning)
        result = (0, False)
    _dot_mode = result
    return result
