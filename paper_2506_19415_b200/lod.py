"""Per-page level-of-detail pyramid on the GPU - drop-in for ``vmsplat.lod``
(pkg/src/vmsplat/lod.py), SURVEY §8(f) F3.

Same names, defaults, argument meaning, errors and results as the
reference module: ``build_pyramid`` returns the reference's level arrays bit
for bit, ``cluster_page`` the reference's assignment (and advances the
caller's Philox ``Generator`` exactly as the reference's draws do),
``merge_cluster`` the reference's merged record.  All three run the
kernels of csrc/lod.cu through the C ABI ``vms_lod_level``: per page one
CTA seeds k-means++ (``lod_seed_k``) and one runs the Lloyd iterations and
the merge (``lod_lloyd_k``), every page of a level in the same launches.
There is no CPU path: without a GPU these raise ``CudaError``.

Limits of this implementation: at most 4096 records per page (the k-means
arrays of a page live in shared memory), and ``rng`` must be a NumPy
``Generator`` over the Philox bit generator (the reference's own per-page
streams always are, lod.py:44-46).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from paper_2506_19415_b200 import _device, _lib
from paper_2506_19415_b200.errors import InvariantViolation
from paper_2506_19415_b200.gaussians import RECORD_SIZE

DEFAULT_LEVELS = 4
DEFAULT_SCALE_FACTOR = 2.0 ** (1.0 / 3.0)  # volume doubles for a 2-to-1 merge
DEFAULT_KMEANS_ITERS = 50
MAX_PAGE_RECORDS = 4096


@dataclass(frozen=True)
class AttributeWeights:
    """Distance weights for clustering (lod.py:26-41); position dominates."""

    position: float = 1.0
    rotation: float = 0.1
    scale: float = 0.1
    opacity: float = 0.05
    sh_dc: float = 0.1

    def validate(self) -> None:
        for name in ("position", "rotation", "scale", "opacity", "sh_dc"):
            if getattr(self, name) < 0:
                raise InvariantViolation(f"negative weight {name}")


def _page_rng(seed: int, page_id: int) -> np.random.Generator:
    """The reference's per-page stream (lod.py:44-46): Philox keyed
    (seed, 1), counter (page_id, 0, 0, 0)."""
    return np.random.Generator(np.random.Philox(key=[seed, 1], counter=[page_id, 0, 0, 0]))


def _fresh_state(seed: int, page_id: int) -> _lib.Philox:
    """State of ``_page_rng(seed, page_id)`` before its first draw."""
    st = _lib.Philox()
    st.counter[0] = page_id & 0xFFFFFFFFFFFFFFFF
    st.key[0] = seed & 0xFFFFFFFFFFFFFFFF
    st.key[1] = 1
    st.buffer_pos = 4
    return st


def _state_of(gen: np.random.Generator) -> _lib.Philox:
    s = gen.bit_generator.state
    if s.get("bit_generator") != "Philox":
        raise ValueError("the GPU k-means draws from NumPy's Philox stream; got "
                         f"{s.get('bit_generator')}")
    st = _lib.Philox()
    for i in range(4):
        st.counter[i] = int(s["state"]["counter"][i])
        st.buffer[i] = int(s["buffer"][i])
    for i in range(2):
        st.key[i] = int(s["state"]["key"][i])
    st.buffer_pos = int(s["buffer_pos"])
    st.has_uint32 = int(s["has_uint32"])
    st.uinteger = int(s["uinteger"])
    return st


def _restore(gen: np.random.Generator, st: _lib.Philox) -> None:
    gen.bit_generator.state = {
        "bit_generator": "Philox",
        "state": {"counter": np.array(list(st.counter), dtype=np.uint64),
                  "key": np.array(list(st.key), dtype=np.uint64)},
        "buffer": np.array(list(st.buffer), dtype=np.uint64),
        "buffer_pos": int(st.buffer_pos),
        "has_uint32": int(st.has_uint32),
        "uinteger": int(st.uinteger),
    }


def _params(weights: AttributeWeights, scale_factor: float, max_iters: int, k: int):
    p = _lib.LodParams()
    for i, v in enumerate((weights.position, weights.rotation, weights.scale,
                           weights.opacity, weights.sh_dc)):
        p.weights[i] = float(v)
    p.scale_factor = float(scale_factor)
    p.max_iters = int(max_iters)
    p.k = int(k)
    return p


def _states_tensor(states):
    t = _device.require_cuda()
    raw = b"".join(bytes(s) for s in states)
    return t.frombuffer(bytearray(raw), dtype=t.uint8).cuda()


def _states_from(dev, n):
    raw = dev.cpu().numpy().tobytes()
    sz = ctypes.sizeof(_lib.Philox)
    return [_lib.Philox.from_buffer_copy(raw[i * sz:(i + 1) * sz]) for i in range(n)]


def _launch(rec_dev, pages, rows_in, out_dev, rows_out, params, rng_dev, assign_dev):
    """One vms_lod_level call; returns the per-page status array (host)."""
    t = _device.require_cuda()
    lib = _lib.load()
    if rows_in > MAX_PAGE_RECORDS:
        raise ValueError(f"GPU k-means supports at most {MAX_PAGE_RECORDS} records per page "
                         f"(got {rows_in})")
    nbytes = int(lib.vms_lod_workspace_bytes(pages, rows_in))
    ws = _device.workspace("lod", max(nbytes, 16))
    status = t.zeros(max(pages, 1), dtype=t.int32, device=rec_dev.device)
    _lib.check(lib.vms_lod_level(rec_dev.data_ptr(), pages, rows_in,
                                 out_dev.data_ptr() if out_dev is not None else None, rows_out,
                                 ctypes.byref(params), rng_dev.data_ptr(),
                                 assign_dev.data_ptr() if assign_dev is not None else None,
                                 status.data_ptr(), ws.data_ptr(), ws.numel(), _device.sptr()),
               "lod_level")
    _device.stream().synchronize()
    return status.cpu().numpy()[:pages]


def cluster_page(page_records: np.ndarray, k: int, weights: AttributeWeights = AttributeWeights(),
                 max_iters: int = DEFAULT_KMEANS_ITERS, rng: np.random.Generator | None = None,
                 seed: int = 0) -> np.ndarray:
    """Lloyd k-means over weighted attributes; a cluster index per record
    (lod.py:83-131).  Empty clusters are reseeded at the point farthest from
    its center; stops at the assignment fixpoint or ``max_iters``."""
    weights.validate()
    recs = np.ascontiguousarray(np.asarray(page_records, dtype=np.float32).reshape(-1, RECORD_SIZE))
    m = len(recs)
    if k >= m:
        return np.arange(m, dtype=np.int64)
    if k < 1:
        raise InvariantViolation("cluster count must be >= 1")
    if rng is None:
        rng = _page_rng(seed, 0)
    t = _device.require_cuda()
    dev = _device.to_dev(recs, np.float32)
    rng_dev = _states_tensor([_state_of(rng)])
    assign = t.full((m,), -1, dtype=t.int32, device=dev.device)
    status = _launch(dev, 1, m, None, 0, _params(weights, DEFAULT_SCALE_FACTOR, max_iters, k),
                     rng_dev, assign)
    if status[0] == 1:
        raise InvariantViolation("k-means inertia increased")
    _restore(rng, _states_from(rng_dev, 1)[0])
    return assign.cpu().numpy().astype(np.int64)


def merge_cluster(members: np.ndarray, scale_factor: float = DEFAULT_SCALE_FACTOR) -> np.ndarray:
    """Merge member records into one (lod.py:134-154): means, except the
    rotation (normalized mean of hemisphere-aligned quaternions) and the
    scale (times the volume-compensation factor)."""
    recs = np.ascontiguousarray(np.asarray(members, dtype=np.float32).reshape(-1, RECORD_SIZE))
    if len(recs) == 0:
        raise InvariantViolation("cannot merge an empty cluster")
    t = _device.require_cuda()
    dev = _device.to_dev(recs, np.float32)
    out = t.empty(RECORD_SIZE, dtype=t.float32, device=dev.device)
    _launch(dev, 1, len(recs), out, 1, _params(AttributeWeights(), scale_factor, 0, -1),
            _states_tensor([_fresh_state(0, 0)]), None)
    return out.cpu().numpy()


def build_pyramid(level0: np.ndarray, page_size: int, level_count: int = DEFAULT_LEVELS,
                  scale_factor: float = DEFAULT_SCALE_FACTOR, max_iters: int = DEFAULT_KMEANS_ITERS,
                  seed: int = 7, weights: AttributeWeights = AttributeWeights()) -> list:
    """Per-level record arrays from padded level-0 pages (lod.py:179-226):
    element k holds page_count pages of page_size / 2^k records; element 0
    is the input, untouched.  Every level of every page is clustered and
    merged on the GPU (one launch per level)."""
    if level_count < 1:
        raise InvariantViolation("level_count must be >= 1")
    if page_size % (1 << (level_count - 1)) != 0:
        raise InvariantViolation(f"page_size {page_size} not divisible by 2^{level_count - 1}")
    level0 = np.asarray(level0, dtype=np.float32).reshape(-1, RECORD_SIZE)
    if page_size and len(level0) % page_size != 0:
        raise InvariantViolation("level-0 size is not a whole number of pages")
    page_count = len(level0) // page_size if page_size else 0
    out = [level0]
    if level_count == 1 or page_count == 0:
        return out + [np.zeros((0, RECORD_SIZE), dtype=np.float32) for _ in range(level_count - 1)]
    weights.validate()
    t = _device.require_cuda()
    cur = _device.to_dev(level0, np.float32)
    rng_dev = _states_tensor([_fresh_state(seed, p + 1) for p in range(page_count)])
    params = _params(weights, scale_factor, max_iters, 0)
    for k in range(1, level_count):
        rows_in, rows_out = page_size >> (k - 1), page_size >> k
        nxt = t.empty(page_count * rows_out * RECORD_SIZE, dtype=t.float32, device=cur.device)
        status = _launch(cur, page_count, rows_in, nxt, rows_out, params, rng_dev, None)
        bad = np.flatnonzero(status)
        if len(bad):
            p = int(bad[0])
            if status[p] == 1:
                raise InvariantViolation("k-means inertia increased")
            raise InvariantViolation(f"page {p + 1}: level {k} overflow")
        out.append(nxt.cpu().numpy().reshape(-1, RECORD_SIZE))
        cur = nxt
    return out


__all__ = ["AttributeWeights", "DEFAULT_KMEANS_ITERS", "DEFAULT_LEVELS", "DEFAULT_SCALE_FACTOR",
           "build_pyramid", "cluster_page", "merge_cluster"]
