"""View sharding across GPUs.

Independent camera views of a trajectory are split into contiguous blocks,
one per rank; every rank owns a full session (page table, device page pool)
over the one shared host-resident scene (a tmpfs `.vms` page-locked in
place by every rank, runtime.HostScene) and renders only its block, so there
is no data-path collective.  The only collective is the final gather of per-frame
stats rows (and optionally images) to rank 0 — NCCL over NVLink on GPUs, gloo
in the CPU tests.  Frame indices stay global, so each shard's page-table LRU
stamps match a single-process session started at the block's first frame.
"""

from __future__ import annotations

import numpy as np

STATS_COLUMNS = ("frame", "required_pages", "missing_pages", "bytes_copied", "resident_pages",
                 "planned_copies")


def frame_block(rank: int, world: int, frame_count: int):
    """Contiguous block [start, stop) of trajectory frames for ``rank``."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    return rank * frame_count // world, (rank + 1) * frame_count // world


def shard_frame(start: int, i: int, frame_count: int) -> int:
    """Trajectory frame of a rank's i-th frame: its block start + i.  A rank
    asked for more frames than its block holds continues into the following
    blocks, and the path wraps from its last frame to frame 0 (the camera
    jumps back to the start; frame indices keep increasing, so the page
    table sees a new viewpoint, not a repeated frame)."""
    return (start + i) % frame_count


def stats_rows(stats) -> np.ndarray:
    return np.array([[int(s[c]) for c in STATS_COLUMNS] for s in stats], dtype=np.int64)


def gather_rows(rows: np.ndarray, dist, device=None):
    """Gather equally-shaped int64 stats blocks to rank 0 (None elsewhere).
    Works with any torch.distributed backend (NCCL needs CUDA tensors)."""
    import torch

    t = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.int64))
    if device is not None:
        t = t.to(device)
    world = dist.get_world_size()
    # blocks may differ in length by one frame: pad to the max with -1 rows
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    m = int(max(int(s.item()) for s in sizes))
    pad = torch.full((m, t.shape[1]), -1, dtype=torch.int64, device=t.device)
    pad[: t.shape[0]] = t
    out = [torch.empty_like(pad) for _ in range(world)] if dist.get_rank() == 0 else None
    dist.gather(pad, out, dst=0)
    if dist.get_rank() != 0:
        return None
    parts = [o[: int(s.item())].cpu().numpy() for o, s in zip(out, sizes)]
    return np.concatenate(parts, axis=0)


def render_shard(session, trajectory, rank: int, world: int, frames: int | None = None,
                 out="device"):
    """Render this rank's block (or ``frames`` consecutive frames from the
    block start, see ``shard_frame``).  Returns the list of stats dicts."""
    F = trajectory.frame_count
    start, stop = frame_block(rank, world, F)
    n = (stop - start) if frames is None else frames
    stats = []
    for i in range(n):
        cam = trajectory.frame_camera(shard_frame(start, i, F))
        _, st = session.render_frame(cam, start + i, out=out)
        stats.append(st)
    return stats
