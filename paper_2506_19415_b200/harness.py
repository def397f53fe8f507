"""Scripted-path benchmark harness: the caller of the hot path (SURVEY
section 8(f) row F1; reference pkg/src/vmsplat/harness.py).

``run_benchmark`` replays a camera path through ``VmSession.render_frame``
and records one ``FrameStats`` per frame; ``emit_reports`` writes the three
report files the reference writes - ``stats.csv`` (deterministic counters,
byte-identical to the reference for the same scene/path/config),
``timings.csv`` (stage durations) and ``summary.json`` (validated against the
reference's schema) - and ``write_frame`` dumps lossless frames.

Differences that are B200 choices, not API changes:
  * stage durations come from CUDA events on the device (the session's
    timing mode), with the host page-table time in ``update`` - the
    reference's ``time.perf_counter`` wall clock around NumPy stages has no
    meaning for work that is asynchronous on a GPU.  ``summary.json`` names
    the clock (``timer.clock``).
  * ``vm=False`` (the no-paging ablation, harness.py:111-146) renders all
    level-0 records through the same device render path (``FlatRenderer``).
  * ``run_sharded`` renders contiguous blocks of the path on several ranks
    (one GPU each) and gathers the FrameStats rows to rank 0 (NCCL on GPUs,
    gloo in the CPU tests) before the reports are written.
"""

from __future__ import annotations

import csv
import json
import statistics
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from paper_2506_19415_b200.errors import DataError, InvariantViolation

STAGES = ("visibility", "reduce", "update", "copy", "sort", "render")
MEDIAN_FRAME_NOTE = "The median frame is not an actual frame"
DEVICE_CLOCK = "cuda events (device stage time; host page-table time in update)"


@dataclass(frozen=True)
class FrameStats:
    """One benchmark frame (harness.py:34-71): counters after the frame's
    copies, the controller's thresholds after its adaptation, and seconds
    per stage keyed by ``STAGES``."""

    frame: int
    required: int
    missing: int
    bytes_copied: int
    usage: float
    resident_per_level: tuple
    thresholds: tuple
    durations: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.missing > self.required:
            raise InvariantViolation(
                f"frame {self.frame}: missing {self.missing} > required {self.required}")
        if set(self.durations) != set(STAGES):
            raise InvariantViolation(f"frame {self.frame}: bad stage keys")
        bad = [k for k, v in self.durations.items() if v < 0]
        if bad:
            raise InvariantViolation(f"frame {self.frame}: {bad[0]} duration < 0")

    @property
    def resident(self) -> int:
        return int(sum(self.resident_per_level))

    @property
    def total_time(self) -> float:
        return float(sum(self.durations.values()))

    @classmethod
    def from_session(cls, frame: int, st: dict) -> "FrameStats":
        """From ``VmSession.render_frame``'s stats dict (runtime.py:471-488 keys)."""
        return cls(frame=frame, required=st["required_pages"], missing=st["missing_pages"],
                   bytes_copied=st["bytes_copied"], usage=st["usage"],
                   resident_per_level=tuple(st["resident_per_level"]),
                   thresholds=tuple(st["thresholds"]),
                   durations={s: float(st[f"time_{s}"]) for s in STAGES})


def level0_equivalents(stats: FrameStats) -> float:
    """Resident footprint in level-0 pages: a level-k page counts 1/2^k."""
    return float(sum(c / float(1 << k) for k, c in enumerate(stats.resident_per_level)))


@dataclass(frozen=True)
class BenchConfig:
    """Run knobs (harness.py:74-89); ``vm=False`` is the no-paging ablation."""

    buffer_pages: int = 500
    staging_pages: float = 40.0
    vis_scale: float = 0.25
    band: tuple = (0.5, 0.8)
    step: float = 0.05
    lod: bool = True
    links: bool = True
    vm: bool = True
    frame_limit: int = 0  # 0 = the whole path


def frames_to_run(path, config: BenchConfig) -> int:
    n = path.frame_count
    return min(n, config.frame_limit) if config.frame_limit > 0 else n


def make_session(scene, config: BenchConfig, **extra):
    from paper_2506_19415_b200.runtime import VmSession

    return VmSession(scene, buffer_pages=config.buffer_pages,
                     staging_pages=config.staging_pages, vis_scale=config.vis_scale,
                     band=config.band, step=config.step, lod_enabled=config.lod,
                     links_enabled=config.links, **extra)


def run_benchmark(scene, path, config: BenchConfig | None = None, frame_sink=None,
                  frames=None, session=None, pipelined: bool = False):
    """Replay ``path`` over ``scene``; returns the list of FrameStats
    (harness.py:101-181).  ``frame_sink(i, image)`` receives each frame
    (float32 (h, w, 3) host array); frames are not kept otherwise.
    B200 extensions: ``frames`` restricts the run to those frame indices, in
    order (a shard of the path); ``session`` reuses an existing one;
    ``pipelined`` keeps the session's slots full (frames i + 1 .. i + slots
    submitted before frame i goes to the sink), so each frame's transfer to
    the host overlaps the next frames' visibility pass and render (the durations are then not measured: zeros)."""
    cfg = config or BenchConfig()
    if scene.page_count == 0:
        raise DataError("benchmark needs a paged scene")
    indices = list(range(frames_to_run(path, cfg))) if frames is None else list(frames)
    if not cfg.vm:
        return _run_flat(scene, path, indices, frame_sink)
    s = session if session is not None else make_session(scene, cfg, timing=not pipelined)
    try:
        return _run_session(s, path, indices, frame_sink, pipelined)
    finally:
        if session is None and hasattr(s, "close"):
            s.close()


def _run_session(s, path, indices, frame_sink, pipelined):
    out = []
    if not pipelined:
        for i in indices:
            image, st = s.render_frame(path.frame_camera(i), i)
            out.append(FrameStats.from_session(i, st))
            if frame_sink is not None:
                frame_sink(i, image)
        return out
    # frames i - slots + 1 .. i in flight after submitting i: the session
    # recycles frame i - slots (its image copy complete) inside
    # render_frame(i), so that frame goes to the sink without a wait, and each
    # frame's copy to the host overlaps the next frames' visibility and render
    held = []  # (index, image) submitted, not yet handed over, oldest first
    depth = getattr(s, "slots", 2)
    for i in indices:
        image, st = s.render_frame(path.frame_camera(i), i, wait=False)
        out.append(FrameStats.from_session(i, {**st, **{f"time_{k}": 0.0 for k in STAGES}}))
        if len(held) == depth:
            done = held.pop(0)
            if frame_sink is not None:
                frame_sink(*done)
        held.append((i, image))
    for k, done in enumerate(held):
        s.wait(len(held) - 1 - k)
        if frame_sink is not None:
            frame_sink(*done)
    return out


def _run_flat(scene, path, indices, frame_sink):
    """No page table, no streaming: every level-0 record each frame; the
    skipped stages report zero so the CSV schema stays uniform."""
    import time

    from paper_2506_19415_b200 import _device
    from paper_2506_19415_b200.render import FlatRenderer

    t = _device.require_cuda()
    records = _device.to_dev(np.asarray(scene.gaussians[: scene.page_count * scene.page_size]),
                             np.float32)
    flat = FlatRenderer()
    resident = (scene.page_count,) + (0,) * (scene.lod_levels - 1)
    out = []
    for i in indices:
        cam = path.frame_camera(i)
        t.cuda.synchronize()
        t0 = time.perf_counter()
        image = flat.render(records, cam).cpu().numpy()
        dt = time.perf_counter() - t0
        out.append(FrameStats(frame=i, required=scene.page_count, missing=0, bytes_copied=0,
                              usage=1.0, resident_per_level=resident, thresholds=(),
                              durations={"visibility": 0.0, "reduce": 0.0, "update": 0.0,
                                         "copy": 0.0, "sort": 0.0, "render": dt}))
        if frame_sink is not None:
            frame_sink(i, image)
    return out


# -- frames -----------------------------------------------------------------------
def write_frame(path, image: np.ndarray, bits: int = 8) -> None:
    """Lossless dump of one linear [0, 1] frame, no gamma (harness.py:186-208):
    8-bit PNG, or 16-bit binary PPM (P6, maxval 65535, big-endian)."""
    img = np.asarray(image, dtype=np.float64)
    if img.ndim != 3 or img.shape[2] != 3:
        raise DataError(f"expected (h, w, 3) image, got {img.shape}")
    img = np.clip(img, 0.0, 1.0)
    target = Path(path)
    if bits == 16:
        h, w = img.shape[:2]
        body = np.round(img * 65535.0).astype(">u2").tobytes()
        target.write_bytes(b"P6\n%d %d\n65535\n" % (w, h) + body)
        return
    if bits != 8:
        raise DataError(f"bits must be 8 or 16, got {bits}")
    from PIL import Image

    Image.fromarray(np.round(img * 255.0).astype(np.uint8), "RGB").save(target, format="PNG")


def frame_name(index: int, bits: int = 8) -> str:
    return "frame_%05d.%s" % (index, "png" if bits == 8 else "ppm")


# -- summary schema (harness.py:217-296), built from its parts ---------------------
def _object(props: dict, required=None, extra=False) -> dict:
    return {"type": "object", "properties": props,
            "required": list(props) if required is None else list(required),
            "additionalProperties": extra}


_NONNEG_NUM = {"type": "number", "minimum": 0}
_NONNEG_INT = {"type": "integer", "minimum": 0}
_STAGE_TIMES = _object({name: dict(_NONNEG_NUM) for name in STAGES})
_REAL_FRAME = _object({"frame": _NONNEG_INT, "durations_s": _STAGE_TIMES, "total_s": _NONNEG_NUM,
                       "resident_pages": _NONNEG_INT, "required_pages": _NONNEG_INT,
                       "missing_pages": _NONNEG_INT, "bytes_copied": _NONNEG_INT})
_MEDIAN_FRAME = _object({"note": {"const": MEDIAN_FRAME_NOTE}, "durations_s": _STAGE_TIMES,
                         "total_s": _NONNEG_NUM})
SUMMARY_SCHEMA = dict(
    _object({
        "frame_count": {"type": "integer", "minimum": 1},
        "timer": _object({"clock": {"type": "string"}, "resolution_s": _NONNEG_NUM}),
        "stage_medians_s": _STAGE_TIMES,
        "frames": _object({"most_pages": _REAL_FRAME, "median": _MEDIAN_FRAME,
                           "shortest": _REAL_FRAME, "largest_transfer": _REAL_FRAME}),
    }),
    **{"$schema": "http://json-schema.org/draft-07/schema#"})


def _entry(fs: FrameStats) -> dict:
    return {"frame": fs.frame, "durations_s": {s: fs.durations[s] for s in STAGES},
            "total_s": fs.total_time, "resident_pages": fs.resident,
            "required_pages": fs.required, "missing_pages": fs.missing,
            "bytes_copied": fs.bytes_copied}


def build_summary(stats, clock: str = DEVICE_CLOCK, resolution_s: float = 5e-7) -> dict:
    """Aggregate (harness.py:299-332): exemplar frames - most resident
    pages, smallest stage sum, largest transfer (ties: earliest frame) - and
    a synthetic median frame of per-stage medians."""
    frames = list(stats)
    if not frames:
        raise DataError("summary needs at least one frame")
    med = {s: float(statistics.median(f.durations[s] for f in frames)) for s in STAGES}

    def pick(key, largest):
        best = frames[0]
        for f in frames[1:]:
            if (key(f) > key(best)) if largest else (key(f) < key(best)):
                best = f
        return best

    return {
        "frame_count": len(frames),
        "timer": {"clock": clock, "resolution_s": float(resolution_s)},
        "stage_medians_s": med,
        "frames": {
            "most_pages": _entry(pick(lambda f: f.resident, True)),
            "median": {"note": MEDIAN_FRAME_NOTE, "durations_s": med,
                       "total_s": float(sum(med.values()))},
            "shortest": _entry(pick(lambda f: f.total_time, False)),
            "largest_transfer": _entry(pick(lambda f: f.bytes_copied, True)),
        },
    }


def stats_table(stats):
    """stats.csv rows (harness.py:335-348): counters only, so identical runs
    give identical bytes; floats as repr, thresholds ';'-joined."""
    frames = list(stats)
    width = len(frames[0].resident_per_level)
    yield (["frame", "required", "missing", "bytes_copied", "usage"]
           + ["resident_l%d" % k for k in range(width)] + ["thresholds"])
    for f in frames:
        if len(f.resident_per_level) != width:
            raise InvariantViolation("per-level resident width changed mid-run")
        yield ([str(f.frame), str(f.required), str(f.missing), str(f.bytes_copied),
                repr(float(f.usage))] + [str(c) for c in f.resident_per_level]
               + [";".join(repr(float(x)) for x in f.thresholds)])


def timings_table(stats):
    """timings.csv rows (harness.py:351-354)."""
    yield ["frame"] + ["%s_s" % s for s in STAGES]
    for f in stats:
        yield [str(f.frame)] + [repr(float(f.durations[s])) for s in STAGES]


def _write_rows(target: Path, rows) -> None:
    with open(target, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        for r in rows:
            w.writerow(r)


def emit_reports(stats, out_dir, clock: str = DEVICE_CLOCK) -> dict:
    """stats.csv, timings.csv and a schema-checked summary.json under
    ``out_dir`` (harness.py:365-387); returns the summary."""
    import jsonschema

    frames = list(stats)
    if not frames:
        raise DataError("no frames to report")
    root = Path(out_dir)
    root.mkdir(parents=True, exist_ok=True)
    _write_rows(root / "stats.csv", stats_table(frames))
    _write_rows(root / "timings.csv", timings_table(frames))
    summary = build_summary(frames, clock=clock)
    try:
        jsonschema.validate(summary, SUMMARY_SCHEMA)
    except jsonschema.ValidationError as exc:
        raise InvariantViolation(f"summary failed its schema: {exc.message}") from exc
    (root / "summary.json").write_text(json.dumps(summary, indent=2, sort_keys=True) + "\n")
    return summary


# -- multi-rank runs ------------------------------------------------------------------
_ROW_INTS = ("frame", "required", "missing", "bytes_copied")


def pack_rows(stats, levels: int, n_thresholds: int) -> np.ndarray:
    """FrameStats -> float64 rows for a collective gather (ints are exact in
    f64 below 2^53; usage / thresholds / durations are f64 already)."""
    rows = []
    for f in stats:
        if len(f.resident_per_level) != levels or len(f.thresholds) != n_thresholds:
            raise InvariantViolation("FrameStats width mismatch")
        rows.append([float(getattr(f, k)) for k in _ROW_INTS] + [float(f.usage)]
                    + [float(c) for c in f.resident_per_level] + [float(x) for x in f.thresholds]
                    + [float(f.durations[s]) for s in STAGES])
    return np.asarray(rows, dtype=np.float64).reshape(len(rows), 5 + levels + n_thresholds + len(STAGES))


def unpack_rows(rows: np.ndarray, levels: int, n_thresholds: int):
    out = []
    for r in rows:
        a = 5 + levels
        b = a + n_thresholds
        out.append(FrameStats(frame=int(r[0]), required=int(r[1]), missing=int(r[2]),
                              bytes_copied=int(r[3]), usage=float(r[4]),
                              resident_per_level=tuple(int(x) for x in r[5:a]),
                              thresholds=tuple(float(x) for x in r[a:b]),
                              durations={s: float(r[b + k]) for k, s in enumerate(STAGES)}))
    return out


def gather_stats(stats, dist, levels: int, n_thresholds: int, device=None):
    """Gather every rank's FrameStats to rank 0 (a list, in rank order);
    None on the other ranks.  One collective over NCCL (CUDA tensors) or
    gloo; blocks may differ in length by one frame."""
    import torch

    local = torch.from_numpy(pack_rows(stats, levels, n_thresholds))
    if device is not None:
        local = local.to(device)
    world, rank = dist.get_world_size(), dist.get_rank()
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    longest = int(max(int(s.item()) for s in sizes))
    padded = torch.zeros((longest, local.shape[1]), dtype=torch.float64, device=local.device)
    padded[: local.shape[0]] = local
    bufs = [torch.empty_like(padded) for _ in range(world)] if rank == 0 else None
    dist.gather(padded, bufs, dst=0)
    if rank != 0:
        return None
    rows = np.concatenate([b[: int(s.item())].cpu().numpy() for b, s in zip(bufs, sizes)], axis=0)
    return unpack_rows(rows, levels, n_thresholds)


def run_sharded(scene, path, config: BenchConfig | None = None, dist=None, frame_sink=None,
                device=None):
    """View sharding: rank r renders the contiguous
    block [r F / G, (r + 1) F / G) of the path with its own session (page
    table, device pool; the host-resident scene is shared: every rank maps the
    same file and page-locks that mapping in place, runtime.HostScene) - no
    data-path collective - and
    the FrameStats are gathered to rank 0, which gets the whole list
    (others get None).  Without ``dist`` this is ``run_benchmark``."""
    from paper_2506_19415_b200.sharding import frame_block

    cfg = config or BenchConfig()
    if dist is None or dist.get_world_size() == 1:
        return run_benchmark(scene, path, cfg, frame_sink=frame_sink)
    start, stop = frame_block(dist.get_rank(), dist.get_world_size(), frames_to_run(path, cfg))
    mine = run_benchmark(scene, path, cfg, frame_sink=frame_sink, frames=range(start, stop))
    levels = scene.lod_levels
    n_thr = (levels - 1) if (cfg.lod and levels > 1) else 0
    return gather_stats(mine, dist, levels, n_thr, device=device)
