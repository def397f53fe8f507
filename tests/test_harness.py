"""Harness / report layer (reference
pkg/src/vmsplat/harness.py): report formats on CPU, the multi-rank stats
gather over gloo, and - on the GPU - run_benchmark against the reference's
golden stats.csv for BASELINE config 1."""

import json
import os
import socket

import numpy as np
import pytest

from paper_2506_19415_b200 import harness
from paper_2506_19415_b200.errors import InvariantViolation


def _fs(i, res=(3, 1, 0), thr=(1.5, 3.0), dur=None):
    d = dur or {s: 0.001 * (i + k + 1) for k, s in enumerate(harness.STAGES)}
    return harness.FrameStats(frame=i, required=5 + i, missing=i % 2, bytes_copied=1000 * i,
                              usage=0.1 * i, resident_per_level=res, thresholds=thr,
                              durations=d)


def test_framestats_invariants():
    with pytest.raises(InvariantViolation):
        harness.FrameStats(0, 1, 2, 0, 0.0, (1,), (), {s: 0.0 for s in harness.STAGES})
    with pytest.raises(InvariantViolation):
        harness.FrameStats(0, 1, 0, 0, 0.0, (1,), (), {"visibility": 0.0})
    with pytest.raises(InvariantViolation):
        harness.FrameStats(0, 1, 0, 0, 0.0, (1,), (), {**{s: 0.0 for s in harness.STAGES},
                                                       "copy": -1.0})
    f = _fs(2)
    assert f.resident == 4 and harness.level0_equivalents(f) == 3.5


def test_stats_csv_matches_oracle_format(tmp_path):
    """stats.csv bytes equal the oracle's restatement of harness._stats_rows
    (which is pinned to the reference's own stats.csv in the golden tests)."""
    from oracle import core

    frames = [_fs(i) for i in range(4)]
    harness.emit_reports(frames, tmp_path)
    dicts = [{"frame": f.frame, "required_pages": f.required, "missing_pages": f.missing,
              "bytes_copied": f.bytes_copied, "usage": f.usage,
              "resident_per_level": f.resident_per_level, "thresholds": f.thresholds}
             for f in frames]
    assert (tmp_path / "stats.csv").read_bytes() == core.stats_csv(dicts).encode()
    lines = (tmp_path / "timings.csv").read_text().splitlines()
    assert lines[0] == "frame," + ",".join(f"{s}_s" for s in harness.STAGES)
    assert len(lines) == 5


def test_summary_exemplars_and_schema(tmp_path):
    import jsonschema

    frames = [_fs(0, res=(1, 0, 0)), _fs(1, res=(5, 0, 0)), _fs(2, res=(5, 0, 0)),
              _fs(3, dur={s: 0.0 for s in harness.STAGES})]
    summary = harness.emit_reports(frames, tmp_path)
    jsonschema.validate(json.loads((tmp_path / "summary.json").read_text()),
                        harness.SUMMARY_SCHEMA)
    fr = summary["frames"]
    assert fr["most_pages"]["frame"] == 1          # ties go to the earliest frame
    assert fr["shortest"]["frame"] == 3
    assert fr["largest_transfer"]["frame"] == 3
    assert fr["median"]["note"] == harness.MEDIAN_FRAME_NOTE
    assert summary["frame_count"] == 4


def test_write_frame_formats(tmp_path):
    img = np.linspace(0, 1.2, 4 * 5 * 3, dtype=np.float32).reshape(4, 5, 3)
    harness.write_frame(tmp_path / "a.png", img, 8)
    harness.write_frame(tmp_path / "a.ppm", img, 16)
    raw = (tmp_path / "a.ppm").read_bytes()
    assert raw.startswith(b"P6\n5 4\n65535\n")
    body = np.frombuffer(raw[len(b"P6\n5 4\n65535\n"):], dtype=">u2").reshape(4, 5, 3)
    assert np.array_equal(body, np.round(np.clip(img.astype(np.float64), 0, 1) * 65535))
    from PIL import Image

    png = np.asarray(Image.open(tmp_path / "a.png"))
    assert np.array_equal(png, np.round(np.clip(img.astype(np.float64), 0, 1) * 255).astype(np.uint8))
    assert harness.frame_name(7) == "frame_00007.png"
    assert harness.frame_name(7, 16) == "frame_00007.ppm"


def test_pack_unpack_roundtrip():
    frames = [_fs(i) for i in range(3)]
    rows = harness.pack_rows(frames, 3, 2)
    assert harness.unpack_rows(rows, 3, 2) == frames


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_19415_b200.sharding import frame_block

    start, stop = frame_block(rank, world, 7)
    mine = [_fs(i) for i in range(start, stop)]
    got = harness.gather_stats(mine, dist, 3, 2)
    if rank == 0:
        q.put([f.frame for f in got] == list(range(7)) and got == [_fs(i) for i in range(7)])
    dist.destroy_process_group()


def test_gather_stats_gloo_two_ranks():
    """The multi-rank report path: blocks of unequal length gathered in
    rank order over a real torch.distributed process group (gloo)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=5) is True


@pytest.mark.gpu
def test_run_benchmark_c1_matches_reference_stats(cuda, tmp_path):
    """BASELINE config 1 through the harness: stats.csv byte-identical to the
    reference run's golden stats.csv; timings from device events; frames
    handed to the sink; the no-paging ablation runs too."""
    from tests.golden import inputs

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c1.npz"))
    sc, _ = inputs.c1_scene()
    path = inputs.c1_path()
    seen = []
    stats = harness.run_benchmark(sc, path, harness.BenchConfig(),
                                  frame_sink=lambda i, im: seen.append((i, im.shape)))
    summary = harness.emit_reports(stats, tmp_path)
    assert (tmp_path / "stats.csv").read_bytes() == g["stats"].tobytes()
    assert [i for i, _ in seen] == list(range(path.frame_count))
    assert summary["timer"]["clock"] == harness.DEVICE_CLOCK
    assert all(f.durations["render"] > 0 for f in stats)
    flat = harness.run_benchmark(sc, path, harness.BenchConfig(vm=False, frame_limit=2))
    assert [f.required for f in flat] == [sc.page_count] * 2


@pytest.mark.gpu
@pytest.mark.parametrize("slots", ["2", "4", "8"])
def test_pipelined_harness_frames_identical(cuda, monkeypatch, slots):
    """run_benchmark(pipelined=True) (the session's frame slots kept full,
    host images written asynchronously) delivers the same frames, in order,
    and the same counters as the synchronous run - with 2, 4 (the default)
    and 8 frames in flight (VMSPLAT_SLOTS)."""
    from paper_2506_19415_b200 import scenegen

    monkeypatch.setenv("VMSPLAT_SLOTS", slots)

    lay = scenegen.CityLayout(n_pages=40, page_size=256, levels=3, seed=5, scale=0.12)
    sc = scenegen.city_scene(lay)
    path = scenegen.street_path(lay, frames=16, width=160, height=96)
    cfg = harness.BenchConfig(buffer_pages=16, staging_pages=6.0, vis_scale=0.5)
    a, b = [], []
    sa = harness.run_benchmark(sc, path, cfg, frame_sink=lambda i, im: a.append((i, im.copy())))
    sb = harness.run_benchmark(sc, path, cfg, frame_sink=lambda i, im: b.append((i, im)),
                               pipelined=True)
    assert [i for i, _ in b] == list(range(path.frame_count))
    for (ia, x), (ib, y) in zip(a, b):
        assert ia == ib and np.array_equal(x, y), ia
    assert [(f.required, f.missing, f.bytes_copied, f.resident_per_level) for f in sa] == \
           [(f.required, f.missing, f.bytes_copied, f.resident_per_level) for f in sb]


@pytest.mark.parametrize("slots", [2, 3, 4])
def test_pipelined_delivery_order_without_gpu(slots):
    """harness.run_benchmark(pipelined=True) against a stand-in session that
    models the real one's recycling with `slots` frames in flight: frame
    i - slots is complete once frame i has been submitted.  Every frame
    reaches the sink exactly once, in order, and only when complete."""

    class Paged:
        page_count = 1

    class Path:
        def frame_camera(self, i):
            return i

    class Session:
        def __init__(self):
            self.submitted = []
            self.done = set()
            self.slots = slots

        def render_frame(self, cam, i, wait=True):
            assert not wait
            self.submitted.append(i)
            if len(self.submitted) > slots:
                self.done.add(self.submitted[-slots - 1])  # recycled inside the call
            st = {"required_pages": 1, "missing_pages": 0, "bytes_copied": 0, "usage": 0.5,
                  "resident_per_level": (1,), "thresholds": (1.0,)}
            st.update({f"time_{s}": 0.1 for s in harness.STAGES})
            return np.full((2, 2, 3), float(i), np.float32), st

        def wait(self, back):
            assert 0 <= back < slots
            self.done.update(self.submitted[len(self.submitted) - 1 - back:])

    for n in (1, 2, 3, 7, 12):
        sess, got = Session(), []

        def sink(i, im, sess=sess, got=got):
            assert i in sess.done, f"frame {i} handed over before it was complete"
            assert float(im[0, 0, 0]) == float(i)
            got.append(i)

        stats = harness.run_benchmark(Paged(), Path(), frames=range(n), session=sess,
                                      frame_sink=sink, pipelined=True)
        assert got == list(range(n)) and [s.frame for s in stats] == list(range(n))
