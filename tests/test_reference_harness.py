"""The reference's benchmark-driver tests (pkg/tests/test_harness.py), run
against this package's harness through the reference's import names
(tests/refsuite.py).  The summary/stat helpers run on CPU; the runs of
``run_benchmark`` (a receding camera over the reference-built "small" scene,
the reference's `small_bundle`) need the GPU."""

import csv
import hashlib
import json
import statistics

import jsonschema
import pytest

from tests import refsuite

refsuite.install()

from vmsplat.camera_path import CameraPath, Checkpoint  # noqa: E402
from vmsplat.errors import DataError  # noqa: E402
from vmsplat.harness import (STAGES, SUMMARY_SCHEMA, BenchConfig, FrameStats,  # noqa: E402
                             build_summary, emit_reports, frame_name, level0_equivalents,
                             run_benchmark, write_frame)
from vmsplat.scene_io import SceneFile  # noqa: E402

gpu = pytest.mark.gpu
IDENT = (1.0, 0.0, 0.0, 0.0)


def _stats(frame=0, resident=(5,), bytes_copied=0, **durations):
    d = {s: 0.001 for s in STAGES}
    d.update(durations)
    return FrameStats(frame=frame, required=5, missing=0, bytes_copied=bytes_copied, usage=0.5,
                      resident_per_level=resident, thresholds=(), durations=d)


def _receding(z0=-2.0, z1=-10.0, fps=10.0, speed=2.0, size=96):
    """harness tests' camera: backing away from the scene along -z."""
    return CameraPath(checkpoints=(Checkpoint(position=(0.0, 0.0, z0), orientation=IDENT),
                                   Checkpoint(position=(0.0, 0.0, z1), orientation=IDENT)),
                      speed=speed, fps=fps, fov_deg=90.0, width=size, height=size)


# -- host-side (test_harness.py:82-187) -------------------------------------------

def test_level0_equivalents_halves_per_level():
    fs = _stats(resident=(4, 2, 1))
    assert level0_equivalents(fs) == pytest.approx(4 + 1 + 0.25)
    assert fs.resident == 7


def test_summary_median_exemplars_and_empty():
    s = build_summary([_stats(0, render=0.009), _stats(1, render=0.001), _stats(2, render=0.002)])
    assert s["stage_medians_s"]["render"] == 0.002
    assert s["frames"]["median"]["durations_s"]["render"] == 0.002
    s = build_summary([_stats(0, (3,), 100, render=0.005), _stats(1, (9,), 700, render=0.001),
                       _stats(2, (9,), 700, render=0.001)])
    f = s["frames"]
    assert f["most_pages"]["frame"] == 1 and f["shortest"]["frame"] == 1  # earliest wins ties
    assert f["largest_transfer"]["frame"] == 1
    assert f["median"]["note"] and "frame" not in f["median"]
    with pytest.raises(DataError):
        build_summary([])


def test_unpaged_scene_rejected():
    with pytest.raises(DataError):
        run_benchmark(SceneFile(stage="raw"), _receding())


# -- runs (test_harness.py:91-250) ------------------------------------------------

@pytest.fixture(scope="module")
def small():
    return refsuite.scene("small")


@gpu
def test_rows_frames_limit_and_sink(cuda, small):
    path = _receding(fps=5.0)  # 4 s -> 21 frames
    stats = run_benchmark(small, path, BenchConfig(buffer_pages=30))
    assert len(stats) == path.frame_count == 21
    assert [fs.frame for fs in stats] == list(range(21))
    assert len(run_benchmark(small, _receding(), BenchConfig(buffer_pages=30, frame_limit=4))) == 4
    seen = []
    run_benchmark(small, _receding(), BenchConfig(buffer_pages=30, frame_limit=3),
                  frame_sink=lambda i, img: seen.append((i, img.shape)))
    assert seen == [(0, (96, 96, 3)), (1, (96, 96, 3)), (2, (96, 96, 3))]


@gpu
def test_vm_off_keeps_everything_resident(cuda, small):
    for fs in run_benchmark(small, _receding(), BenchConfig(vm=False, frame_limit=3)):
        assert fs.resident_per_level[0] == small.page_count
        assert sum(fs.resident_per_level[1:]) == 0
        assert fs.missing == 0 and fs.usage == 1.0 and fs.thresholds == ()


@gpu
def test_links_add_pages_and_lod_saves_footprint(cuda, small):
    path = _receding(fps=5.0, z1=-6.0)
    on = run_benchmark(small, path, BenchConfig(buffer_pages=30, lod=False, links=True))
    off = run_benchmark(small, path, BenchConfig(buffer_pages=30, lod=False, links=False))
    assert all(a.required >= b.required for a, b in zip(on, off))
    assert sum(a.required for a in on) > sum(b.required for b in off)
    path = _receding(z0=-3.0, z1=-20.0, fps=5.0)
    lod = run_benchmark(small, path, BenchConfig(buffer_pages=12, lod=True))
    flat = run_benchmark(small, path, BenchConfig(buffer_pages=12, lod=False))
    for a, b in zip(lod, flat):
        assert level0_equivalents(a) <= level0_equivalents(b) + 1e-9


@gpu
def test_reports_schema_single_frame_and_median(cuda, small, tmp_path):
    stats = run_benchmark(small, _receding(), BenchConfig(buffer_pages=30, frame_limit=5))
    summary = emit_reports(stats, tmp_path)
    for name in ("stats.csv", "timings.csv", "summary.json"):
        assert (tmp_path / name).is_file()
    jsonschema.validate(summary, SUMMARY_SCHEMA)
    assert json.loads((tmp_path / "summary.json").read_text()) == summary
    with open(tmp_path / "stats.csv", newline="") as fh:
        rows = list(csv.reader(fh))
    assert len(rows) == 6
    assert rows[0] == (["frame", "required", "missing", "bytes_copied", "usage"]
                       + [f"resident_l{k}" for k in range(small.lod_levels)] + ["thresholds"])
    one = tmp_path / "one"
    one.mkdir()
    s1 = emit_reports(run_benchmark(small, _receding(), BenchConfig(buffer_pages=30,
                                                                    frame_limit=1)), one)
    assert s1["frame_count"] == 1
    seven = tmp_path / "seven"
    seven.mkdir()
    s7 = emit_reports(run_benchmark(small, _receding(), BenchConfig(buffer_pages=30,
                                                                    frame_limit=7)), seven)
    with open(seven / "timings.csv", newline="") as fh:
        rows = list(csv.DictReader(fh))
    for stage in STAGES:
        assert s7["frames"]["median"]["durations_s"][stage] == \
            statistics.median(float(r[f"{stage}_s"]) for r in rows)


@gpu
def test_stats_and_frames_deterministic(cuda, small, tmp_path):
    def run(tag):
        out = tmp_path / tag
        out.mkdir()
        digests = {}

        def sink(i, img):
            write_frame(out / frame_name(i), img)
            digests[i] = hashlib.sha256((out / frame_name(i)).read_bytes()).hexdigest()

        emit_reports(run_benchmark(small, _receding(), BenchConfig(buffer_pages=20,
                                                                   frame_limit=6),
                                   frame_sink=sink), out)
        digests["stats.csv"] = hashlib.sha256((out / "stats.csv").read_bytes()).hexdigest()
        return digests

    assert run("a") == run("b")
