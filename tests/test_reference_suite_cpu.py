"""The reference suite's host-side tests of the modules this package mirrors,
run on CPU through the reference's import names (tests/refsuite.py):
camera paths (pkg/tests/test_camera_path.py) and the `.vms` scene file
(pkg/tests/test_scene_io.py, the parts on the per-frame path: the binary
format, memory-mapped reads, page arithmetic, validation).  Scenes come from
the reference's own pipeline (tests/golden/ref_scenes), so the byte-for-byte
write test also pins the format against the reference's writer.
"""

import json
import math

import numpy as np
import pytest

from tests import refsuite

refsuite.install()

from vmsplat.camera_path import CameraPath, Checkpoint, load_path, save_path, slerp  # noqa: E402
from vmsplat.errors import ParseError, SceneFormatError  # noqa: E402
from vmsplat.gaussians import RECORD_SIZE  # noqa: E402
from vmsplat.scene_io import read_scene, write_scene  # noqa: E402

IDENT = (1.0, 0.0, 0.0, 0.0)


def _path(points, speed=1.0, **kw):
    return CameraPath(checkpoints=tuple(Checkpoint(position=tuple(p), orientation=IDENT)
                                        for p in points), speed=speed, **kw)


# -- camera paths (pkg/tests/test_camera_path.py:20-121) -----------------------------

def test_path_arc_length_timing():
    p = _path([(0, 0, 0), (3, 0, 4)])  # one segment of length 5
    assert np.array_equal(p.pose_at(0.0)[0], [0, 0, 0])
    assert np.array_equal(p.pose_at(p.duration)[0], [3, 0, 4])
    p = _path([(0, 0, 0), (2, 0, 0), (2, 4, 0)])  # lengths 2 and 4, unit speed
    assert p.total_length == pytest.approx(6.0) and p.duration == pytest.approx(6.0)
    assert np.allclose(p.pose_at(1.0)[0], [1, 0, 0])
    assert np.allclose(p.pose_at(4.0)[0], [2, 2, 0])
    p = _path([(0, 0, 0), (10, 0, 0)], speed=4.0, fps=30.0)
    assert p.duration == pytest.approx(2.5) and p.frame_count == 76
    assert np.allclose(p.pose_at(1.0)[0], [4, 0, 0])
    p = _path([(0, 0, 0), (0, 0, 0), (4, 0, 0)])  # the zero-length segment is skipped
    assert p.lengths == (0.0, 4.0)
    assert np.allclose(p.pose_at(2.0)[0], [2, 0, 0])
    assert np.allclose(p.pose_at(0.0)[0], [0, 0, 0])
    p = _path([(0, 0, 0), (1, 0, 0)])  # clamped at both ends
    assert np.array_equal(p.pose_at(99.0)[0], [1, 0, 0])
    assert np.array_equal(p.pose_at(-1.0)[0], [0, 0, 0])


def test_path_orientation_and_short_arc():
    q1 = (math.cos(math.pi / 4), 0.0, 0.0, math.sin(math.pi / 4))  # 90 degrees about z
    p = CameraPath(checkpoints=(Checkpoint(position=(0, 0, 0), orientation=IDENT),
                                Checkpoint(position=(2, 0, 0), orientation=q1)))
    _, quat = p.pose_at(1.0)
    assert np.allclose(quat, [math.cos(math.pi / 8), 0, 0, math.sin(math.pi / 8)], atol=1e-12)
    q = np.array([math.cos(0.4), 0, 0, math.sin(0.4)])
    mid = slerp(np.array([1.0, 0, 0, 0]), -q, 0.5)  # -q: the same rotation, short arc
    assert abs(abs(mid @ np.array([math.cos(0.2), 0, 0, math.sin(0.2)])) - 1.0) < 1e-12


def test_frame_camera_uses_fps_and_lens():
    p = _path([(0, 0, 0), (6, 0, 0)], speed=2.0, fps=10.0, fov_deg=60.0, width=128, height=96)
    cam = p.frame_camera(5)  # t = 0.5 s -> arc length 1
    assert np.allclose(cam.position, [1, 0, 0])
    assert cam.fov_y == pytest.approx(math.radians(60.0))
    assert (cam.width, cam.height) == (128, 96)


def test_path_json_round_trip_and_errors(tmp_path):
    p = _path([(0, 0, 0), (1, 2, 3), (4, 4, 4)], speed=2.5, fps=24.0, fov_deg=70.0)
    f = tmp_path / "path.json"
    save_path(p, f)
    q = load_path(f)
    assert q == p
    for t in (0.0, 0.7, 1.9):
        (pa, qa), (pb, qb) = p.pose_at(t), q.pose_at(t)
        assert np.array_equal(pa, pb) and np.array_equal(qa, qb)
    f.write_text("{not json")
    with pytest.raises(ParseError):
        load_path(f)
    f.write_text(json.dumps({"checkpoints": [{"position": [0, 0, 0]}]}))
    with pytest.raises(ParseError):
        load_path(f)


def test_path_validation():
    for kw, pts in (({}, [(0, 0, 0)]), ({"speed": 0.0}, [(0, 0, 0), (1, 0, 0)]),
                    ({"fps": -1.0}, [(0, 0, 0), (1, 0, 0)])):
        with pytest.raises(ValueError):
            _path(pts, **kw)


# -- the .vms scene file (pkg/tests/test_scene_io.py:69-173) ------------------------

@pytest.fixture(scope="module")
def ref_vms():
    """(path, bytes) of a paged, LOD'd scene the reference pipeline wrote."""
    path = refsuite.scene_path("small")
    with open(path, "rb") as fh:
        return path, fh.read()


def test_write_reproduces_the_reference_file(ref_vms, tmp_path):
    path, blob = ref_vms
    out = tmp_path / "again.vms"
    write_scene(read_scene(path), out)
    assert out.read_bytes() == blob  # byte-compatible with the reference writer
    out2 = tmp_path / "again2.vms"
    write_scene(read_scene(out), out2)
    assert out2.read_bytes() == blob  # and deterministic


def test_mmap_read_matches_eager(ref_vms):
    path, _ = ref_vms
    eager = read_scene(path)
    lazy = read_scene(path, mmap_gaussians=True)
    assert isinstance(lazy.gaussians, np.memmap)
    assert np.array_equal(np.asarray(lazy.gaussians), eager.gaussians)
    for name in ("vertices", "faces", "face_page", "link_offsets", "link_targets"):
        assert np.array_equal(getattr(lazy, name), getattr(eager, name)), name
    assert (lazy.stage, lazy.page_size, lazy.lod_levels, lazy.page_counts) == \
        (eager.stage, eager.page_size, eager.lod_levels, eager.page_counts)


def test_page_record_arithmetic(ref_vms):
    scene = read_scene(ref_vms[0])
    size, pages = scene.page_size, scene.page_count
    assert scene.level_record_count(0) == size
    assert scene.level_record_count(1) == size // 2
    assert scene.page_record_range(0, 1) == (0, size)
    assert scene.page_record_range(0, pages)[1] == pages * size
    assert scene.page_record_range(1, 1)[0] == pages * size  # level blocks in order
    total = sum(pages * scene.level_record_count(k) for k in range(scene.lod_levels))
    assert scene.total_records() == total == len(scene.gaussians)


def test_corrupt_files_rejected(ref_vms, tmp_path):
    _, blob = ref_vms
    bad = tmp_path / "bad.vms"
    bad.write_bytes(b"JUNK" + blob[4:])
    with pytest.raises(SceneFormatError):
        read_scene(bad)
    bad.write_bytes(blob[: len(blob) - 64])
    with pytest.raises(SceneFormatError):
        read_scene(bad)


def test_validate_rejects_inconsistent_scenes(ref_vms):
    scene = read_scene(ref_vms[0])
    scene.faces = scene.faces.copy()
    scene.faces[0, 2] = len(scene.vertices) + 5
    with pytest.raises(SceneFormatError):
        scene.validate()
    scene = read_scene(ref_vms[0])
    scene.gaussians = np.zeros((4, RECORD_SIZE - 1), dtype=np.float32)
    with pytest.raises(SceneFormatError):
        scene.validate()
    scene = read_scene(ref_vms[0])
    scene.stage = "bogus"
    with pytest.raises(SceneFormatError):
        scene.validate()
