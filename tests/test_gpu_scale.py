"""GPU parity at the benchmark scales the oracle cannot run end to end
(SURVEY 8(c)): C3 (20.5M records, 10K pages, 4 LOD levels) at 1080p and at
4K (the C5 resolution), the box-limited out-of-core C4 (609.3M records in
3 LOD levels, 144 GB in host DRAM), plus the blend's exp kernel against libm, caller-owned
device output, and view sharding with real sessions.

Tolerances as in test_gpu_parity: page sets / plans / residency / stats
bit-exact, images max-abs <= 1e-5 (exact blend).
"""

import os

import numpy as np
import pytest

from oracle import core

pytestmark = pytest.mark.gpu

EXACT_TOL = 1e-5
STAT_KEYS = ("required_pages", "resident_pages", "resident_per_level", "planned_copies",
             "missing_pages", "bytes_copied", "usage", "lod_step", "thresholds")


def _maxabs(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


def _check_stats(st, rst, f):
    for k in STAT_KEYS:
        assert st[k] == rst[k], (f, k, st[k], rst[k])


# -- C3 -------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c3_scene(tmp_path_factory):
    from paper_2506_19415_b200 import scenegen
    from paper_2506_19415_b200.scene_io import read_scene

    p = tmp_path_factory.mktemp("c3") / "c3.vms"
    scenegen.write_city(p, scenegen.C3)
    yield read_scene(p, mmap_gaussians=True)
    os.unlink(p)


C3_BUFFER = 4096   # bench.py CONFIGS["c3"]: ~1.9 GB page pool, 8.4M records


def _run_pair(scene, traj, image_frames, last, **kw):
    from paper_2506_19415_b200.runtime import VmSession

    s = VmSession(scene, **kw)
    o = core.OSession(scene, **kw)
    worst, req = 0.0, []
    for f in range(last + 1):
        cam = traj.frame_camera(f)
        want = f in image_frames
        img, st = s.render_frame(cam, f, out=None if want else "device")
        ref, rst = o.render_frame(cam, f, want_image=want)
        _check_stats(st, rst, f)
        req.append(st["required_pages"])
        if want:
            assert sorted(s.table.resident.items()) == sorted(o.table.resident.items()), f
            assert float(ref.max()) > 0.0
            err = _maxabs(img, ref)
            assert err <= EXACT_TOL, (f, err)
            worst = max(worst, err)
    return worst, req, s


def test_c3_frames_match_oracle(cuda, c3_scene):
    """C3 at 1080p with the bench's 4096-page buffer: the whole 120-frame
    path with page sets, plans, residency and stats bit-exact on every frame
    and full images at frames 12, 30, 48, 80 and 119 (up to 8.4M resident
    records per frame on both sides)."""
    from paper_2506_19415_b200 import scenegen

    traj = scenegen.street_path(scenegen.C3, frames=120)
    worst, req, s = _run_pair(c3_scene, traj, {12, 30, 48, 80, 119}, 119,
                              buffer_pages=C3_BUFFER, staging_pages=40, vis_scale=0.25)
    assert s.dot_mode_exact
    assert max(req) > 100
    print(f"C3 1080p: worst max-abs {worst:.2e}, required pages {min(req)}-{max(req)}")


def test_c3_4k_frames_match_oracle(cuda, c3_scene):
    """C5's resolution on the C3 scene: 3840x2160 (vis 960x540), frames 0-60
    with stats bit-exact on every frame and full 4K images at frames 8, 24
    and 60."""
    from paper_2506_19415_b200 import scenegen

    traj = scenegen.street_path(scenegen.C3, frames=120, width=3840, height=2160)
    worst, req, _ = _run_pair(c3_scene, traj, {8, 24, 60}, 60, buffer_pages=C3_BUFFER,
                              staging_pages=40, vis_scale=0.25)
    print(f"C3 4K: worst max-abs {worst:.2e}, required pages {min(req)}-{max(req)}")


# -- C4 (out-of-core, host DRAM) ----------------------------------------------------
C4_BUFFER = 2048
C4_STAGING = 160
C4_BLOCKS = 24


@pytest.fixture(scope="module")
def c4_scene():
    """The box-limited C4 city in tmpfs (host DRAM), removed afterwards."""
    from paper_2506_19415_b200 import scenegen
    from paper_2506_19415_b200.scene_io import read_scene

    lay = scenegen.C4
    need = sum(lay.n_pages * (lay.page_size >> k) for k in range(lay.levels)) * 236
    st = os.statvfs("/dev/shm")
    if st.f_bavail * st.f_frsize < need * 1.05:
        pytest.skip(f"C4 needs {need >> 30} GB of tmpfs (host DRAM); /dev/shm has "
                    f"{(st.f_bavail * st.f_frsize) >> 30} GB")
    d = "/dev/shm/vmsplat_test_c4"
    os.makedirs(d, exist_ok=True)
    p = os.path.join(d, "c4.vms")
    scenegen.write_city(p, lay)
    try:
        yield read_scene(p, mmap_gaussians=True)
    finally:
        os.unlink(p)
        os.rmdir(d)


def test_c4_page_sets_and_window_match_oracle(cuda, c4_scene):
    """SURVEY 8(c)(i)+(ii) on the out-of-core scene (170K pages, 340K faces:
    the multi-kernel visibility back end past 32K pages): frames 0-40 of the
    long street path with visibility, required lists, plans, residency and
    stats bit-exact on every frame against the oracle's visibility + reduce +
    update_page_table; then the rendered frame 40 against the oracle's
    windowed render (render_window: every window pixel exact by
    construction) on three 96x96 windows, one at the vanishing point."""
    from paper_2506_19415_b200 import scenegen
    from paper_2506_19415_b200.runtime import VmSession

    traj = scenegen.street_path(scenegen.C4, frames=120, blocks=C4_BLOCKS)
    kw = dict(buffer_pages=C4_BUFFER, staging_pages=C4_STAGING, vis_scale=0.25)
    s = VmSession(c4_scene, **kw)
    o = core.OSession(c4_scene, **kw)
    last = 40
    copied = 0
    for f in range(last + 1):
        cam = traj.frame_camera(f)
        img, st = s.render_frame(cam, f, out=None if f == last else "device")
        _, rst = o.render_frame(cam, f, want_image=False)
        _check_stats(st, rst, f)
        copied += st["bytes_copied"]
    assert sorted(s.table.resident.items()) == sorted(o.table.resident.items())
    assert copied > 512 << 20
    records = o.resident_records()
    cam = traj.frame_camera(last)
    W, H = cam.width, cam.height
    for x0, y0 in ((W // 2 - 48, H // 2 - 48), (100, 200), (W - 400, H - 300)):
        win, n = core.render_window(records, core.as_ocam(cam), (x0, x0 + 96, y0, y0 + 96))
        assert n > 0
        err = _maxabs(img[y0:y0 + 96, x0:x0 + 96], win)
        assert err <= EXACT_TOL, ((x0, y0), err)


# -- exp kernel, device output, sharding ---------------------------------------------
def test_blend_exp_within_one_ulp_of_libm(cuda):
    """The exact blend's table-driven FP64 exp against libm (NumPy) over
    2e7 points of [-700, 0] plus the edges: at most 1 ulp apart."""
    import torch

    from paper_2506_19415_b200 import _device, _lib

    rng = np.random.default_rng(11)
    x = np.concatenate([-rng.exponential(3.0, 10_000_000), rng.uniform(-700.0, 0.0, 10_000_000),
                        [0.0, -0.0, -1e-300, -5e-324, -np.log(2) / 128, -700.0,
                         -np.log(2) * 64, -np.log(2) / 64]])
    x = x[x >= -700.0]
    dx = torch.from_numpy(x).cuda()
    out = torch.empty_like(dx)
    _lib.check(_lib.load().vms_debug_exp(dx.data_ptr(), len(x), out.data_ptr(), _device.sptr()))
    got = out.cpu().numpy()
    ref = np.exp(x)
    ulp = np.abs(got.view(np.int64) - ref.view(np.int64))
    assert int(ulp.max()) <= 1, (int(ulp.max()), x[int(np.argmax(ulp))])
    print(f"exp: {len(x)} points, {int((ulp == 1).sum())} at 1 ulp, rest exact")


def test_render_into_caller_device_tensor(cuda):
    """render_frame(out=<CUDA tensor>) writes the caller's tensor (a frame
    stack slot) with the same image as host output."""
    import torch

    from paper_2506_19415_b200 import scenegen
    from paper_2506_19415_b200.runtime import VmSession
    from tests.golden import inputs

    sc = scenegen.city_scene(inputs.CITY_SMALL)
    path = inputs.city_path(inputs.CITY_SMALL)
    a = VmSession(sc, buffer_pages=16, staging_pages=6.0, vis_scale=0.5)
    b = VmSession(sc, buffer_pages=16, staging_pages=6.0, vis_scale=0.5)
    cam0 = path.frame_camera(0)
    stack = torch.zeros((path.frame_count, cam0.height, cam0.width, 3), device="cuda")
    refs = []
    for f in range(path.frame_count):
        cam = path.frame_camera(f)
        refs.append(a.render_frame(cam, f)[0])
        b.render_frame(cam, f, out=stack[f])
    torch.cuda.synchronize()
    for f, r in enumerate(refs):
        assert np.array_equal(stack[f].cpu().numpy(), r), f
    with pytest.raises(ValueError):
        b.render_frame(cam0, 99, out=torch.zeros((3, 3, 3), device="cuda"))


def test_sharded_sessions_match_per_shard_oracle(cuda, tmp_path):
    """SURVEY 8(e) with real sessions: two ranks (gloo, one process each, both
    on this GPU) run harness.run_sharded over their blocks of a paged city,
    both streaming from ONE host-resident copy of the scene (a tmpfs file
    each rank page-locks in place); the gathered stats.csv equals one oracle
    session per block."""
    import subprocess
    import sys

    from paper_2506_19415_b200 import scenegen

    lay = scenegen.CityLayout(n_pages=200, page_size=512, levels=3, seed=2, scale=0.1)
    d = f"/dev/shm/vmsplat_test_shard_{os.getpid()}"
    os.makedirs(d, exist_ok=True)
    p = os.path.join(d, "shard.vms")
    scenegen.write_city(p, lay)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root, MASTER_ADDR="127.0.0.1", MASTER_PORT="29531")
    script = os.path.join(root, "tests", "shard_worker.py")
    procs = [subprocess.Popen([sys.executable, script, str(p), str(tmp_path), str(r), "2"],
                              env=dict(env, RANK=str(r), WORLD_SIZE="2"),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(2)]
    try:
        outs = [pr.communicate(timeout=600)[0] for pr in procs]
    finally:
        os.unlink(p)
        os.rmdir(d)
    for pr, o in zip(procs, outs):
        assert pr.returncode == 0, o
    assert all("shard ok" in o for o in outs), outs


def test_binned_visibility_raster_is_bit_exact(cuda):
    """The binned, chunk-parallel visibility raster (per-tile triangle lists,
    long lists split over CTAs and merged in chunk order; on by default from
    65536 faces) forced on for the small meshes: the visibility goldens, the
    session goldens and C1 still match bit for bit (a subprocess, since the
    raster variant is fixed per process)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VMSPLAT_VIS_BIN="1", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_parity.py"), "-k",
                        "visibility or session_matches or c1_session or rasterize or nothing"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_hot_tile_blend_is_exact(cuda):
    """The hot-tile blend (blend_hot_k: one CTA per 8x4 block, producer warps
    computing the FP64 weights of a long list, one consumer warp applying
    them in list order; on by default for lists >= 32768 instances) forced
    on for every list >= 256: the composite goldens, the session goldens and
    C2's first 35 frames still match (a subprocess: the threshold is read
    once per process)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VMSPLAT_HOT_LEN="256", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_parity.py"), "-k",
                        "composite or session_matches or c1_session or output_modes or overflow "
                        "or c2_whole"],
                       env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_upload_modes_from_registered_tmpfs_scene(cuda):
    """A scene file on tmpfs is page-locked in place (HostScene), so its
    record section starts at the mapping plus the file header - not 16-byte
    aligned.  All three upload modes (copy engines, the gather kernel, the
    streaming bounce buffer) give the same frames and stats from it (the
    gather kernel once used 16-byte vectors on the misaligned base)."""
    import numpy as np
    from paper_2506_19415_b200 import scenegen
    from paper_2506_19415_b200.runtime import HostScene, VmSession
    from paper_2506_19415_b200.scene_io import read_scene

    lay = scenegen.CityLayout(n_pages=60, page_size=256, levels=3, seed=4, scale=0.1)
    d = f"/dev/shm/vmsplat_test_upload_{os.getpid()}"
    os.makedirs(d, exist_ok=True)
    p = os.path.join(d, "city.vms")
    try:
        scenegen.write_city(p, lay)
        sc = read_scene(p, mmap_gaussians=True)
        path = scenegen.street_path(lay, frames=12, width=160, height=96)
        hs = HostScene.of(sc)
        runs = {}
        for mode in (0, 1, 2):
            s = VmSession(sc, buffer_pages=24, staging_pages=6.0, vis_scale=0.5, upload_mode=mode,
                          timing=False)
            runs[mode] = [s.render_frame(path.frame_camera(f), f) for f in range(12)]
            s.close()
        copied = 0
        for f in range(12):
            (i0, s0), (i1, s1), (i2, s2) = runs[0][f], runs[1][f], runs[2][f]
            for k in ("required_pages", "resident_pages", "bytes_copied", "missing_pages"):
                assert s0[k] == s1[k] == s2[k], (f, k)
            copied += s0["bytes_copied"]
            assert np.array_equal(i0, i1) and np.array_equal(i0, i2), f
        assert copied > 0
        del hs
    finally:
        if os.path.exists(p):
            os.unlink(p)
        os.rmdir(d)
