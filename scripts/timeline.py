"""Per-frame host/device timeline of the device-output loop (VMSPLAT_TRACE=2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["VMSPLAT_TRACE"] = "2"
import torch
import bench
from paper_2506_19415_b200 import scenegen
from paper_2506_19415_b200.runtime import VmSession
from paper_2506_19415_b200.scene_io import read_scene
class A:
    scene_dir = os.environ.get("VMSPLAT_SCENE_DIR", "/tmp/vmsplat_bench")
lay, path = bench.ensure_scene(A, 0)
scene = read_scene(path, mmap_gaussians=True)
traj = scenegen.street_path(lay, frames=120)
s = VmSession(scene, buffer_pages=500, staging_pages=40, vis_scale=0.25, timing=False)
for f in range(64):
    s.render_frame(traj.frame_camera(f), f, out="device")
torch.cuda.synchronize()
import time
cams = [traj.frame_camera(f) for f in range(64, 96)]
ts = []
for k, f in enumerate(range(64, 96)):
    t0 = time.perf_counter()
    c = traj.frame_camera(f)
    t1 = time.perf_counter()
    s.render_frame(cams[k], f, out="device")
    t2 = time.perf_counter()
    ts.append((t1 - t0, t2 - t1))
torch.cuda.synchronize()
for a, b in ts[-10:]:
    print("frame_camera %.1f us  render_frame %.1f us" % (a * 1e6, b * 1e6))
class Proxy:
    def __init__(self, lib):
        self._l = lib
        self.t = []
    def __getattr__(self, k):
        return getattr(self._l, k)
    def vms_session_frame(self, *a):
        t0 = time.perf_counter()
        r = self._l.vms_session_frame(*a)
        self.t.append((t0, time.perf_counter()))
        return r
p = Proxy(s._lib)
s._lib = p
ts = []
for k, f in enumerate(range(64, 96)):
    t1 = time.perf_counter()
    s.render_frame(cams[k], f, out="device")
    t2 = time.perf_counter()
    ts.append((t1, t2))
torch.cuda.synchronize()
for (t1, t2), (c0, c1) in list(zip(ts, p.t))[-8:]:
    print("py-pre %.1f us  C %.1f us  py-post %.1f us" % ((c0 - t1) * 1e6, (c1 - c0) * 1e6, (t2 - c1) * 1e6))
for (t1, t2), (c0, c1) in list(zip(ts, p.t))[-8:]:
    print("abs py call %.1f  C enter %.1f  C exit %.1f  py ret %.1f" % (t1 * 1e6, c0 * 1e6, c1 * 1e6, t2 * 1e6))
