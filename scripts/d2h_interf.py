"""Does a concurrent 25 MB device->host copy per frame slow the render?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
x = torch.empty((1080, 1920, 3), device="cuda")
hs = [torch.empty((1080, 1920, 3)).pin_memory() for _ in range(2)]
side = torch.cuda.Stream()
for mode in ("none", "d2h", "d2h_l2"):
    s = VmSession(scene, buffer_pages=500, staging_pages=40, vis_scale=0.25, timing=False)
    for f in range(5):
        s.render_frame(traj.frame_camera(f), f, out="device")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for f in range(5, 65):
        img, _ = s.render_frame(traj.frame_camera(f), f, out="device")
        if mode != "none":
            ev = torch.cuda.Event()
            ev.record()
            side.wait_event(ev)
            with torch.cuda.stream(side):
                hs[f % 2].copy_(img if mode == "d2h" else x, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(mode, "fps", 60 / (e0.elapsed_time(e1) * 1e-3))
    del s
