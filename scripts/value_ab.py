"""Device-timed A/B helper: C2 frames 5-64 left in HBM (out="device"),
CUDA events on the caller's stream, 5 repetitions in one process (fresh
session each), median frames/s.  Knobs from the environment (VMSPLAT_*)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2506_19415_b200.runtime import VmSession
from paper_2506_19415_b200.scene_io import read_scene


class A:
    config = "c2"
    scene_dir = None
    frames = 120
    width = 1920
    height = 1080


lay, path = bench.ensure_scene(A, 0)
scene = read_scene(path, mmap_gaussians=True)
traj = bench.trajectory(A, lay)
lo, hi = int(os.environ.get("AB_FROM", "5")), int(os.environ.get("AB_TO", "65"))
fps = []
for rep in range(int(os.environ.get("AB_REPS", "5"))):
    s = VmSession(scene, buffer_pages=500, staging_pages=40, vis_scale=0.25, timing=False,
                  upload_mode=int(os.environ["AB_UPLOAD"]) if os.environ.get("AB_UPLOAD") else None)
    for f in range(lo):
        s.render_frame(traj.frame_camera(f), f, out="device")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for f in range(lo, hi):
        s.render_frame(traj.frame_camera(f), f, out="device")
    e1.record()
    torch.cuda.synchronize()
    fps.append((hi - lo) / (e0.elapsed_time(e1) * 1e-3))
    s.close()
print(os.environ.get("AB_TAG", ""), "value median", round(statistics.median(fps), 1),
      "all", [round(x) for x in fps])
