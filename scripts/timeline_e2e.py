"""Per-frame timeline of the pipelined harness (host output), VMSPLAT_TRACE=2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["VMSPLAT_TRACE"] = "2"
import torch
import bench
from paper_2506_19415_b200 import scenegen, harness
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
s = VmSession(scene, buffer_pages=500, staging_pages=40, vis_scale=0.25, timing=False)
got = []
harness.run_benchmark(scene, traj, frames=range(0, 64), session=s, pipelined=True,
                      frame_sink=lambda i, im: got.append(float(im[0, 0, 0])))
torch.cuda.synchronize()
t0 = time.perf_counter()
harness.run_benchmark(scene, traj, frames=range(64, 96), session=s, pipelined=True,
                      frame_sink=lambda i, im: got.append(float(im[0, 0, 0])))
torch.cuda.synchronize()
print("e2e fps", 32 / (time.perf_counter() - t0))
x = torch.empty((1080, 1920, 3), device="cuda")
h = torch.empty((1080, 1920, 3)).pin_memory()
for _ in range(3):
    h.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    h.copy_(x, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print("d2h GB/s alone", 10 * x.numel() * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
