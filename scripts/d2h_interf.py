"""Does a concurrent 25 MB copy per frame slow the render, and through what?

Modes (C2, frames 5-64, frame left in HBM, fps from CUDA events):
  none       no copy
  d2h        the frame's image -> page-locked host (what the e2e path does)
  d2h_unrel  an unrelated 25 MB device buffer -> page-locked host
  h2d_unrel  page-locked host -> an unrelated device buffer (PCIe, other direction)
  d2d_unrel  25 MB device -> device over the copy engine (HBM/L2 only, no PCIe)
  d2h_chunk8 the image copy as 8 row bands
  d2h_sm     the image written into the mapped page-locked array by an SM kernel
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2506_19415_b200 import scenegen
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
x = torch.empty((1080, 1920, 3), device="cuda")
y = torch.empty((1080, 1920, 3), device="cuda")
hs = [torch.empty((1080, 1920, 3)).pin_memory() for _ in range(2)]
side = torch.cuda.Stream()


class _HostView:  # a page-locked tensor seen as CUDA memory (UVA-mapped)
    def __init__(self, t):
        self.__cuda_array_interface__ = {"shape": tuple(t.shape), "typestr": "<f4",
                                         "data": (t.data_ptr(), False), "version": 3}


hview = [torch.as_tensor(_HostView(h), device="cuda") for h in hs]
modes = sys.argv[1:] or ["none", "d2h", "d2h_unrel", "h2d_unrel", "d2d_unrel", "none"]
for mode in modes:
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
                if mode == "d2h":
                    hs[f % 2].copy_(img, non_blocking=True)
                elif mode == "d2h_chunk8":  # the same copy as 8 row bands
                    for a, b in zip(hs[f % 2].chunk(8), img.chunk(8)):
                        a.copy_(b, non_blocking=True)
                elif mode == "d2h_sm":  # SM stores into the mapped page-locked array
                    torch.mul(img, 1.0, out=hview[f % 2])
                elif mode == "d2h_unrel":
                    hs[f % 2].copy_(x, non_blocking=True)
                elif mode == "h2d_unrel":
                    x.copy_(hs[f % 2], non_blocking=True)
                else:
                    y.copy_(x, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(mode, "fps", round(60 / (e0.elapsed_time(e1) * 1e-3), 1), flush=True)
    del s
