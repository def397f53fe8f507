import os, sys
sys.path.insert(0, "/root/repo")
os.chdir("/root/repo")
import torch, bench
from paper_2506_19415_b200.runtime import VmSession
from paper_2506_19415_b200.scene_io import read_scene
class A:
    config = "c2"; scene_dir = None; frames = 120; width = 1920; height = 1080
lay, path = bench.ensure_scene(A, 0)
scene = read_scene(path, mmap_gaussians=True)
traj = bench.trajectory(A, lay)
s = VmSession(scene, buffer_pages=500, staging_pages=40, vis_scale=0.25, timing=True)
for f in range(0, 14):
    img, st = s.render_frame(traj.frame_camera(f), f, out="device")
    print(f, {k: st[k] for k in st if k in ("n_kept", "n_instances", "overflow", "n_need", "time_tiles", "time_blend", "planned_copies")}, flush=True)
