"""Per-warp blend phase split (VMSPLAT_BLEND_PROF=1): batch barrier, staging,
splat walk, end barrier - cycles summed over every warp of a frame's blend."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2506_19415_b200 import _lib
from paper_2506_19415_b200.runtime import VmSession
from paper_2506_19415_b200.scene_io import read_scene


class A:
    scene_dir = None; config = "c2"; frames = 120; width = 1920; height = 1080; upload_mode = None


lay, path = bench.ensure_scene(A, 0)
scene = read_scene(path, mmap_gaussians=True)
traj = bench.trajectory(A, lay)
s = VmSession(scene, timing=False)
lib = _lib.load()
acc = np.zeros(4, np.uint64)
for f in range(0, 35):
    s.render_frame(traj.frame_camera(f), f, out="device")
    s.flush()
    lib.vms_debug_blend_prof(acc.ctypes.data)
    tot = float(acc.sum()) or 1.0
    if f in (5, 12, 20, 25, 30):
        print(f"frame {f}: batch barrier {acc[0] / tot:.1%}, staging {acc[1] / tot:.1%}, "
              f"splat walk {acc[2] / tot:.1%}, end barrier {acc[3] / tot:.1%} "
              f"(warp-cycles {tot:.3g})", flush=True)
