import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2506_19415_b200 import _lib
from paper_2506_19415_b200.runtime import VmSession
from paper_2506_19415_b200.scene_io import read_scene
class A:
    scene_dir=None; config="c2"; frames=120; width=1920; height=1080; upload_mode=None
cfg = bench.config_of(A); lay, path = bench.ensure_scene(A, 0)
scene = read_scene(path, mmap_gaussians=True); traj = bench.trajectory(A, lay)
s = VmSession(scene, exact=False)
lib = _lib.load()
for f in range(0, 36):
    s.render_frame(traj.frame_camera(f), f, out="device"); s.flush()
    n = np.zeros(1, np.uint32); lib.vms_session_cert_count(s._h, n.ctypes.data)
    print(f, int(n[0]), flush=True)
