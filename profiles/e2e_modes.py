"""End-to-end output modes on the bench workload: ms per frame for
render_frame into (a) a page-locked numpy array (zero-copy blend writes),
(b) a pageable numpy array (device image -> pinned staging -> array),
(c) out=None (fresh page-locked array per frame), (d) device only."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
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
    pinned = torch.empty((1080, 1920, 3), dtype=torch.float32).pin_memory().numpy()
    pageable = np.empty((1080, 1920, 3), np.float32)
    modes = {"pinned": pinned, "pageable": pageable, "none": None, "device": "device"}
    for name, out in modes.items():
        s = VmSession(scene, timing=False)
        for f in range(5):
            s.render_frame(traj.frame_camera(f), f, out=out)
        s.flush()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for f in range(5, 65):
            s.render_frame(traj.frame_camera(f), f, out=out)
        s.flush()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 60
        print(f"{name:9s} {1e3 * dt:7.3f} ms/frame  {1 / dt:8.1f} fps", flush=True)
        del s
    # where an end-to-end frame goes: device stage events + host wall per call
    s = VmSession(scene, timing=True)
    sts = [s.render_frame(traj.frame_camera(f), f, out=pinned)[1] for f in range(65)][5:]
    keys = ("visibility", "update", "copy", "preprocess", "sort", "tiles", "blend",
            "device_frame", "frame_wall")
    print("pinned+timing mean ms:", {k: round(1e3 * float(np.mean([x["time_" + k] for x in sts])), 4)
                                      for k in keys})


if __name__ == "__main__":
    main()
