"""Host-side timeline of the pipelined harness loop (bench workload):
per frame, the time spent in render_frame(wait=False) and in wait(1)."""
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
    s = VmSession(scene, timing=False)
    for f in range(5):
        s.render_frame(traj.frame_camera(f), f, out="device")
    s.flush()
    for mode in ("none-async", "pinned-sync", "none-sync"):
        pinned = torch.empty((1080, 1920, 3), dtype=torch.float32).pin_memory().numpy()
        t_sub, t_wait = [], []
        held = None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for f in range(5, 35):
            a = time.perf_counter()
            if mode == "none-async":
                img, _ = s.render_frame(traj.frame_camera(f), f, wait=False)
            elif mode == "pinned-sync":
                img, _ = s.render_frame(traj.frame_camera(f), f, out=pinned)
            else:
                img, _ = s.render_frame(traj.frame_camera(f), f)
            b = time.perf_counter()
            if mode == "none-async" and held is not None:
                s.wait(1)
            c = time.perf_counter()
            held = img
            t_sub.append(b - a)
            t_wait.append(c - b)
        s.wait(0)
        dt = time.perf_counter() - t0
        print(f"{mode:12s} {30 / dt:7.1f} fps  submit ms median {1e3 * np.median(t_sub):.3f} "
              f"max {1e3 * np.max(t_sub):.3f}  wait ms median {1e3 * np.median(t_wait):.3f}",
              flush=True)


if __name__ == "__main__":
    main()
