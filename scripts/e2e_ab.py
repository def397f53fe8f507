"""e2e A/B helper: the pipelined harness over C2 frames 5-64, 5 repetitions
in one process (fresh session each), prints the median frames/s.  Knobs are
read from the environment (VMSPLAT_*) by the session."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2506_19415_b200 import harness
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
fps = []
reps = int(os.environ.get("AB_REPS", "5"))
for rep in range(reps):
    t_a = time.perf_counter()
    s = VmSession(scene, buffer_pages=500, staging_pages=40, vis_scale=0.25, timing=False,
                  upload_mode=int(os.environ["AB_UPLOAD"]) if os.environ.get("AB_UPLOAD") else None)
    t_b = time.perf_counter()
    harness.run_benchmark(scene, traj, frames=range(5), session=s, pipelined=True)
    torch.cuda.synchronize()
    if os.environ.get("AB_VERBOSE"):
        print(f"rep {rep}: session {1e3 * (t_b - t_a):.1f} ms, warm-up "
              f"{1e3 * (time.perf_counter() - t_b):.1f} ms", flush=True)
    t0 = time.perf_counter()
    harness.run_benchmark(scene, traj, frames=range(5, 65), session=s, pipelined=True,
                          frame_sink=lambda i, im: None)
    torch.cuda.synchronize()
    fps.append(60 / (time.perf_counter() - t0))
    if os.environ.get("AB_VERBOSE"):
        print(f"rep {rep}: {fps[-1]:.0f} frames/s", flush=True)
    s.close()
print(os.environ.get("AB_TAG", ""), "e2e median", round(statistics.median(fps), 1),
      "all", [round(x) for x in fps])
