"""Profiling driver: warm a C2 session (bench workload) for --warm frames,
then render --frames frames between cudaProfilerStart/Stop so that
`ncu --profile-from-start off` sees only steady-state frames.

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/launches.csv python profiles/profile_frames.py
  ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:blend_k -c 1 -o gpurun_out/blend python profiles/profile_frames.py
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--warm", type=int, default=10)
    p.add_argument("--frames", type=int, default=2)
    p.add_argument("--fast", action="store_true")
    p.add_argument("--config", choices=("c2", "c3"), default="c2")
    a = p.parse_args()
    import torch

    import bench
    from paper_2506_19415_b200 import scenegen
    from paper_2506_19415_b200.runtime import VmSession
    from paper_2506_19415_b200.scene_io import read_scene

    class A:
        scene_dir = os.environ.get("VMSPLAT_SCENE_DIR", "/tmp/vmsplat_bench")
        config = a.config

    lay, path = bench.ensure_scene(A, 0)
    scene = read_scene(path, mmap_gaussians=True)
    traj = scenegen.street_path(lay, frames=120)
    s = VmSession(scene, exact=not a.fast, timing=False)
    for f in range(a.warm):
        s.render_frame(traj.frame_camera(f), f, out="device")
    s.flush()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for f in range(a.warm, a.warm + a.frames):
        _, st = s.render_frame(traj.frame_camera(f), f, out="device")
    s.flush()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print({k: st[k] for k in ("n_kept", "n_instances", "n_resident_records", "required_pages",
                              "bytes_copied")})


if __name__ == "__main__":
    main()
