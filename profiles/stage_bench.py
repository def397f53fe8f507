"""Per-kernel device time of steady-state frames of the bench workload (C2,
1080p street path): warm a session, then render --frames frames with the
library's per-launch event marks enabled (vms_profile_enable) and print the
per-kernel device time per frame plus the per-frame stage events."""

import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--warm", type=int, default=10)
    p.add_argument("--frames", type=int, default=10)
    p.add_argument("--fast", action="store_true")
    a = p.parse_args()
    import torch

    import bench
    from paper_2506_19415_b200 import _lib, scenegen
    from paper_2506_19415_b200.runtime import VmSession
    from paper_2506_19415_b200.scene_io import read_scene

    class A:
        scene_dir = os.environ.get("VMSPLAT_SCENE_DIR")
        config = "c2"
        frames = 120
        width = 1920
        height = 1080
        upload_mode = None

    lay, path = bench.ensure_scene(A, 0)
    scene = read_scene(path, mmap_gaussians=True)
    traj = bench.trajectory(A, lay)
    s = VmSession(scene, exact=not a.fast, timing=False)
    for f in range(a.warm):
        s.render_frame(traj.frame_camera(f), f, out="device")
    s.flush()
    lib = _lib.load()
    lib.vms_profile_enable(1)
    sts = []
    for f in range(a.warm, a.warm + a.frames):
        sts.append(s.render_frame(traj.frame_camera(f), f, out="device")[1])
    s.flush()
    torch.cuda.synchronize()
    rep = _lib.profile_report()
    lib.vms_profile_enable(0)
    rows = []
    for line in rep.strip().splitlines():
        name, cnt, tot = line.split(",")
        rows.append((float(tot) / a.frames, int(cnt) / a.frames, name))
    print(f"per-kernel device time per frame (us), frames {a.warm}..{a.warm + a.frames - 1}:")
    for us, cnt, name in sorted(rows, reverse=True):
        print(f"  {us:9.1f} us  x{cnt:5.1f}  {name}")
    print(f"  {sum(r[0] for r in rows):9.1f} us  total kernel time")
    print("mean counters:", {k: int(statistics.mean(st[k] for st in sts)) for k in
                             ("n_kept", "n_instances", "n_resident_records", "n_chunks",
                              "required_pages", "bytes_copied", "n_tris")})
    # stage events (one sync per frame)
    s.timing = True
    ts = [s.render_frame(traj.frame_camera(f), f, out="device")[1]
          for f in range(a.warm + a.frames, a.warm + 2 * a.frames)]
    print("stage ms (timing pass):", {k: round(1e3 * statistics.mean(t[f"time_{k}"] for t in ts), 4)
                                      for k in ("visibility", "update", "copy", "preprocess",
                                                "sort", "tiles", "blend", "device_frame",
                                                "frame_wall")})


if __name__ == "__main__":
    main()
