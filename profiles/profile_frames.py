"""Profiling driver: warm a session of a bench configuration (bench.CONFIGS:
scene, buffer, staging, path) for --warm frames, then render --frames frames
between cudaProfilerStart/Stop so that `ncu --profile-from-start off` sees
only steady-state frames.  --trace also prints the blend's per-CTA schedule
of the last frame (vms_debug_blend_trace).

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \\
      --csv --log-file gpurun_out/launches.csv python profiles/profile_frames.py
  ncu --profile-from-start off --set full --clock-control none --import-source on \\
      -k regex:blend_k -c 1 -o gpurun_out/blend python profiles/profile_frames.py --warm 25
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
    p.add_argument("--config", choices=("c2", "c3", "c4"), default="c2")
    p.add_argument("--width", type=int, default=1920)
    p.add_argument("--height", type=int, default=1080)
    p.add_argument("--trace", action="store_true")
    p.add_argument("--timing", action="store_true", help="print per-stage device times")
    a = p.parse_args()
    import numpy as np
    import torch

    import bench
    from paper_2506_19415_b200 import _lib
    from paper_2506_19415_b200.runtime import VmSession
    from paper_2506_19415_b200.scene_io import read_scene

    class A:
        scene_dir = os.environ.get("VMSPLAT_SCENE_DIR")
        config = a.config
        frames = 120
        width = a.width
        height = a.height
        upload_mode = None

    cfg = bench.config_of(A)
    lay, path = bench.ensure_scene(A, 0)
    scene = read_scene(path, mmap_gaussians=True)
    traj = bench.trajectory(A, lay)
    s = VmSession(scene, buffer_pages=cfg["buffer"], staging_pages=cfg["staging"],
                  vis_scale=0.25, exact=not a.fast, timing=a.timing,
                  upload_mode=bench.upload_mode_of(A))
    for f in range(a.warm):
        s.render_frame(traj.frame_camera(f), f, out="device")
    s.flush()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for f in range(a.warm, a.warm + a.frames):
        trace = None
        if a.trace and f == a.warm + a.frames - 1:
            trace = torch.zeros(8 * 200000, dtype=torch.int64, device="cuda")
            _lib.load().vms_debug_blend_trace(trace.data_ptr())
        _, st = s.render_frame(traj.frame_camera(f), f, out="device")
        if a.timing:
            print(f, {k: round(st[k] * 1e3, 3) for k in st if k.startswith("time_")})
    s.flush()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print({k: st[k] for k in ("n_kept", "n_instances", "n_resident_records", "required_pages",
                              "bytes_copied", "n_tris")})
    if trace is not None:
        _lib.load().vms_debug_blend_trace(None)
        t = trace.view(-1, 8).cpu().numpy()
        t = t[t[:, 1] > 0]
        t0 = t[:, 0].min()
        st_, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
        dur = en - st_
        ln = (t[:, 3] >> 32).astype(np.int64)
        print(f"blend: {len(t)} CTAs, span {en.max():.1f} us, sum {dur.sum():.0f} us, "
              f"median CTA {np.median(dur):.1f} us")
        for q in (50, 90, 99, 100):
            print(f"  list length p{q}: {np.percentile(ln, q):.0f}, CTA us p{q}: "
                  f"{np.percentile(dur, q):.1f}")
        for i in np.argsort(-dur)[:10]:
            print(f"  CTA start {st_[i]:.1f} dur {dur[i]:.1f} list {ln[i]} tile "
                  f"{int(t[i, 3] & 0xffffffff)} sm {t[i, 2]}")


if __name__ == "__main__":
    main()
