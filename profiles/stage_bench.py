"""Stage timing without host launch overhead: warm a C2 session, then time the
render stage of one steady-state frame (a) enqueued back-to-back from the
host and (b) captured once in a CUDA graph and replayed, plus the host-side
enqueue cost of one vms_render call.  Device time is CUDA-event time."""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--warm", type=int, default=10)
    p.add_argument("--reps", type=int, default=30)
    p.add_argument("--fast", action="store_true")
    a = p.parse_args()
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
    s = VmSession(scene, exact=not a.fast)
    for f in range(a.warm):
        _, st = s.render_frame(traj.frame_camera(f), f, out="device")
    cam = traj.frame_camera(a.warm - 1)
    img = s._frame_image(cam)
    n_chunks, n_res = st["n_chunks"], st["n_resident_records"]
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # (a) back-to-back host enqueue
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(a.reps):
        s._launch_render(cam, img, n_chunks, n_res, record_events=False)
    e1.record(stream)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"render back-to-back: {e0.elapsed_time(e1) / a.reps * 1e3:.1f} us/frame device, "
          f"{(t1 - t0) / a.reps * 1e6:.1f} us/frame host enqueue")
    # (b) CUDA graph replay
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        s._launch_render(cam, img, n_chunks, n_res, record_events=False)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=side):
        s._launch_render(cam, img, n_chunks, n_res, record_events=False)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(a.reps):
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"render graph replay: {e0.elapsed_time(e1) / a.reps * 1e3:.1f} us/frame device")
    print({k: st[k] for k in ("n_kept", "n_instances", "n_resident_records", "n_chunks")})
    # (c) per-kernel device time, back-to-back enqueue (GPU stays busy)
    from paper_2506_19415_b200 import _lib

    lib = _lib.load()
    lib.vms_profile_enable(1)
    for _ in range(a.reps):
        s._launch_render(cam, img, n_chunks, n_res, record_events=False)
    torch.cuda.synchronize()
    rep = _lib.profile_report()
    lib.vms_profile_enable(0)
    print("per-kernel device time per render (us):")
    rows = []
    for line in rep.strip().splitlines():
        name, cnt, tot = line.split(",")
        rows.append((float(tot) / a.reps, int(cnt) / a.reps, name))
    for us, cnt, name in sorted(rows, reverse=True):
        print(f"  {us:9.1f} us  x{cnt:4.1f}  {name}")
    print(f"  {sum(r[0] for r in rows):9.1f} us  total")
    # (d) the visibility stage alone
    lib.vms_profile_enable(1)
    thr = s.controller.thresholds if s.controller.thresholds.size else ()
    for _ in range(a.reps):
        s.vis.launch(cam.scaled(s.vis_scale), thr, s.dot_mode)
    torch.cuda.synchronize()
    rep = _lib.profile_report()
    lib.vms_profile_enable(0)
    print("visibility per frame (us):")
    for line in rep.strip().splitlines():
        name, cnt, tot = line.split(",")
        print(f"  {float(tot) / a.reps:9.1f} us  {name}")


if __name__ == "__main__":
    main()
