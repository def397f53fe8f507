"""Per-frame table over the whole C2 trajectory (timing mode): counters and
stage device times, to see how the work varies along the path."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2506_19415_b200 import scenegen
    from paper_2506_19415_b200.runtime import VmSession
    from paper_2506_19415_b200.scene_io import read_scene

    class A:
        scene_dir = os.environ.get("VMSPLAT_SCENE_DIR", "/tmp/vmsplat_bench")

    fast = "--fast" in sys.argv
    lay, path = bench.ensure_scene(A, 0)
    scene = read_scene(path, mmap_gaussians=True)
    traj = scenegen.street_path(lay, frames=120)
    s = VmSession(scene, exact=not fast, timing=True)
    print("frame req res_rec kept inst(M) need(M) copiedMB | vis pre sort tiles blend frame wall (ms)")
    for f in range(traj.frame_count):
        _, t = s.render_frame(traj.frame_camera(f), f, out="device")
        print(f"{f:4d} {t['required_pages']:4d} {t['n_resident_records']:7d} {t['n_kept']:7d} "
              f"{t['n_instances'] / 1e6:6.2f} {t['n_need'] / 1e6:6.2f} {t['bytes_copied'] / 1e6:6.1f} | "
              + " ".join(f"{1e3 * t['time_' + k]:6.3f}" for k in
                         ("visibility", "preprocess", "sort", "tiles", "blend", "device_frame",
                          "frame_wall")))
    if "--device" in sys.argv:
        # untimed, pipelined pass: host wall time per call
        import time
        s2 = VmSession(scene, exact=not fast, timing=False)
        walls = []
        for f in range(traj.frame_count):
            t0 = time.perf_counter()
            s2.render_frame(traj.frame_camera(f), f, out="device")
            walls.append(1e3 * (time.perf_counter() - t0))
        s2.flush()
        print("device-mode host ms per call:", " ".join(f"{w:.2f}" for w in walls))


if __name__ == "__main__":
    main()
