"""Per-CTA blend schedule of one steady-state frame (bench workload): CTA
start/end times, SM, tile list length -> how much of the kernel is tail."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import bench
    from paper_2506_19415_b200 import _lib, scenegen
    from paper_2506_19415_b200.runtime import VmSession
    from paper_2506_19415_b200.scene_io import read_scene

    class A:
        config = "c2"
        scene_dir = None
        frames = 120
        width = 1920
        height = 1080

    frame = int(sys.argv[1]) if len(sys.argv) > 1 else 25
    lay, path = bench.ensure_scene(A, 0)
    scene = read_scene(path, mmap_gaussians=True)
    traj = bench.trajectory(A, lay)
    s = VmSession(scene, timing=False)
    lib = _lib.load()
    for f in range(frame):
        s.render_frame(traj.frame_camera(f), f, out="device")
    s.flush()
    buf = torch.zeros(8 * 40000, dtype=torch.int64, device="cuda")
    lib.vms_debug_blend_trace(buf.data_ptr())
    s.render_frame(traj.frame_camera(frame), frame, out="device")
    s.flush()
    torch.cuda.synchronize()
    lib.vms_debug_blend_trace(None)
    t = buf.view(-1, 8).cpu().numpy()
    t = t[t[:, 1] > 0]
    t0 = t[:, 0].min()
    st = (t[:, 0] - t0) / 1e3
    en = (t[:, 1] - t0) / 1e3
    dur = en - st
    ln = (t[:, 3] >> 32).astype(np.int64)
    total = en.max()
    print(f"frame {frame}: {len(t)} CTAs, kernel span {total:.1f} us, "
          f"sum CTA time {dur.sum():.0f} us, mean {dur.mean():.1f} us")
    for q in (50, 90, 99, 99.9, 100):
        print(f"  CTA duration p{q}: {np.percentile(dur, q):.1f} us")
    order = np.argsort(-dur)[:12]
    print("  longest CTAs: (start, dur, list length, launch index, stages, stage us, proc us)")
    for i in order:
        print(f"    {st[i]:8.1f} {dur[i]:8.1f} {ln[i]:7d} {i:6d} {t[i, 4]:5d} "
              f"{t[i, 5] / 1965:8.1f} {t[i, 6] / 1965:8.1f}")
    print(f"  all CTAs: staging {t[:, 5].sum() / 1965 / 1e3:.1f} ms, processing {t[:, 6].sum() / 1965 / 1e3:.1f} ms (CTA-sum)")
    # SM busy fraction over time
    sms = t[:, 2].astype(np.int64) & 0xFFFF
    last = np.zeros(sms.max() + 1)
    for i in range(len(t)):
        last[sms[i]] = max(last[sms[i]], en[i])
    print(f"  SM finish time: min {last.min():.1f} median {np.median(last):.1f} max {last.max():.1f} us")
    slots = 148 * (8 if len(t) > 9000 else 4)
    print(f"  bound: CTA-time / {slots} slots {dur.sum() / slots:.1f} us, longest CTA {dur.max():.1f} us")
    for cut in (2048, 4096, 8192):
        m = ln >= cut
        print(f"  lists >= {cut}: {m.sum()} CTAs, {dur[m].sum() / dur.sum():.1%} of CTA time, "
              f"longest {dur[m].max() if m.any() else 0:.1f} us")
    big = np.flatnonzero(ln >= 4096)
    print(f"  CTAs with lists >= 4096: {len(big)}; launch index, start, dur, length:")
    for i in big[:64]:
        print(f"    {i:6d} {st[i]:8.1f} {dur[i]:8.1f} {ln[i]:7d}")
    corr = np.corrcoef(ln, dur)[0, 1]
    print(f"  corr(list length, CTA duration) = {corr:.3f}; launch index of longest: "
          f"{sorted(order.tolist())}")


if __name__ == "__main__":
    main()
