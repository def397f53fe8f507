"""Benchmark: frames/sec of the per-frame VM/LOD splat path at 1080p.

Workload (BASELINE.json configs[1], "C2"): synthetic 2M-Gaussian paged city
(1000 pages x 2048 records, 3 LOD levels, written by scenegen.write_city),
1080p 120-frame street fly-through, reference session defaults (buffer 500
pages, staging 40 pages/frame, vis scale 0.25, LOD + links on).  One step =
one ``VmSession.render_frame``: visibility -> required pages -> page table ->
page uploads (pinned host -> HBM) -> preprocess -> sorts -> blend.

  value  frames/s with the image left in HBM (out="device"); page uploads are
         part of every step (the scene lives in host memory by design).
  e2e    frames/s with every frame delivered to host memory through the
         public API: the benchmark harness (harness.run_benchmark, pipelined:
         frame i + 1 is submitted before frame i is handed to the sink, so each
         frame's PCIe transfer overlaps the next frame's render; host wall
         clock, device synchronised on both sides).  e2e_sync: one synchronous
         render_frame(out=<page-locked numpy>) per step (also the N > 1 e2e).

Multi-GPU (torchrun): views are sharded - rank r renders its contiguous
block of the trajectory with its own page cache over its own pinned host copy
of the scene ("scaling": "weak": K frames per rank); the only collective is
the final NCCL gather of per-frame stats and each rank's last image.

--impl reference: the reference's CPU path (its Cython kernels compiled into
oracle/_ref, driven by the NumPy restatement in oracle/core.py) on the same
scene/path, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec at 1080p (device-timed)"
UNIT = "frames/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--fast", action="store_true", help="FP32 blend (default: FP64, reference-exact)")
    p.add_argument("--upload-mode", type=int, default=0)
    p.add_argument("--frames", type=int, default=120, help="trajectory length")
    p.add_argument("--width", type=int, default=1920)
    p.add_argument("--height", type=int, default=1080)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-frames", type=int, default=1)
    p.add_argument("--scene-dir", default=os.environ.get("VMSPLAT_SCENE_DIR", "/tmp/vmsplat_bench"))
    p.add_argument("--config", choices=("c2", "c3"), default="c2",
                   help="c2 (BASELINE configs[1], the default bench line) or c3 (20M records, "
                        "10k pages, 4 LOD levels; the scene is generated on first use, ~3 min)")
    return p.parse_args()


def scene_path(args):
    from paper_2506_19415_b200 import scenegen

    lay = scenegen.C3 if getattr(args, "config", "c2") == "c3" else scenegen.C2
    os.makedirs(args.scene_dir, exist_ok=True)
    path = os.path.join(args.scene_dir, f"city_p{lay.n_pages}_s{lay.page_size}_l{lay.levels}"
                                        f"_seed{lay.seed}.vms")
    return lay, path


def ensure_scene(args, rank):
    from paper_2506_19415_b200 import scenegen

    lay, path = scene_path(args)
    if rank == 0 and not os.path.exists(path):
        tmp = path + f".tmp{os.getpid()}"
        scenegen.write_city(tmp, lay)
        os.replace(tmp, path)
    return lay, path


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def launches_per_frame(stats, n_faces, upload_mode, n_pages=1000):
    """Kernels of libvmsplat_b200.so launched per frame (static count of the
    captured sequences in vis.cu / prims.cu / preprocess.cu / blend.cu and the
    per-frame copies in session.cu):
      visibility graph  vis_count, scan, vis_emit, vis_raster, vis_back
                        (links + flags + compaction + LOD)                5
                        (4 separate back-end kernels past 32767 pages)
      page copies       scatter_k (the uploads are copy-engine DMA;
                        upload_mode 1 adds the upload_k gather kernel)   1
      render graph      preprocess, scan, compact, radix hist + 4 passes,
                        dup_count, scan, dup_emit, clamp, radix hist + 2
                        passes, ranges, tile_order, blend                18
    (host output without zero-copy runs the blend as 4 band launches)."""
    vis = 5 if n_pages <= 32767 else 8
    up = 2 if stats["planned_copies"] else 0
    if up and upload_mode != 1:
        up = 1  # per-page cudaMemcpyAsync + scatter
    render = 18
    return vis + up + render


def workload_name(args, lay):
    n = lay.n_pages * lay.page_size
    return (f"{args.config.upper()}: {n / 1e6:.2f}M-Gaussian paged city ({lay.n_pages} pages x "
            f"{lay.page_size}, {lay.levels} LOD), {args.height}p {args.frames}-frame street "
            f"fly-through, buffer 500, staging 40, vis 0.25, LOD+links on")


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2506_19415_b200.runtime import VmSession
    from paper_2506_19415_b200.scene_io import read_scene
    from paper_2506_19415_b200 import scenegen

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    lay, path = ensure_scene(args, rank)
    if dist:
        dist.barrier()
    scene = read_scene(path, mmap_gaussians=True)
    traj = scenegen.street_path(lay, frames=args.frames, width=args.width, height=args.height)
    F = traj.frame_count
    from paper_2506_19415_b200.sharding import frame_block

    start, stop = frame_block(rank, world, F)
    block = max(1, stop - start)
    holder = {}
    step = [0]

    def fresh_session(timing=False):
        # same knobs, same warm-up frames: the device-resident, the e2e and
        # the stage-timing passes cover identical frames with identical state
        holder.pop("s", None)
        torch.cuda.empty_cache()
        holder["s"] = VmSession(scene, buffer_pages=500, staging_pages=40, vis_scale=0.25,
                                exact=not args.fast, upload_mode=args.upload_mode,
                                timing=timing)
        step[0] = 0
        for _ in range(args.warmup):
            frame("device")

    def frame(out):
        i = step[0]
        step[0] += 1
        cam = traj.frame_camera(start + (i % block))
        return holder["s"].render_frame(cam, start + i, out=out)

    fresh_session()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local_rank)

    def timed(out):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        sts = [frame(out)[1] for _ in range(args.steps)]
        e1.record(stream)
        torch.cuda.synchronize()
        holder["s"].flush()
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, sts

    sampler.start()
    ms_dev, stats = timed("device")
    clocks = sampler.stop()
    pinned = torch.empty((args.height, args.width, 3), dtype=torch.float32).pin_memory()
    fresh_session()
    ms_e2e, stats_e2e = timed(pinned.numpy())
    # e2e through the benchmark harness (harness.run_benchmark, pipelined:
    # frame i + 1 is submitted before frame i is handed to the sink, each a
    # fresh page-locked array written by the blend) - single-GPU line only
    e2e_pipe = None
    if world == 1:
        from paper_2506_19415_b200 import harness

        # warm-up frames through the same pipelined path (this also sizes the
        # session's pool of page-locked output arrays: two in flight)
        holder.pop("s", None)
        torch.cuda.empty_cache()
        holder["s"] = VmSession(scene, buffer_pages=500, staging_pages=40, vis_scale=0.25,
                                exact=not args.fast, upload_mode=args.upload_mode, timing=False)
        harness.run_benchmark(scene, traj, frames=range(args.warmup), session=holder["s"],
                              pipelined=True)
        got = []
        sink = lambda i, im: got.append(float(im[0, 0, 0]))  # noqa: E731 - touch each frame
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        harness.run_benchmark(scene, traj, frames=range(args.warmup, args.warmup + args.steps),
                              session=holder["s"], frame_sink=sink, pipelined=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        assert len(got) == args.steps
        e2e_pipe = {"value": round(args.steps / dt, 3), "unit": UNIT,
                    "api": "harness.run_benchmark(pipelined=True) -> frame_sink(i, host image)",
                    "clock": "host wall (time.perf_counter), device synchronised on both sides"}
    # third pass over the same frames with per-stage CUDA events (one sync per
    # frame): the stage breakdown and the roofline come from here
    fresh_session(timing=True)
    _, stats_t = timed("device")
    sess = holder["s"]

    # final NCCL gather of per-frame stats rows and each rank's last image
    from paper_2506_19415_b200 import sharding

    last = sess.render_frame(traj.frame_camera(start), start + step[0], out="device")[0]
    if dist:
        sharding.gather_rows(sharding.stats_rows(stats + stats_e2e), dist, device="cuda")
        imgs = [torch.empty_like(last) for _ in range(world)] if rank == 0 else None
        dist.gather(last.contiguous(), imgs, dst=0)
        dist.barrier()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return None

    hbm, peak_kind = peaks()
    W, H = args.width, args.height
    blend_s = sum(s["time_blend"] for s in stats_t)
    pre_s = sum(s["time_preprocess"] for s in stats_t)
    blend_bytes = sum(s["n_instances"] * (4 + 48) + W * H * 12 for s in stats_t)
    pre_bytes = sum(s["n_resident_records"] * (236 + 4 + 4) + s["n_kept"] * 48 for s in stats_t)
    stages = {k: 1e3 * statistics.mean(s[f"time_{k}"] for s in stats_t)
              for k in ("visibility", "update", "copy", "sort", "render", "preprocess", "tiles",
                        "blend", "device_frame")}
    dominant = "blend" if blend_s >= pre_s else "preprocess"
    if dominant == "blend":
        ach = blend_bytes / blend_s / 1e9
    else:
        ach = pre_bytes / pre_s / 1e9
    # DRAM bytes per launch of the dominant kernel from one ncu --set full
    # capture (profiles/traffic.json, written by profiles/ncu_summary.py)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            ent = json.load(open(tf)).get(dominant + "_k")
            traffic = int(ent["bytes_per_launch"]) if ent else None
        except (ValueError, KeyError, TypeError):
            traffic = None
    up_bytes = sum(s["bytes_copied"] for s in stats_t)
    up_s = sum(s["time_copy"] for s in stats_t if s["bytes_copied"])
    h2d_step = int(statistics.mean(s["bytes_copied"] for s in stats_e2e)) + 16 * int(
        statistics.mean(s.get("n_chunks", 0) for s in stats_e2e))
    d2h_step = W * H * 12 + 10 * int(statistics.mean(s["required_pages"] for s in stats_e2e))
    value = world * args.steps / (ms_dev / 1e3)
    e2e = world * args.steps / (ms_e2e / 1e3)
    launches = sum(launches_per_frame(s, len(scene.faces), args.upload_mode, scene.page_count)
                   for s in stats)
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_dev / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32",
        "data": "synthetic (scenegen city, seed 0)",
        "config": {"workload": workload_name(args, lay),
                   "width": W, "height": H, "frames": F, "parallelism": f"view-shard x{world}",
                   "blend": "fp32" if args.fast else "fp64-exact",
                   "l2": "inputs larger than L2 (resident pool up to 241 MB > 126 MB L2)",
                   "upload_mode": args.upload_mode},
        # e2e: frames delivered to host memory through the public API - the
        # benchmark harness (pipelined: frame i + 1 renders while frame i
        # crosses PCIe) on the single-GPU line; e2e_sync: one synchronous
        # render_frame(out=<page-locked array>) per step (also the N > 1 value)
        "e2e": dict(e2e_pipe or {"value": round(e2e, 3), "unit": UNIT,
                                 "api": "VmSession.render_frame(out=<page-locked numpy>)"},
                    h2d_bytes_per_step=h2d_step, d2h_bytes_per_step=d2h_step),
        "e2e_sync": {"value": round(e2e, 3), "unit": UNIT,
                     "api": "VmSession.render_frame(out=<page-locked numpy>), one call per step",
                     "h2d_bytes_per_step": h2d_step, "d2h_bytes_per_step": d2h_step},
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": round(ach, 2),
                     "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(ach / hbm, 4), "traffic": traffic,
                     "limiter": ("FP64 + XU (f32<->f64 conversion) issue in the exact blend, "
                                 "not HBM: see profiles/r1/SUMMARY.md")
                     if dominant == "blend" else "HBM read of the resident records"},
        "stages_ms": {k: round(v, 4) for k, v in stages.items()},
        "upload": {"gbs": round(up_bytes / up_s / 1e9, 2) if up_s else None,
                   "bytes": up_bytes, "frames_with_copies": sum(1 for s in stats_t if s["bytes_copied"])},
        "mean_instances": int(statistics.mean(s["n_instances"] for s in stats_t)),
        "mean_resident_records": int(statistics.mean(s["n_resident_records"] for s in stats_t)),
        "gpu_launches": int(launches),
        "host_wall_ms": {
            name: {"median": round(1e3 * statistics.median(x["time_frame_wall"] for x in st), 4),
                   "max": round(1e3 * max(x["time_frame_wall"] for x in st), 4)}
            for name, st in (("device", stats), ("e2e", stats_e2e))},
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(scene, traj, args, start_frame=args.warmup,
                                           frames=args.cpu_frames)
    if dist:
        dist.destroy_process_group()
    return out


def reference_session(scene, traj, args, warm_to):
    """Oracle session (reference kernels when built) warmed to frame
    ``warm_to`` without compositing (visibility + paging + copies only)."""
    from oracle import core, refkernels

    kern = refkernels if refkernels.available() else None
    s = core.OSession(scene, buffer_pages=500, staging_pages=40, vis_scale=0.25, kern=kern)
    for f in range(warm_to):
        s.render_frame(traj.frame_camera(f), f, want_image=False)
    return s, ("reference" if kern is not None else "port")


def cpu_baseline(scene, traj, args, start_frame, frames):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    s, kind = reference_session(scene, traj, args, start_frame)
    t0 = time.perf_counter()
    for f in range(start_frame, start_frame + frames):
        s.render_frame(traj.frame_camera(f), f)
    dt = time.perf_counter() - t0
    return {"value": round(frames / dt, 5), "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{frames} full 1080p frame(s) of the C2 trajectory at frames "
                      f"{start_frame}..{start_frame + frames - 1} after warming the page table "
                      f"(visibility+paging only) through frame {start_frame - 1}; reference "
                      f"Cython kernels (oracle/_ref) driven by oracle/core.py, 1 thread"}


def _reference_worker(job):
    """One host core's share of the reference arm: a fresh reference session
    (oracle/_ref Cython kernels driven by oracle/core.py) on its own block of
    the trajectory, warmed without compositing, then n timed frames."""
    args, start, n = job
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from paper_2506_19415_b200 import scenegen
    from paper_2506_19415_b200.scene_io import read_scene

    lay, path = ensure_scene(args, 0)
    scene = read_scene(path, mmap_gaussians=True)
    traj = scenegen.street_path(lay, frames=args.frames, width=args.width, height=args.height)
    s, kind = reference_session(scene, traj, args, 0)
    f = start
    for _ in range(args.warmup):
        s.render_frame(traj.frame_camera(f % traj.frame_count), f, want_image=False)
        f += 1
    t0 = time.perf_counter()
    for _ in range(n):
        s.render_frame(traj.frame_camera(f % traj.frame_count), f)
        f += 1
    return n, time.perf_counter() - t0, kind


def reference_workers() -> int:
    """Host cores for the reference arm (one single-threaded session each),
    capped so the per-session render buffers (~0.25 GB each) stay modest."""
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        cores = os.cpu_count() or 1
    cap = int(os.environ.get("VMSPLAT_REF_WORKERS", "32"))
    return max(1, min(cores, cap))


def run_reference(args, rank, world):
    """The reference's own CPU path on all the host cores it can use: the
    reference session is sequential per frame (page-table state), so each
    core runs an independent session on a contiguous block of the trajectory
    (the view sharding of the GPU arm); value = frames / slowest worker."""
    if rank != 0:
        return None
    import multiprocessing as mp

    lay, _ = ensure_scene(args, 0)  # written once, before the workers start
    P = reference_workers()
    n = min(args.steps, 12)  # bounded sample: ~1.3 s per 1080p frame per core
    F = args.frames
    jobs = [(args, (w * F) // P, n) for w in range(P)]
    if P == 1:
        res = [_reference_worker(jobs[0])]
    else:
        with mp.get_context("fork").Pool(P) as pool:
            res = pool.map(_reference_worker, jobs)
    frames = sum(r[0] for r in res)
    dt = max(r[1] for r in res)
    kind = res[0][2]
    v = frames / dt
    return {"metric": METRIC, "value": round(v, 5), "unit": UNIT, "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * dt / n, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (scenegen city, seed 0)", "impl": "reference",
            "config": {"workload": workload_name(args, lay), "width": args.width,
                       "height": args.height},
            "cpu_baseline": {"value": round(v, 5), "unit": UNIT, "cores": P, "kind": kind,
                             "sample": f"{P} worker process(es), one core and one reference "
                                       f"session each on its own block of the {F}-frame "
                                       f"trajectory: {args.warmup} warm-up frames without "
                                       f"compositing, then {n} timed full 1080p frames "
                                       "(step count capped at 12); frames / slowest worker"},
            "e2e": {"value": round(v, 5), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    if os.environ.get("VMSPLAT_WATCHDOG"):
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["VMSPLAT_WATCHDOG"]), repeat=True)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_ours(args, rank, world, local_rank)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
