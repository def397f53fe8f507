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
         the session's four frame slots stay full - frame i goes to the sink
         once frame i + 4 is submitted - so each frame's PCIe transfer
         overlaps the next frames' renders; host wall
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

import os

# The reference's host path goes through NumPy -> OpenBLAS (Camera.world_to_view,
# project_records).  Its hot loops are single-threaded, and an all-core BLAS
# pool per worker oversubscribes the host when several reference sessions run
# side by side.  The pool size is fixed when OpenBLAS loads, i.e. at the first
# NumPy import, so it is pinned here, before anything imports NumPy.
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[_v] = "1"

import argparse  # noqa: E402
import gc  # noqa: E402
import json  # noqa: E402
import statistics
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402,F401

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
    p.add_argument("--upload-mode", type=int, default=None,
                   help="0 DMA from the page-locked scene, 1 gather kernel, 2 host-thread "
                        "streaming; default: the config's (auto for c2/c3, 2 for c4)")
    p.add_argument("--frames", type=int, default=120, help="trajectory length")
    p.add_argument("--width", type=int, default=1920)
    p.add_argument("--height", type=int, default=1080)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-frames", type=int, default=8)
    p.add_argument("--scene-dir", default=os.environ.get("VMSPLAT_SCENE_DIR"))
    p.add_argument("--config", choices=("c2", "c3", "c4"), default="c2",
                   help="c2 (BASELINE configs[1], the default bench line); c3 (20M records, "
                        "10k pages, 4 LOD levels); c4 (609M records, 144 GB in host DRAM) - "
                        "scenes are generated on first use")
    return p.parse_args()


DATA = "synthetic (scenegen city, seed 0; records generated, not captured)"

# Benchmark configurations (BASELINE.json "configs").  Session
# knobs follow the reference defaults for C2 (buffer 500, staging 40); the
# larger scenes get a page cache sized for their working set.
CONFIGS = {
    "c2": {"layout": "C2", "buffer": 500, "staging": 40, "blocks": 3, "scene_dir": "/dev/shm"},
    "c3": {"layout": "C3", "buffer": 4096, "staging": 40, "blocks": 3, "scene_dir": "/dev/shm"},
    # C4: the largest scene this box can hold (see scenegen.C4), written to
    # tmpfs (host DRAM) and paged from there; the camera flies down a long
    # street so pages stream in every frame
    "c4": {"layout": "C4", "buffer": 2048, "staging": 160, "blocks": 24,
           "scene_dir": "/dev/shm", "upload_mode": 2},
}


def config_of(args):
    return CONFIGS[args.config]


def upload_mode_of(args):
    """--upload-mode, else the config's default (None = the session's auto:
    DMA from the page-locked scene when it can be page-locked).  C4's 144 GB
    tmpfs scene cannot be page-locked reliably (the boxes pin ~116 GB at
    most), so it streams through the session's bounce buffer."""
    if args.upload_mode is not None:
        return args.upload_mode
    return config_of(args).get("upload_mode")


def scene_path(args):
    from paper_2506_19415_b200 import scenegen

    cfg = config_of(args)
    lay = getattr(scenegen, cfg["layout"])
    d = args.scene_dir or os.path.join(cfg["scene_dir"], "vmsplat_bench")
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, f"city_p{lay.n_pages}_s{lay.page_size}_l{lay.levels}"
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


def trajectory(args, lay):
    from paper_2506_19415_b200 import scenegen

    return scenegen.street_path(lay, frames=args.frames, width=args.width, height=args.height,
                                blocks=config_of(args)["blocks"])


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    polled every 2 ms on a thread (the timed region of a default run is only
    ~20 ms, shorter than nvidia-smi's sampling period); nvidia-smi -lms as the
    fallback when NVML is unavailable."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.nvml = None
        self.samples = []  # (sm MHz, set of reasons)
        self.max_mhz = None
        self.stop_ev = threading.Event()

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            self.nvml = (nv, h, bits)
            self._poll_once()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:  # noqa: BLE001 - any NVML failure -> nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)  # nvidia-smi start-up: let its first samples land
        except (OSError, FileNotFoundError):
            self.proc = None

    def _poll_once(self):
        nv, h, bits = self.nvml
        mhz = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.samples.append((mhz, {n for n, b in bits.items() if r & b}))

    def _poll(self):
        while not self.stop_ev.is_set():
            try:
                self._poll_once()
            except Exception:  # noqa: BLE001
                return
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.strip().split(",")]
            if len(parts) < 6:
                continue
            try:
                mhz, self.max_mhz = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            self.samples.append((mhz, {n for n, v in zip(self.NAMES, parts[2:6])
                                       if v.lower().startswith("active")}))

    def stop(self):
        if self.nvml is not None:
            self.stop_ev.set()
            self.thread.join(timeout=1.0)
            self._poll_once()
            src = "nvml, 2 ms period"
        elif self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            src = "nvidia-smi -lms 100"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml and nvidia-smi unavailable"]}
        sm = [m for m, _ in self.samples]
        reasons = set().union(*[r for _, r in self.samples]) if self.samples else set()
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm), "source": src}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def launches_per_frame(stats, n_faces, upload_mode, n_pages=1000, device_table=False,
                       exact=True):
    """Kernels of libvmsplat_b200.so launched per frame (static count of the
    captured sequences in vis.cu / prims.cu / preprocess.cu / blend.cu and the
    per-frame copies in session.cu):
      visibility graph  vis_count, scan, vis_emit, vis_raster, vis_back
                        (links + flags + compaction + LOD)                5
                        (4 separate back-end kernels past 32767 pages)   +3
                        (binned raster from 65536 faces: bin count, scan,
                         bin emit, radix hist + 2 passes, tile ranges,
                         chunk count, scan, merge)                       +10
      page copies       scatter_k (the uploads are copy-engine DMA;
                        upload_mode 1 adds the upload_k gather kernel)   1
                        (the device page table: dpt_update_k and the
                         chunk-table sums / scan / emit kernels)         +4
      render graph      preprocess, scan, compact, radix hist + 4 passes,
                        dup_count, scan, dup_emit, tile_prep, 2 radix
                        passes, blend                                    15
                        (exact blend: hot_list_k + blend_hot_k on the
                         forked stream; fast blend: blend_repair_k)      +2 / +1
    (host output without zero-copy runs the blend as 4 band launches).
    Checked against the ncu launch list of the bench command
    (profiles/r2/launches_bench.csv: 26.9 launches per frame)."""
    vis = 5 if n_pages <= 32767 else 8
    if n_faces >= 65536 and os.environ.get("VMSPLAT_VIS_BIN", "") != "0":
        vis += 10
    up = 0
    if stats["planned_copies"]:
        up = 2 if upload_mode == 1 else 1
    if device_table:
        vis += 4
    render = 15 + (2 if exact else 1)
    return vis + up + render


def workload_name(args, lay):
    cfg = config_of(args)
    n = lay.n_pages * lay.page_size
    return (f"{args.config.upper()}: {n / 1e6:.2f}M-Gaussian paged city ({lay.n_pages} pages x "
            f"{lay.page_size}, {lay.levels} LOD), {args.height}p {args.frames}-frame street "
            f"fly-through ({cfg['blocks']} blocks), buffer {cfg['buffer']}, staging "
            f"{cfg['staging']}, vis 0.25, LOD+links on")


def bench_config(args, lay, world=1):
    """The ``config`` object of BOTH arms' lines (same workload, same frames)."""
    cfg = config_of(args)
    pool_mb = cfg["buffer"] * lay.page_size * 236 / 1e6
    return {"workload": workload_name(args, lay), "width": args.width, "height": args.height,
            "frames": args.frames, "timed_frames": [args.warmup, args.warmup + args.steps - 1],
            "parallelism": f"view-shard x{world}",
            "blend": "fp32-certified (<= 1e-3, uncertifiable pixels re-blended in FP64)"
            if args.fast else "fp64-exact",
            "l2": f"inputs larger than L2 (resident page pool up to {pool_mb:.0f} MB, "
                  f"126 MB L2; the frame's records stream from it every step)",
            "upload_mode": upload_mode_of(args),
            "page_table": "host" if os.environ.get("VMSPLAT_DEVICE_TABLE") == "0"
            else "device (dpt_update_k) when capacity <= 8192 and levels <= 6, else host"}


def measure_pcie(torch, nbytes=256 << 20, reps=10):
    """Pinned host <-> device copy peaks (best of ``reps``, CUDA events on a
    side stream): the PCIe roofline of the page uploads."""
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    best = {"h2d": 0.0, "d2h": 0.0}
    for _ in range(reps):
        for k, (dst, src) in (("h2d", (d, h)), ("d2h", (h, d))):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record()
                dst.copy_(src, non_blocking=True)
                e1.record()
            e1.synchronize()
            best[k] = max(best[k], nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del h, d
    return {"h2d_gbs": round(best["h2d"], 2), "d2h_gbs": round(best["d2h"], 2),
            "how": f"pinned {nbytes >> 20} MB cudaMemcpyAsync, best of {reps}"}


def frame_bytes(s, W, H, P):
    """Algorithmic bytes of one frame per SURVEY §8(d) (HBM side, PCIe side).
    S_splat = 48 B (BlendRec), S_out = 48 B; L_dir (link targets of directly
    visible pages) is not counted by the session and is left out (< 1 %)."""
    V = s["vis_pixels"]
    T, Nres, Nk, M = s["n_tris"], s["n_resident_records"], s["n_kept"], s["n_instances"]
    hbm = {
        "visibility": T * 72 + V * 12,
        "reduce": V * 12 + (P + 1) * 4.125,
        "preprocess": Nres * 236 + Nk * 48,
        "depth_sort": Nk * 4 + 4 * Nk * 16,
        "tile_dup": Nk * 12 + M * 8,
        "tile_sort": 2 * M * 16,
        "blend": M * (4 + 48) + W * H * 12,
    }
    return hbm, s["bytes_copied"]


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2506_19415_b200.runtime import VmSession
    from paper_2506_19415_b200.scene_io import read_scene

    # one GPU per rank; VMSPLAT_DIST_BACKEND=gloo (with ranks sharing the
    # visible GPUs round-robin) only exercises the multi-rank code path on a
    # box with fewer GPUs than ranks - its numbers are not a scaling result
    backend = os.environ.get("VMSPLAT_DIST_BACKEND", "nccl")
    dev_index = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev_index)
    coll = "cuda" if backend == "nccl" else "cpu"
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    cfg = config_of(args)
    lay, path = ensure_scene(args, rank)
    if dist:
        dist.barrier()
    # every rank maps the same file; the sessions register that mapping
    # (runtime.HostScene), so the ranks share one host-resident copy
    scene = read_scene(path, mmap_gaussians=True)
    traj = trajectory(args, lay)
    F = traj.frame_count
    from paper_2506_19415_b200.sharding import frame_block, shard_frame

    start, _ = frame_block(rank, world, F)
    holder = {}
    step = [0]
    W, H = args.width, args.height

    def new_session(timing=False):
        old = holder.pop("s", None)
        if old is not None:
            old.close()  # now, not inside a later timed region (cycle collector)
        gc.collect()
        torch.cuda.empty_cache()
        holder["s"] = VmSession(scene, buffer_pages=cfg["buffer"], staging_pages=cfg["staging"],
                                vis_scale=0.25, exact=not args.fast,
                                upload_mode=upload_mode_of(args), timing=timing)
        step[0] = 0
        return holder["s"]

    def fresh_session(timing=False):
        # same knobs, same warm-up frames: the device-resident, the e2e and
        # the stage-timing passes cover identical frames with identical state
        new_session(timing)
        for _ in range(args.warmup):
            frame("device")

    def frame(out):
        # rank r renders trajectory frames start, start + 1, ... (its block,
        # continuing into the next block when more frames are timed than a
        # block holds; frame F wraps to frame 0); frame indices are global
        i = step[0]
        step[0] += 1
        f = shard_frame(start, i, F)
        return holder["s"].render_frame(traj.frame_camera(f), start + i, out=out)

    fresh_session()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(dev_index)
    # N > 1: each timed frame is rendered into its own slot of a
    # device-resident frame stack, gathered to rank 0 after the timed region
    # (N = 1 leaves each frame in the session's two alternating device
    # buffers: writing a fresh 25 MB slot per frame measured ~7 % slower)
    stack = torch.empty((args.steps, H, W, 3), dtype=torch.float32, device="cuda") \
        if world > 1 else None

    def timed(out):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        sts = [frame(out if out is not None else
                     (stack[k] if stack is not None else "device"))[1]
               for k in range(args.steps)]
        e1.record(stream)
        torch.cuda.synchronize()
        holder["s"].flush()
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms], device=coll)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, sts

    sampler.start()
    ms_dev, stats = timed(None)
    clocks = sampler.stop()
    # the only collective of the path: every timed frame's image and stats
    # row to rank 0 (NCCL over NVLink), after the timed region
    from paper_2506_19415_b200 import sharding

    gathered = None
    if dist:
        sharding.gather_rows(sharding.stats_rows(stats), dist, device=coll)
        src = stack if coll == "cuda" else stack.cpu()
        frames_all = [torch.empty_like(src) for _ in range(world)] if rank == 0 else None
        dist.gather(src, frames_all, dst=0)
        if rank == 0:
            gathered = {"frames": world * args.steps,
                        "bytes": world * stack.numel() * 4,
                        "nonzero_frames": int(sum(int((fr.flatten(1).amax(1) > 0).sum())
                                                  for fr in frames_all))}
        del frames_all
    pinned = torch.empty((H, W, 3), dtype=torch.float32).pin_memory()
    fresh_session()
    ms_e2e, stats_e2e = timed(pinned.numpy())
    # e2e through the benchmark harness (harness.run_benchmark, pipelined:
    # frames i + 1 .. i + 4 are submitted before frame i goes to the sink, each a
    # fresh page-locked array written by the blend) - single-GPU line only
    e2e_pipe = None
    traj_fps = None
    if world == 1:
        from paper_2506_19415_b200 import harness

        # warm-up frames through the same pipelined path (this also sizes the
        # session's pool of page-locked output arrays: slots + 2 of them)
        sess = new_session()
        harness.run_benchmark(scene, traj, frames=range(args.warmup), session=sess,
                              pipelined=True)
        got = []
        sink = lambda i, im: got.append(float(im[0, 0, 0]))  # noqa: E731 - touch each frame
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        harness.run_benchmark(scene, traj, frames=range(args.warmup, args.warmup + args.steps),
                              session=sess, frame_sink=sink, pipelined=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        assert len(got) == args.steps
        e2e_pipe = {"value": round(args.steps / dt, 3), "unit": UNIT,
                    "api": "harness.run_benchmark(pipelined=True) -> frame_sink(i, host image)",
                    "clock": "host wall (time.perf_counter), device synchronised on both sides"}
        # the whole trajectory from a cold session (frame 0 included), device
        # output, CUDA events: the mean over every frame of the path
        sess = new_session()
        sess.prepare(traj.frame_camera(0))  # workspaces: setup, not a frame
        torch.cuda.synchronize()
        e0.record(stream)
        call_ms = []
        for f in range(F):
            t1 = time.perf_counter()
            sess.render_frame(traj.frame_camera(f), f, out="device")
            call_ms.append((time.perf_counter() - t1) * 1e3)
        e1.record(stream)
        torch.cuda.synchronize()
        sess.flush()
        ms_traj = e0.elapsed_time(e1)
        slow = max(range(F), key=lambda k: call_ms[k])
        traj_fps = {"value": round(F / (ms_traj / 1e3), 3), "unit": UNIT, "frames": F,
                    "ms_per_frame": round(ms_traj / F, 4),
                    "slowest_call": {"frame": slow, "host_ms": round(call_ms[slow], 3)},
                    "what": "every frame 0..F-1 of the trajectory from a fresh session "
                            "(cold page cache at frame 0; its render workspaces allocated "
                            "before the timer), frame left in HBM"}
    # last pass over the timed frames with per-stage CUDA events (one sync
    # per frame): the stage breakdown and the rooflines come from here
    fresh_session(timing=True)
    _, stats_t = timed("device")
    pcie = measure_pcie(torch) if rank == 0 else None
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return None

    hbm, peak_kind = peaks()
    vw, vh = max(1, round(W * 0.25)), max(1, round(H * 0.25))
    for s in stats_t:
        s["vis_pixels"] = vw * vh
    blend_s = sum(s["time_blend"] for s in stats_t)
    pre_s = sum(s["time_preprocess"] for s in stats_t)
    per_frame = [frame_bytes(s, W, H, scene.page_count) for s in stats_t]
    blend_bytes = sum(b["blend"] for b, _ in per_frame)
    pre_bytes = sum(b["preprocess"] for b, _ in per_frame)
    stages = {k: 1e3 * statistics.mean(s[f"time_{k}"] for s in stats_t)
              for k in ("visibility", "update", "copy", "sort", "render", "preprocess", "tiles",
                        "blend", "device_frame")}
    dominant = "blend" if blend_s >= pre_s else "preprocess"
    ach = (blend_bytes / blend_s if dominant == "blend" else pre_bytes / pre_s) / 1e9
    # DRAM bytes per launch (and the issue-side limits) of the dominant kernel
    # from one ncu --set full capture (profiles/traffic.json, written by
    # profiles/ncu_summary.py --traffic)
    traffic, limits = None, None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            ent = json.load(open(tf)).get(dominant + "_k")
            if ent:
                traffic = int(ent["bytes_per_launch"])
                limits = {k: ent[k] for k in ("fp64_pct", "xu_pct", "ipc", "issue_frac",
                                              "sm_pct", "top_stalls", "dur_us", "frame",
                                              "source") if k in ent}
        except (ValueError, KeyError, TypeError):
            traffic = None
    up_bytes = sum(s["bytes_copied"] for s in stats_t)
    up_s = sum(s["time_copy"] for s in stats_t if s["bytes_copied"])
    up_gbs = up_bytes / up_s / 1e9 if up_s else None
    # whole-frame roofline: HBM bytes at the measured HBM peak + page bytes
    # at the measured H2D peak, per frame, against the device time per frame
    hbm_b = statistics.mean(sum(b.values()) for b, _ in per_frame)
    pcie_b = statistics.mean(p for _, p in per_frame)
    t_roof = hbm_b / (hbm * 1e9) + pcie_b / (pcie["h2d_gbs"] * 1e9)
    h2d_step = int(statistics.mean(s["bytes_copied"] for s in stats_e2e)) + 16 * int(
        statistics.mean(s.get("n_chunks", 0) for s in stats_e2e))
    d2h_step = W * H * 12 + 10 * int(statistics.mean(s["required_pages"] for s in stats_e2e))
    value = world * args.steps / (ms_dev / 1e3)
    e2e = world * args.steps / (ms_e2e / 1e3)
    launches = sum(launches_per_frame(s, len(scene.faces), holder["s"].upload_mode,
                                      scene.page_count, holder["s"].device_table,
                                      not args.fast)
                   for s in stats)
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_dev / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32",
        "data": DATA,
        "config": bench_config(args, lay, world),
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
        "trajectory": traj_fps,
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": round(ach, 2),
                     "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(ach / hbm, 4), "traffic": traffic,
                     "bytes_per_launch": round((blend_bytes if dominant == "blend" else pre_bytes)
                                               / len(stats_t)),
                     "limiter": ("not HBM: the exact blend's inputs are L2-resident (traffic "
                                 "<< algorithmic bytes); it is issue-bound (limits: ncu of the "
                                 "same kernel) and, on the vanishing-point frames, waits at "
                                 "the end-of-batch barrier for the 8x4 blocks that reach the sky "
                                 "(DESIGN section 4)")
                     if dominant == "blend" else "HBM read of the resident records",
                     "limits": limits},
        # the roofline that binds the blend: SM issue (4 warp-instructions per
        # cycle per SM), from the same ncu capture of the kernel
        "roofline_issue": ({"bound": "issue", "kernel": dominant, "achieved": limits["ipc"],
                            "peak": 4.0, "unit": "warp-instr/cycle/SM",
                            "frac": round(limits["ipc"] / 4.0, 3),
                            "fp64_pipe_frac": round(limits.get("fp64_pct", 0.0) / 100.0, 3),
                            "source": limits.get("source"), "frame": limits.get("frame")}
                           if limits and "ipc" in limits else None),
        "frame_roofline": {"hbm_bytes": int(hbm_b), "pcie_bytes": int(pcie_b),
                           "fps": round(1.0 / t_roof, 1),
                           "frac": round((args.steps / sum(s["time_device_frame"]
                                                           for s in stats_t)) * t_roof, 4),
                           "how": "SURVEY 8(d) per-stage algorithmic bytes at the measured HBM "
                                  "peak + the frame's page bytes at the measured H2D peak, vs "
                                  "the device time per frame of the stage-timing pass"},
        "pcie": pcie,
        "stages_ms": {k: round(v, 4) for k, v in stages.items()},
        "upload": {"gbs": round(up_gbs, 2) if up_gbs else None,
                   "frac_of_h2d_peak": round(up_gbs / pcie["h2d_gbs"], 4) if up_gbs else None,
                   "bytes": up_bytes,
                   "frames_with_copies": sum(1 for s in stats_t if s["bytes_copied"]),
                   "how": "reference bytes_copied / the copy stage's device time (copy stream "
                          "events), frames with copies only"},
        "mean_kept": int(statistics.mean(s["n_kept"] for s in stats_t)),
        "mean_instances": int(statistics.mean(s["n_instances"] for s in stats_t)),
        "mean_resident_records": int(statistics.mean(s["n_resident_records"] for s in stats_t)),
        "mean_required_pages": round(statistics.mean(s["required_pages"] for s in stats_t), 1),
        "host_scene": holder["s"].host.kind if hasattr(holder["s"].host, "kind") else "mmap",
        "gpu_launches": int(launches),
        "host_wall_ms": {
            name: {"median": round(1e3 * statistics.median(x["time_frame_wall"] for x in st), 4),
                   "max": round(1e3 * max(x["time_frame_wall"] for x in st), 4)}
            for name, st in (("device", stats), ("e2e", stats_e2e))},
        "clocks": clocks,
    }
    if gathered:
        out["gather"] = gathered
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

    cfg = config_of(args)
    kern = refkernels if refkernels.available() else None
    s = core.OSession(scene, buffer_pages=cfg["buffer"], staging_pages=cfg["staging"],
                      vis_scale=0.25, kern=kern)
    for f in range(warm_to):
        s.render_frame(traj.frame_camera(f % traj.frame_count), f, want_image=False)
    return s, ("reference" if kern is not None else "port")


def cpu_baseline(scene, traj, args, start_frame, frames):
    """The reference's CPU path on one core (one BLAS thread) over a bounded
    sample of the timed frames (``--cpu-frames``, ~1.3 s each at 1080p)."""
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        s, kind = reference_session(scene, traj, args, start_frame)
        t0 = time.perf_counter()
        for f in range(start_frame, start_frame + frames):
            s.render_frame(traj.frame_camera(f % traj.frame_count), f)
        dt = time.perf_counter() - t0
    return {"value": round(frames / dt, 5), "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{frames} full {args.height}p frame(s) of the {args.config.upper()} "
                      f"trajectory (frames {start_frame}..{start_frame + frames - 1}, the first "
                      f"timed frames) after stepping the page table through frame "
                      f"{start_frame - 1} without compositing; reference Cython kernels "
                      "(oracle/_ref) driven by oracle/core.py, 1 core, 1 BLAS thread",
            "cpu": cpu_model()}


def _reference_worker(job):
    """One host core's share of the reference arm: a fresh reference session
    (oracle/_ref Cython kernels driven by oracle/core.py) stepped through
    frames 0..start-1 without compositing (visibility + paging + copies only:
    compositing does not change the session state, so the state at ``start``
    is the sequential run's), then its frames [start, stop) timed in full."""
    args, start, stop = job
    from threadpoolctl import threadpool_limits

    from paper_2506_19415_b200 import scenegen
    from paper_2506_19415_b200.scene_io import read_scene

    with threadpool_limits(1):
        lay, path = ensure_scene(args, 0)
        scene = read_scene(path, mmap_gaussians=True)
        traj = trajectory(args, lay)
        s, kind = reference_session(scene, traj, args, start)
        t0 = time.perf_counter()
        for f in range(start, stop):
            s.render_frame(traj.frame_camera(f % traj.frame_count), f)
        return stop - start, time.perf_counter() - t0, kind


def reference_workers(frames: int) -> int:
    """Host cores for the reference arm (one single-threaded session each,
    never more than there are timed frames)."""
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        cores = os.cpu_count() or 1
    cap = int(os.environ.get("VMSPLAT_REF_WORKERS", "32"))
    return max(1, min(cores, cap, frames))


def run_reference(args, rank, world):
    """The reference's own CPU path on all the host cores it can use, over
    exactly the frames the GPU arm times (trajectory frames W..W+K-1, with
    the page-table state of a sequential run): the K frames are split into
    contiguous blocks, one single-threaded reference session per core; value
    = K / the slowest worker's time."""
    if rank != 0:
        return None
    import multiprocessing as mp

    from oracle import refkernels

    # load the reference's compiled core in this process too (the workers
    # are forked from it, so the library the arm runs is visible here)
    refkernels.available()
    lay, _ = ensure_scene(args, 0)  # written once, before the workers start
    K, W = args.steps, args.warmup
    P = reference_workers(K)
    bounds = [W + (w * K) // P for w in range(P + 1)]
    jobs = [(args, bounds[w], bounds[w + 1]) for w in range(P)]
    if P == 1:
        res = [_reference_worker(jobs[0])]
    else:
        with mp.get_context("fork").Pool(P) as pool:
            res = pool.map(_reference_worker, jobs)
    frames = sum(r[0] for r in res)
    assert frames == K, (frames, K)
    dt = max(r[1] for r in res)
    kind = res[0][2]
    v = frames / dt
    return {"metric": METRIC, "value": round(v, 5), "unit": UNIT, "n_gpus": 0,
            "steps": K, "warmup": W, "ms_per_step": round(1e3 * dt * P / K, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": DATA, "impl": "reference",
            "config": bench_config(args, lay),
            "timed_frames": [W, W + K - 1],
            "cpu_baseline": {"value": round(v, 5), "unit": UNIT, "cores": P, "kind": kind,
                             "sample": f"trajectory frames {W}..{W + K - 1} (the GPU arm's timed "
                                       f"frames), split over {P} worker process(es), one core, "
                                       "one BLAS thread and one reference session each; every "
                                       "worker first steps its session through the earlier "
                                       "frames without compositing; value = frames / slowest "
                                       "worker",
                             "cpu": cpu_model()},
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
