"""Nearest-face query throughput: the sm_100a kernel behind
kernels.bvh_nearest_points vs the reference's Cython core
(oracle/_ref/_core.bvh_nearest_points, one core) on the same BVH.

Workload: the C2 bench city's proxy mesh scaled up (--faces random facade
triangles) queried at --points record-like positions - the link-sampling
call (paging.py:336).  Device time by CUDA events with inputs resident;
the CPU arm times a bounded sample and reports queries/s."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--faces", type=int, default=200_000)
    p.add_argument("--points", type=int, default=2_000_000)
    p.add_argument("--cpu-points", type=int, default=20_000)
    a = p.parse_args()
    import numpy as np
    import torch

    from oracle import refkernels
    from paper_2506_19415_b200 import _device, _lib
    from paper_2506_19415_b200.geometry import FaceBvh

    rng = np.random.default_rng(0)
    tv = rng.uniform(-200, 200, (a.faces, 1, 3)) + rng.normal(0, 1.5, (a.faces, 3, 3))
    pts = rng.uniform(-220, 220, (a.points, 3))
    t0 = time.perf_counter()
    bvh = FaceBvh(tv)
    build_s = time.perf_counter() - t0
    dev = torch.device("cuda")
    P = torch.from_numpy(pts).to(dev)
    B = torch.from_numpy(bvh.bounds).to(dev)
    C = torch.from_numpy(bvh.children).to(dev)
    R = torch.from_numpy(bvh.ranges).to(dev)
    O = torch.from_numpy(bvh.order).to(dev)
    T = torch.from_numpy(bvh.tri_verts).to(dev)
    face = torch.empty(a.points, dtype=torch.int64, device=dev)
    dist = torch.empty(a.points, dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.load()

    def run():
        _lib.check(lib.vms_bvh_nearest_points(P.data_ptr(), a.points, B.data_ptr(), C.data_ptr(),
                                              R.data_ptr(), len(B), O.data_ptr(), T.data_ptr(),
                                              len(T), face.data_ptr(), dist.data_ptr(),
                                              flag.data_ptr(), _device.sptr()), "bvh")

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    gpu_qps = 10 * a.points / (e0.elapsed_time(e1) * 1e-3)
    f_gpu = face.cpu().numpy()
    d_gpu = dist.cpu().numpy()
    line = {"faces": a.faces, "points": a.points, "bvh_nodes": len(bvh.bounds),
            "host_build_s": round(build_s, 3), "gpu_queries_per_s": round(gpu_qps, 1)}
    if refkernels.available():
        core = refkernels._load()
        n = a.cpu_points
        t0 = time.perf_counter()
        f_ref, d_ref = core.bvh_nearest_points(pts[:n], bvh.bounds, bvh.children, bvh.ranges,
                                               bvh.order, bvh.tri_verts)
        cpu_s = time.perf_counter() - t0
        line["cpu_reference_queries_per_s"] = round(n / cpu_s, 1)
        line["cpu_sample"] = n
        line["bit_exact_on_sample"] = bool(np.array_equal(f_ref, f_gpu[:n]) and
                                           np.array_equal(d_ref.view(np.uint64),
                                                          d_gpu[:n].view(np.uint64)))
        line["speedup"] = round(gpu_qps / (n / cpu_s), 1)
    print(line)


if __name__ == "__main__":
    main()
