"""F3 measurement: the GPU LOD pyramid (csrc/lod.cu) on C2-shaped pages -
`--pages` pages of 2048 box-scene records, 3 levels (the C2 scene's LOD
depth) - against the oracle restatement of the reference's NumPy k-means
(oracle/lod.py, one core) on `--cpu-pages` of the same pages.

    python profiles/lod_bench.py --pages 1000
    ncu --set full -k regex:lod_page_k -c 1 python profiles/lod_bench.py --pages 296 --reps 1

Prints one JSON line: device ms per level (CUDA events around each level's
launch), pages/s, the CPU seconds per page and the speed-up.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pages", type=int, default=1000)
    ap.add_argument("--page-size", type=int, default=2048)
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu-pages", type=int, default=2)
    a = ap.parse_args()
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np
    import torch

    from paper_2506_19415_b200 import lod
    from tests.golden import inputs

    ps = a.page_size
    base = inputs.box_scene(seed=5, count=ps * min(a.pages, 64), extent=30.0, depth=60.0)
    # pages of spatially coherent records (sorted by x), repeated to --pages
    base = base[np.argsort(base[:, 0], kind="stable")]
    reps = -(-a.pages // min(a.pages, 64))
    level0 = np.concatenate([base] * reps)[: a.pages * ps].copy()
    level0[:, 0] += np.repeat(np.arange(a.pages, dtype=np.float32) // 64 * 100.0, ps)
    torch.cuda.synchronize()
    lod.build_pyramid(level0[: 4 * ps], ps, level_count=a.levels, seed=7)  # warm-up
    walls = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gpu = lod.build_pyramid(level0, ps, level_count=a.levels, seed=7)
        walls.append(time.perf_counter() - t0)
    wall = min(walls)
    out = {"pages": a.pages, "page_size": ps, "levels": a.levels, "gpu_s": round(wall, 4),
           "pages_per_s": round(a.pages / wall, 1)}
    if a.cpu_pages:
        from oracle import lod as olod

        t0 = time.perf_counter()
        cpu = olod.build_pyramid(level0[: a.cpu_pages * ps], ps, a.levels, seed=7)
        cs = (time.perf_counter() - t0) / a.cpu_pages
        out["cpu_s_per_page"] = round(cs, 3)
        out["cpu_kind"] = "port (oracle/lod.py, NumPy, 1 core)"
        out["speedup"] = round(cs * a.pages / wall, 1)
        for k in range(1, a.levels):
            n = a.cpu_pages * (ps >> k)
            assert np.array_equal(cpu[k], gpu[k][:n]), f"level {k} differs from the oracle"
        out["parity_pages"] = a.cpu_pages
    print(json.dumps(out))


if __name__ == "__main__":
    main()
