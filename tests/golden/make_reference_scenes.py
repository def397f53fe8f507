"""Build the reference test suite's scene bundles with the LIVE reference
preprocessing pipeline and store them as .vms fixtures for
tests/test_reference_suite.py.

Run in the build container only (needs /root/reference):

    cp -r /root/reference/pkg /tmp/refbuild
    (cd /tmp/refbuild && python setup.py build_ext --inplace)
    PYTHONPATH=/tmp/refbuild/src OPENBLAS_NUM_THREADS=1 python tests/golden/make_reference_scenes.py

The bundles and their preprocessing arguments are those of the reference's
pkg/tests/conftest.py:37-54,78-94 (occluder, small), pkg/tests/test_cli.py:15-36
(the CLI chain's full.vms) and pkg/tests/test_acceptance.py:296-327
(criterion 10's scene).  The files are stored gzip-compressed.  The offline
pipeline (meshing, paging, k-means LOD) is outside the B200 hot path, so its
outputs are fixtures here, exactly as the reference's own tests consume them.
"""

from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))

from vmsplat import synthetic  # noqa: E402  (the reference)
from vmsplat.pipeline import preprocess  # noqa: E402
from vmsplat.scene_io import write_scene  # noqa: E402

OUT = os.path.join(HERE, "ref_scenes")


def main():
    os.makedirs(OUT, exist_ok=True)
    layouts = {}
    # conftest.py:37-54
    records, layout = synthetic.occluder_scene(seed=1)
    sc = preprocess(records, page_size=448, grid=96, close_radius=1, open_radius=1,
                    target_faces=700, level_count=1)
    write_scene(sc, os.path.join(OUT, "occluder.vms"))
    layouts["occluder"] = {k: float(v) if isinstance(v, (int, float)) else v
                           for k, v in layout.items()}
    # conftest.py:78-94
    records = synthetic.wall_scene(seed=5, count=5000, extent=6.0, z=8.0)
    sc = preprocess(records, page_size=128, grid=48, close_radius=1, open_radius=1,
                    target_faces=300, level_count=3, kmeans_iters=10)
    write_scene(sc, os.path.join(OUT, "small.vms"))
    # test_cli.py:15-36 ("full.vms" through the reference's own verb chain)

    sys.path.insert(0, "/root/reference/pkg/tests")
    from helpers import write_ply  # the reference's test helper
    from vmsplat.cli import main as cli_main

    tmp = tempfile.mkdtemp()
    write_ply(os.path.join(tmp, "input.ply"), synthetic.wall_scene(seed=3, count=400,
                                                                   extent=3.0, z=4.0))
    for argv in (["convert", f"{tmp}/input.ply", f"{tmp}/raw.vms"],
                 ["mesh", "--grid", "32", "--close", "1", "--open", "1", "--target-faces",
                  "200", f"{tmp}/raw.vms", f"{tmp}/meshed.vms"],
                 ["page", "--page-size", "64", "--seed", "0", f"{tmp}/meshed.vms",
                  f"{tmp}/paged.vms"],
                 ["lod", "--levels", "2", "--kmeans-iters", "5", "--seed", "0",
                  f"{tmp}/paged.vms", f"{tmp}/full.vms"]):
        assert cli_main(argv) == 0, argv[0]
    shutil.copy(f"{tmp}/full.vms", os.path.join(OUT, "cli_full.vms"))
    shutil.rmtree(tmp)
    # test_acceptance.py:303-307 (criterion 10)
    records = synthetic.wall_scene(seed=21, count=3000, extent=5.0, z=7.0)
    sc = preprocess(records, page_size=128, grid=48, close_radius=1, open_radius=1,
                    target_faces=250, level_count=3, kmeans_iters=10)
    write_scene(sc, os.path.join(OUT, "determinism.vms"))
    # the reference's own stats.csv for criterion 10's 100-frame bench
    import math

    from vmsplat.camera_path import CameraPath, Checkpoint
    from vmsplat.harness import BenchConfig, emit_reports, run_benchmark

    ident = (1.0, 0.0, 0.0, 0.0)
    path = CameraPath(checkpoints=(Checkpoint(position=(0, 0, -2.0), orientation=ident),
                                   Checkpoint(position=(0, 0, -12.0), orientation=ident)),
                      speed=1.0, fps=9.9, fov_deg=90.0, width=96, height=96)
    stats = run_benchmark(sc, path, BenchConfig(buffer_pages=20, staging_pages=20.0,
                                                frame_limit=100))
    rep = tempfile.mkdtemp()
    emit_reports(stats, rep)
    shutil.copy(os.path.join(rep, "stats.csv"), os.path.join(OUT, "determinism_stats.csv"))
    shutil.rmtree(rep)
    assert not math.isnan(stats[0].usage)
    with open(os.path.join(OUT, "layouts.json"), "w") as fh:
        json.dump(layouts, fh, indent=1, sort_keys=True, default=str)
    import gzip

    for name in os.listdir(OUT):
        if name.endswith(".vms"):
            src = os.path.join(OUT, name)
            with open(src, "rb") as fi, gzip.open(src + ".gz", "wb", compresslevel=9) as fo:
                fo.write(fi.read())
            os.unlink(src)


if __name__ == "__main__":
    main()
