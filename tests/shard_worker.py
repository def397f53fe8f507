"""One rank of tests/test_gpu_scale.py::test_sharded_sessions_match_per_shard_oracle.

argv: scene path, output dir, rank, world.  Each rank maps the same .vms
file, runs harness.run_sharded (its own VmSession over its block of the
path, gloo for the final stats gather) and rank 0 checks the gathered
stats.csv against one oracle session per block; every rank
also checks that its session streamed from the shared, registered mapping.
"""

import csv
import io
import os
import sys

import numpy as np


def main():
    path, out_dir, rank, world = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    import torch
    import torch.distributed as dist

    from oracle import core
    from paper_2506_19415_b200 import harness, scenegen
    from paper_2506_19415_b200.runtime import HostScene
    from paper_2506_19415_b200.scene_io import read_scene
    from paper_2506_19415_b200.sharding import frame_block

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene = read_scene(path, mmap_gaussians=True)
    lay = scenegen.CityLayout(n_pages=200, page_size=512, levels=3, seed=2, scale=0.1)
    traj = scenegen.street_path(lay, frames=24, width=320, height=180)
    cfg = harness.BenchConfig(buffer_pages=40, staging_pages=8.0, vis_scale=0.5)
    assert HostScene.of(scene).kind == "registered-tmpfs-mapping", HostScene.of(scene).kind
    got = harness.run_sharded(scene, traj, cfg, dist=dist)
    if rank == 0:
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        for r in harness.stats_table(got):
            w.writerow(r)
        ref = []
        for r in range(world):
            a, b = frame_block(r, world, traj.frame_count)
            o = core.OSession(scene, buffer_pages=40, staging_pages=8.0, vis_scale=0.5)
            for f in range(a, b):
                ref.append(o.render_frame(traj.frame_camera(f), f, want_image=False)[1])
        assert buf.getvalue() == core.stats_csv(ref), (buf.getvalue(), core.stats_csv(ref))
        assert [f.frame for f in got] == list(range(traj.frame_count))
        assert sum(f.bytes_copied for f in got) > 0
        np.save(os.path.join(out_dir, "rows.npy"), np.array([f.required for f in got]))
    dist.barrier()
    dist.destroy_process_group()
    print(f"shard ok rank {rank}")


if __name__ == "__main__":
    main()
