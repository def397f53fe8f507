"""Multi-process view sharding on CPU (gloo, world size 2): each rank runs a
session over its contiguous block of the trajectory and the stats rows are
gathered to rank 0; the gathered table must equal per-block single-process
runs.  The sessions here are the CPU oracle (the GPU path runs the same
sharding code in bench.py under torchrun with NCCL)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2506_19415_b200 import sharding
from tests.golden import inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    import torch.distributed as dist

    from oracle import core
    from paper_2506_19415_b200 import scenegen

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = scenegen.city_scene(inputs.CITY_SMALL)
    path = inputs.city_path(inputs.CITY_SMALL)

    class Sess:
        def __init__(self):
            self.o = core.OSession(sc, buffer_pages=16, staging_pages=6.0, vis_scale=0.5)

        def render_frame(self, cam, f, out=None):
            return self.o.render_frame(cam, f, want_image=False)

    stats = sharding.render_shard(Sess(), path, rank, world, out=None)
    rows = sharding.gather_rows(sharding.stats_rows(stats), dist)
    if rank == 0:
        np.save(result_path, rows)
    dist.barrier()
    dist.destroy_process_group()


def test_frame_blocks_cover_trajectory():
    for world in (1, 2, 3, 4, 8):
        blocks = [sharding.frame_block(r, world, 121) for r in range(world)]
        assert blocks[0][0] == 0 and blocks[-1][1] == 121
        assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
    with pytest.raises(ValueError):
        sharding.frame_block(2, 2, 10)


def test_gloo_two_rank_sharded_stats_gather(tmp_path):
    from oracle import core
    from paper_2506_19415_b200 import scenegen

    world = 2
    out = tmp_path / "rows.npy"
    mp.start_processes(_worker, args=(world, _free_port(), str(out)), nprocs=world,
                       join=True, start_method="spawn")
    rows = np.load(out)
    # reference: each block rendered by its own fresh single-process session
    sc = scenegen.city_scene(inputs.CITY_SMALL)
    path = inputs.city_path(inputs.CITY_SMALL)
    expect = []
    for r in range(world):
        a, b = sharding.frame_block(r, world, path.frame_count)
        o = core.OSession(sc, buffer_pages=16, staging_pages=6.0, vis_scale=0.5)
        for f in range(a, b):
            expect.append(o.render_frame(path.frame_camera(f), f, want_image=False)[1])
    assert np.array_equal(rows, sharding.stats_rows(expect))
    assert rows[:, 0].tolist() == list(range(path.frame_count))
