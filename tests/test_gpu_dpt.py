"""the device-resident page table (csrc/dpt.cu) against the
host C++ table (itself pinned to the reference, tests/test_abi_cpu.py) and
the reference's golden traces: plans, missing counts, residency, per-entry
levels / slots / LRU stamps, frame by frame."""

import numpy as np
import pytest

from paper_2506_19415_b200.runtime import (DevicePageTable, LodController, PageTable,
                                           RequiredList, encode_depth, initial_thresholds,
                                           update_page_table)
from tests.golden import inputs

pytestmark = pytest.mark.gpu


def _levels(spec):
    return len(spec["thresholds"]) + 1


def _same_state(a, b):
    ea, eb = a.entries, b.entries
    for i, (x, y) in enumerate(zip(ea, eb)):
        assert (x.lod_level, x.last_used_frame, x.slots) == \
            (y.lod_level, y.last_used_frame, y.slots), i
    assert a.resident == b.resident


def test_device_table_matches_reference_traces(cuda, golden):
    g = golden["pagetable"]
    for trace in range(40):
        spec = inputs.table_trace(trace)
        pages = len(spec["frames"][0][0]) - 1
        table = DevicePageTable(spec["capacity"], pages, _levels(spec))
        ctl = LodController(spec["thresholds"])
        plans, missing, res = [], [], []
        for f, (depths, direct) in enumerate(spec["frames"]):
            plan, miss = update_page_table(table, RequiredList(depths, direct), ctl, f,
                                           spec["budget"])
            plans.extend((p.page_id, p.level, p.entry, p.slot) for p in plan)
            missing.append(miss)
            res.extend(sorted((k, v[0], v[1]) for k, v in table.resident.items()))
        table.check()
        assert np.array_equal(np.array(plans, np.int64).reshape(-1, 4), g[f"t{trace}_plan"]), trace
        assert np.array_equal(missing, g[f"t{trace}_missing"]), trace
        assert np.array_equal(np.array(res, np.int64).reshape(-1, 3), g[f"t{trace}_res"]), trace


def test_device_table_matches_host_table_on_random_traces(cuda):
    for trace in range(40, 240):
        spec = inputs.table_trace(trace)
        pages = len(spec["frames"][0][0]) - 1
        a = DevicePageTable(spec["capacity"], pages, _levels(spec))
        b = PageTable(spec["capacity"])
        ca, cb = LodController(spec["thresholds"]), LodController(spec["thresholds"])
        for f, (depths, direct) in enumerate(spec["frames"]):
            pa, ma = update_page_table(a, RequiredList(depths, direct), ca, f, spec["budget"])
            pb, mb = update_page_table(b, RequiredList(depths, direct), cb, f, spec["budget"])
            assert pa == pb and ma == mb, (trace, f)
        _same_state(a, b)


def test_device_table_large_tables_and_global_sort(cuda):
    """Capacities up to the 8192-entry limit, 20000 pages (more than 8192
    required pages: the sort spills to global memory), 4 levels."""
    rng = np.random.default_rng(7)
    for capacity, pages, levels, budget in ((8192, 20000, 4, 160.0), (3000, 12000, 3, 40.0),
                                            (64, 20000, 2, np.inf)):
        thr = np.sort(rng.uniform(1.0, 60.0, size=levels - 1))
        a = DevicePageTable(capacity, pages, levels)
        b = PageTable(capacity)
        ca, cb = LodController(thr), LodController(thr)
        for f in range(12):
            depths = np.zeros(pages + 1, np.uint32)
            direct = np.zeros(pages + 1, bool)
            k = int(rng.integers(0, pages + 1))
            ids = rng.choice(np.arange(1, pages + 1), size=k, replace=False)
            d = rng.uniform(0.5, 80.0, size=k).astype(np.float32)
            d[rng.random(k) < 0.1] = np.float32(7.5)
            depths[ids] = np.uint32(0xFFFFFFFF) - d.view(np.uint32)
            direct[ids] = rng.random(k) < 0.7
            pa, ma = update_page_table(a, RequiredList(depths, direct), ca, f, budget)
            pb, mb = update_page_table(b, RequiredList(depths, direct), cb, f, budget)
            assert pa == pb and ma == mb, (capacity, f)
        _same_state(a, b)
        a.check()


def _required(n, entries):
    depths = np.zeros(n + 1, dtype=np.uint32)
    direct = np.zeros(n + 1, dtype=bool)
    for pid, (d, dr) in entries.items():
        depths[pid] = encode_depth(d)
        direct[pid] = dr
    return RequiredList(depths=depths, direct=direct)


def _both(capacity, levels, steps):
    """Run (required entries, frame, budget) steps on both tables; compare."""
    ctl_a = LodController(initial_thresholds(100.0, levels) if levels > 1 else np.zeros(0))
    ctl_b = LodController(ctl_a.thresholds.copy())
    a, b = DevicePageTable(capacity, 9, levels), PageTable(capacity)
    for entries, f, budget in steps:
        ra, ma = update_page_table(a, _required(9, entries), ctl_a, f, budget)
        rb, mb = update_page_table(b, _required(9, entries), ctl_b, f, budget)
        assert ra == rb and ma == mb, (entries, f)
    _same_state(a, b)
    a.check()
    assert a.occupied_entries() == b.occupied_entries()
    assert a.resident_counts(levels) == b.resident_counts(levels)
    return a


def test_device_table_reference_unit_cases(cuda):
    # the reference's unit cases (pkg/tests/test_runtime.py:147-257; the
    # host-table versions are in tests/test_abi_cpu.py)
    _both(8, 1, [({p: (float(p), True) for p in range(1, 7)}, 0, 3)])   # budget breaks
    _both(8, 1, [({2: (5.0, False), 3: (1.0, True)}, 0, 10)])           # direct first
    _both(8, 1, [({4: (2.0, True), 2: (2.0, True), 7: (1.0, True)}, 0, 10)])  # ties
    a = _both(2, 1, [({1: (1.0, True)}, 0, 10), ({2: (1.0, True)}, 1, 10),
                     ({2: (1.0, True), 3: (1.0, True)}, 2, 10)])         # LRU
    assert set(a.resident) == {2, 3}
    _both(2, 1, [({1: (1.0, True), 2: (2.0, True)}, 0, 10),
                 ({1: (1.0, True), 2: (2.0, True), 3: (0.5, True)}, 1, 10)])  # protection
    _both(2, 4, [({p: (60.0, True) for p in (1, 2, 3, 4)}, 0, 10)])     # same-level packing
    a = _both(4, 4, [({1: (60.0, True)}, 0, 10), ({1: (1.0, True)}, 1, 10)])  # transition
    assert a.resident_counts(4) == (1, 0, 0, 0)


# -- the device table inside a session ----------------------------------------------

STAT_KEYS = ("required_pages", "resident_pages", "resident_per_level", "planned_copies",
             "missing_pages", "bytes_copied", "usage", "lod_step", "thresholds")


@pytest.fixture(scope="module")
def c2_scene(tmp_path_factory):
    from paper_2506_19415_b200 import scenegen
    from paper_2506_19415_b200.scene_io import read_scene

    p = tmp_path_factory.mktemp("c2dpt") / "c2.vms"
    scenegen.write_city(p, scenegen.C2)
    return read_scene(p, mmap_gaussians=True)


def test_session_device_table_matches_host_table_c2(cuda, c2_scene):
    """C2 (1000 pages, 3 LOD levels, buffer 500, staging 40) over all 120
    frames: a session whose page table runs on the device gives the host-table
    session's stats on every frame, the same residency, and identical images
    (the host table is pinned to the oracle, tests/test_gpu_parity.py)."""
    from paper_2506_19415_b200 import scenegen
    from paper_2506_19415_b200.runtime import VmSession

    traj = scenegen.street_path(scenegen.C2, frames=120)
    d = VmSession(c2_scene, device_table=True)
    h = VmSession(c2_scene)
    for f in range(traj.frame_count):
        cam = traj.frame_camera(f)
        a, sa = d.render_frame(cam, f)
        b, sb = h.render_frame(cam, f)
        for k in STAT_KEYS:
            assert sa[k] == sb[k], (f, k)
        assert np.array_equal(a, b), f
        if f % 10 == 0:
            assert d.table.resident == h.table.resident, f
    d.table.check()
    ea, eb = d.table.entries, h.table.entries
    assert [(e.lod_level, e.last_used_frame, e.slots) for e in ea] == \
        [(e.lod_level, e.last_used_frame, e.slots) for e in eb]


def test_session_device_table_pipelined(cuda):
    """Two frames in flight (the bench's asynchronous device output): every
    frame rendered into its own device tensor, compared after a flush."""
    import torch

    from paper_2506_19415_b200.runtime import VmSession

    from paper_2506_19415_b200 import scenegen

    sc = scenegen.city_scene(inputs.CITY_SMALL)
    path = inputs.city_path(inputs.CITY_SMALL)
    d = VmSession(sc, buffer_pages=16, staging_pages=6.0, vis_scale=0.5, device_table=True)
    h = VmSession(sc, buffer_pages=16, staging_pages=6.0, vis_scale=0.5)
    cam0 = path.frame_camera(0)
    outs = [torch.empty((cam0.height, cam0.width, 3), dtype=torch.float32, device="cuda")
            for _ in range(path.frame_count)]
    stats = []
    for f in range(path.frame_count):
        _, st = d.render_frame(path.frame_camera(f), f, out=outs[f])
        stats.append(st)
    d.flush()
    for f in range(path.frame_count):
        ref, st = h.render_frame(path.frame_camera(f), f)
        for k in STAT_KEYS:
            assert stats[f][k] == st[k], (f, k)
        assert np.array_equal(outs[f].cpu().numpy(), ref), f
