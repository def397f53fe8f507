"""C-ABI library checks that need no GPU: the .so loads, exports every
symbol include/vmsplat_b200.h declares, and its host C++ page table
reproduces the reference's update_page_table on the golden traces."""

import os
import re

import numpy as np
import pytest

from paper_2506_19415_b200 import _lib
from paper_2506_19415_b200.errors import InvariantViolation
from paper_2506_19415_b200.runtime import (LodController, PageTable, RequiredList,
                                           encode_depth, initial_thresholds,
                                           update_page_table)
from tests.golden import inputs

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "vmsplat_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(vms_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} missing from the ctypes binding"
    assert set(_lib.SIGNATURES) == set(names)
    assert lib.vms_abi_version() == 1


def test_invalid_arguments_report_errors():
    lib = _lib.load()
    assert lib.vms_pt_create(0) is None
    assert b"at least one entry" in lib.vms_last_error()
    st = lib.vms_radix_sort_pairs(None, None, -1, None, 0, None)
    assert st == _lib.VMS_ERR_INVALID
    with pytest.raises(ValueError):
        _lib.check(st, "radix")


def test_cpp_page_table_matches_reference_traces(golden):
    g = golden["pagetable"]
    for trace in range(40):
        spec = inputs.table_trace(trace)
        table = PageTable(spec["capacity"])
        ctl = LodController(spec["thresholds"])
        plans, missing, res = [], [], []
        for f, (depths, direct) in enumerate(spec["frames"]):
            plan, miss = update_page_table(table, RequiredList(depths, direct), ctl, f,
                                           spec["budget"])
            table.check()
            plans.extend((p.page_id, p.level, p.entry, p.slot) for p in plan)
            missing.append(miss)
            res.extend(sorted((k, v[0], v[1]) for k, v in table.resident.items()))
        assert np.array_equal(np.array(plans, np.int64).reshape(-1, 4), g[f"t{trace}_plan"])
        assert np.array_equal(missing, g[f"t{trace}_missing"])
        assert np.array_equal(np.array(res, np.int64).reshape(-1, 3), g[f"t{trace}_res"])


def test_cpp_page_table_matches_oracle_on_long_random_traces():
    """Beyond the golden traces: 300 more random traces against the pinned
    oracle restatement, including per-entry level/slots/LRU stamps."""
    from oracle import core

    for trace in range(40, 340):
        spec = inputs.table_trace(trace)
        a = PageTable(spec["capacity"])
        b = core.OTable(spec["capacity"])
        ca = LodController(spec["thresholds"])
        cb = core.OController(spec["thresholds"])
        for f, (depths, direct) in enumerate(spec["frames"]):
            pa, ma = update_page_table(a, RequiredList(depths, direct), ca, f, spec["budget"])
            pb, mb = core.update_table(b, core.ORequired(depths, direct), cb, f, spec["budget"])
            assert [(p.page_id, p.level, p.entry, p.slot) for p in pa] == pb
            assert ma == mb
            a.check()
        ea = a.entries
        for x, y in zip(ea, b.entries):
            assert (x.lod_level, x.last_used_frame, x.slots) == (y.level, y.last, y.slots)


# -- reference unit cases (pkg/tests/test_runtime.py:147-257) -----------------
def _required(n, entries):
    depths = np.zeros(n + 1, dtype=np.uint32)
    direct = np.zeros(n + 1, dtype=bool)
    for pid, (d, dr) in entries.items():
        depths[pid] = encode_depth(d)
        direct[pid] = dr
    return RequiredList(depths=depths, direct=direct)


def _controller(levels=1):
    if levels == 1:
        return LodController(np.zeros(0))
    return LodController(initial_thresholds(100.0, levels))


def test_budget_breaks_not_skips():
    table = PageTable(8)
    req = _required(8, {p: (float(p), True) for p in range(1, 7)})
    plan, missing = update_page_table(table, req, _controller(), 0, 3)
    assert [p.page_id for p in plan] == [1, 2, 3]
    assert missing == 3


def test_direct_before_linked_and_ties_to_lower_id():
    table = PageTable(8)
    plan, _ = update_page_table(table, _required(8, {2: (5.0, False), 3: (1.0, True)}),
                                _controller(), 0, 10)
    assert [p.page_id for p in plan] == [3, 2]
    table = PageTable(8)
    plan, _ = update_page_table(
        table, _required(8, {4: (2.0, True), 2: (2.0, True), 7: (1.0, True)}), _controller(),
        0, 10)
    assert [p.page_id for p in plan] == [7, 2, 4]


def test_lru_and_protection():
    table = PageTable(2)
    ctl = _controller()
    update_page_table(table, _required(9, {1: (1.0, True)}), ctl, 0, 10)
    update_page_table(table, _required(9, {2: (1.0, True)}), ctl, 1, 10)
    update_page_table(table, _required(9, {2: (1.0, True), 3: (1.0, True)}), ctl, 2, 10)
    assert set(table.resident) == {2, 3}
    table = PageTable(2)
    update_page_table(table, _required(9, {1: (1.0, True), 2: (2.0, True)}), ctl, 0, 10)
    _, missing = update_page_table(
        table, _required(9, {1: (1.0, True), 2: (2.0, True), 3: (0.5, True)}), ctl, 1, 10)
    assert set(table.resident) == {1, 2} and missing == 1
    table.check()


def test_same_level_packing_and_transition():
    table = PageTable(2)
    ctl = _controller(levels=4)
    plan, missing = update_page_table(
        table, _required(9, {p: (60.0, True) for p in (1, 2, 3, 4)}), ctl, 0, 10)
    assert missing == 0 and len({p.entry for p in plan}) == 1
    assert table.occupied_entries() == 1 and table.usage_ratio() == pytest.approx(0.5)
    table = PageTable(4)
    update_page_table(table, _required(9, {1: (60.0, True)}), ctl, 0, 10)
    assert table.resident_level(1) == 2
    plan, _ = update_page_table(table, _required(9, {1: (1.0, True)}), ctl, 1, 10)
    assert [(p.page_id, p.level) for p in plan] == [(1, 0)]
    assert table.resident_counts(4) == (1, 0, 0, 0)
    table.check()


def test_table_capacity_validated():
    with pytest.raises(InvariantViolation):
        PageTable(0)


def test_frame_camera_fill_matches_struct():
    """The per-frame fast camera fill equals Camera.struct() and
    Camera.scaled(s).struct() field for field (bit-exact doubles)."""
    import numpy as np

    from paper_2506_19415_b200 import _lib, scenegen
    from paper_2506_19415_b200.runtime import fill_frame_cameras

    traj = scenegen.street_path(scenegen.C2, frames=120)
    fields = ("focal", "half_w", "half_h", "near", "width", "height", "dot_mode")
    for f in range(0, 120, 7):
        cam = traj.frame_camera(f)
        for scale in (0.25, 0.5, 1.0 / 3.0):
            a = _lib.FrameArgs()
            fill_frame_cameras(a, cam, scale, 1)
            for got, ref in ((a.cam, cam.struct(1)), (a.vis_cam, cam.scaled(scale).struct(1))):
                assert np.array_equal(np.array(got.pos[:]), np.array(ref.pos[:]))
                assert np.array(got.rot[:]).tobytes() == np.array(ref.rot[:]).tobytes()
                for k in fields:
                    assert getattr(got, k) == getattr(ref, k), (f, scale, k)
