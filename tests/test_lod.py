"""the weighted k-means LOD pyramid (pkg/src/vmsplat/lod.py).

CPU tests pin the oracle restatement (oracle/lod.py) - its Philox stream,
``choice`` and reduction orders against NumPy itself, and its outputs against
the live reference's goldens (tests/golden/lod.npz, make_lod_golden.py).
GPU tests check ``paper_2506_19415_b200.lod`` (kernel csrc/lod.cu) bit for
bit against the goldens and the oracle, and run the reference's own
test_lod.py cases through the ``vmsplat.lod`` import name.
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import lod as olod
from tests import refsuite
from tests.golden import inputs

refsuite.install()

from vmsplat import lod  # noqa: E402  (this package, via the reference's name)
from vmsplat.errors import InvariantViolation  # noqa: E402
from vmsplat.gaussians import RECORD_SIZE, is_padding, padding_records  # noqa: E402

gpu = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "lod.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def _cluster_cases():
    walls = inputs.wall_scene(seed=6, count=120, extent=2.0, z=0.0)
    blobs = np.concatenate([inputs.wall_scene(seed=1, count=30, extent=0.5, z=0.0),
                            inputs.wall_scene(seed=2, count=30, extent=0.5, z=50.0)])
    dups = np.repeat(inputs.wall_scene(seed=9, count=40, extent=1.0, z=0.0), 3, axis=0)
    return [("w16", walls, 16, 3, 50), ("w10", walls, 10, 3, 50), ("blobs", blobs, 2, 1, 50),
            ("dups", dups, 70, 5, 50), ("w60i3", walls, 60, 8, 3)]


def _merge_cases():
    rec = inputs.wall_scene(seed=7, count=1, extent=1.0, z=0.0)[0]
    flipped = rec.copy()
    flipped[3:7] *= -1.0
    return {"six": inputs.wall_scene(seed=7, count=6, extent=1.0, z=0.0),
            "hemi": np.stack([rec, flipped]), "one": rec[None],
            "many": inputs.box_scene(seed=4, count=300, extent=2.0, depth=5.0)}


# -- the oracle, pinned (CPU) -------------------------------------------------

def test_philox_and_choice_restate_numpy():
    for seed, pid in ((7, 1), (0, 0), (123456789, 2**40 + 3)):
        g = np.random.Generator(np.random.Philox(key=[seed, 1], counter=[pid, 0, 0, 0]))
        p = olod.Philox.page(seed, pid)
        rng = np.random.default_rng(seed % 1000)
        for _ in range(60):
            m = int(rng.integers(1, 5000))
            assert int(g.integers(m)) == p.integers(m)
            w = rng.random(m) ** 3
            w[rng.random(m) < 0.2] = 0.0
            w[0] += 1e-3
            assert int(g.choice(m, p=w / olod.pairwise_sum(w))) == p.choice(w / olod.pairwise_sum(w))
            assert g.random() == p.random()


def test_reduction_orders_restate_numpy():
    rng = np.random.default_rng(0)
    for n in (1, 7, 8, 13, 14, 100, 128, 129, 1000, 2047, 2048, 4096):
        x = rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3, n)
        assert olod.pairwise_sum(x) == x.sum()
        x2 = rng.standard_normal((max(n // 14, 1), 59))
        assert np.array_equal(olod.colmean(x2[:, 11:]), x2[:, 11:].mean(axis=0))
        assert olod.pairwise_sum(x2[:, 10]) / len(x2) == x2[:, 10].mean()
    d = rng.standard_normal((50, 30, 14)) * 10.0 ** rng.uniform(-2, 2, (50, 30, 14))
    assert np.array_equal(olod.row_dist14(d), (d ** 2).sum(axis=2))
    for _ in range(2000):
        q = rng.standard_normal(4)
        assert olod.fdot4(q, q) == np.dot(q, q)


def test_oracle_matches_reference_goldens(gold):
    for name, recs, k, seed, iters in _cluster_cases():
        p = olod.Philox.page(seed, 0)
        a = olod.cluster_page(recs, k, max_iters=iters, rng=p)
        assert np.array_equal(a, gold[f"cluster_{name}"]), name
    for name, m in _merge_cases().items():
        assert np.array_equal(olod.merge_cluster(m), gold[f"merge_{name}"]), name
    for name, counts, ps, levels, iters, seed, dup in inputs.LOD_PYRAMIDS:
        lv = olod.build_pyramid(inputs.padded_pages(counts, ps, dup=dup), ps, levels,
                                max_iters=iters, seed=seed)
        for k in range(1, levels):
            assert np.array_equal(lv[k], gold[f"pyr_{name}_{k}"]), (name, k)


def test_weights_must_not_be_negative():
    # pkg/tests/test_lod.py:123-126
    lod.AttributeWeights(opacity=0.0).validate()
    with pytest.raises(InvariantViolation):
        lod.AttributeWeights(position=-1.0).validate()


def test_pyramid_rejects_bad_level_count():
    # pkg/tests/test_lod.py:116-120
    level0 = _padded_page(inputs.wall_scene(seed=12, count=8, extent=2.0, z=0.0), 16)
    with pytest.raises(InvariantViolation):
        lod.build_pyramid(level0, 16, level_count=0)


def _padded_page(records, page_size):
    return np.concatenate([records, padding_records(page_size - len(records))])


# -- the GPU kernel -------------------------------------------------------------

@gpu
def test_cluster_page_matches_reference(cuda, gold):
    for name, recs, k, seed, iters in _cluster_cases():
        g = lod._page_rng(seed, 0)
        a = lod.cluster_page(recs, k, max_iters=iters, rng=g)
        assert a.dtype == np.int64
        assert np.array_equal(a, gold[f"cluster_{name}"]), name
        # the caller's Generator continues where the reference's would
        assert np.array_equal(g.integers(0, 2**62, size=3), gold[f"cluster_{name}_next"]), name


@gpu
def test_merge_cluster_matches_reference(cuda, gold):
    for name, m in _merge_cases().items():
        assert np.array_equal(lod.merge_cluster(m), gold[f"merge_{name}"]), name


@gpu
def test_build_pyramid_matches_reference(cuda, gold):
    for name, counts, ps, levels, iters, seed, dup in inputs.LOD_PYRAMIDS:
        level0 = inputs.padded_pages(counts, ps, dup=dup)
        lv = lod.build_pyramid(level0, ps, level_count=levels, max_iters=iters, seed=seed)
        assert lv[0] is level0 or np.array_equal(lv[0], level0)
        for k in range(1, levels):
            assert np.array_equal(lv[k], gold[f"pyr_{name}_{k}"]), (name, k)
    # the C2-size page: 2048 records, k = 1024 (digest of the reference output)
    name, counts, ps, levels, iters, seed, dup = inputs.LOD_BIG
    lv = lod.build_pyramid(inputs.padded_pages(counts, ps, dup=dup), ps, level_count=levels,
                           max_iters=iters, seed=seed)
    for k in range(1, levels):
        got = hashlib.sha256(np.ascontiguousarray(lv[k]).tobytes()).digest()
        assert got == gold[f"pyr_{name}_{k}_sha256"].tobytes(), k


@gpu
def test_build_pyramid_matches_oracle_random(cuda):
    rng = np.random.default_rng(21)
    for trial in range(3):
        ps = 512
        counts = [int(c) for c in rng.integers(0, ps + 1, size=5)]
        counts[0] = ps
        dup = int(trial + 1)
        level0 = inputs.padded_pages(counts, ps, seed0=40 + 10 * trial, dup=dup)
        seed = int(rng.integers(0, 1000))
        want = olod.build_pyramid(level0, ps, 3, max_iters=20, seed=seed)
        got = lod.build_pyramid(level0, ps, level_count=3, max_iters=20, seed=seed)
        for k in (1, 2):
            assert np.array_equal(got[k], want[k]), (trial, k)


# -- pkg/tests/test_lod.py through vmsplat.lod (GPU) -------------------------------

@gpu
def test_ref_cluster_assignment_shape_and_range(cuda):
    records = inputs.wall_scene(seed=6, count=120, extent=2.0, z=0.0)
    assign = lod.cluster_page(records, 16, seed=3)
    assert assign.shape == (120,)
    assert assign.min() >= 0 and assign.max() < 16
    assert len(np.unique(assign)) == 16


@gpu
def test_ref_cluster_deterministic_and_identity(cuda):
    records = inputs.wall_scene(seed=6, count=120, extent=2.0, z=0.0)
    assert np.array_equal(lod.cluster_page(records, 10, seed=3), lod.cluster_page(records, 10, seed=3))
    eight = inputs.wall_scene(seed=6, count=8, extent=2.0, z=0.0)
    assert np.array_equal(lod.cluster_page(eight, 8, seed=0), np.arange(8))
    assert np.array_equal(lod.cluster_page(eight, 20, seed=0), np.arange(8))


@gpu
def test_ref_cluster_groups_separated_blobs(cuda):
    a = inputs.wall_scene(seed=1, count=30, extent=0.5, z=0.0)
    b = inputs.wall_scene(seed=2, count=30, extent=0.5, z=50.0)
    assign = lod.cluster_page(np.concatenate([a, b]), 2, seed=1)
    assert len(np.unique(assign[:30])) == 1 and len(np.unique(assign[30:])) == 1
    assert assign[0] != assign[30]


@gpu
def test_ref_merge_means_scale_and_hemisphere(cuda):
    records = inputs.wall_scene(seed=7, count=6, extent=1.0, z=0.0)
    merged = lod.merge_cluster(records)
    assert merged.shape == (RECORD_SIZE,)
    assert np.allclose(merged[0:3], records[:, 0:3].mean(axis=0), atol=1e-6)
    assert np.allclose(merged[10], records[:, 10].mean(), atol=1e-6)
    assert np.allclose(merged[11:], records[:, 11:].mean(axis=0), atol=1e-5)
    assert np.allclose(merged[7:10], records[:, 7:10].mean(axis=0) * 2.0 ** (1.0 / 3.0), rtol=1e-6)
    assert np.isclose(np.linalg.norm(merged[3:7]), 1.0, atol=1e-6)
    rec = records[0]
    flipped = rec.copy()
    flipped[3:7] *= -1.0
    m2 = lod.merge_cluster(np.stack([rec, flipped]))
    assert abs(float(np.dot(m2[3:7], rec[3:7]))) > 0.999999


@gpu
def test_ref_pyramid_counts_padding_determinism(cuda):
    page_size, counts = 64, [64, 50, 7]
    level0 = np.concatenate([_padded_page(inputs.wall_scene(seed=10 + i, count=c, extent=2.0,
                                                            z=0.0), page_size)
                             for i, c in enumerate(counts)])
    levels = lod.build_pyramid(level0, page_size, level_count=3, max_iters=10, seed=7)
    again = lod.build_pyramid(level0, page_size, level_count=3, max_iters=10, seed=7)
    assert len(levels) == 3
    for k, arr in enumerate(levels):
        per = page_size >> k
        assert arr.shape == (len(counts) * per, RECORD_SIZE)
        assert np.array_equal(arr, again[k])
    for p, c in enumerate(counts):
        want = c
        for k, arr in enumerate(levels):
            per = page_size >> k
            live = ~is_padding(arr[p * per:(p + 1) * per])
            assert not live[int(live.sum()):].any()
            assert int(live.sum()) == want
            want = (want + 1) // 2 if want > 1 else 1
