"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's level-of-detail pyramid
(pkg/src/vmsplat/lod.py) with every reduction order and random draw written
out explicitly - the specification the GPU kernel csrc/lod.cu follows:

* NumPy's Philox4x64-10 stream (numpy/random/src/philox/philox.h: counter
  increment before each 4-word block, 10 rounds with key bumps, the 32-bit
  draw splitting a 64-bit word low half first), ``Generator.integers`` as
  Lemire's bounded 32-bit draw, ``Generator.random`` as the 53-bit double,
  ``Generator.choice(m, p)`` as searchsorted(cumsum(p) / cumsum(p)[-1],
  random(), 'right');
* NumPy's pairwise summation for 1-D sums and for the contiguous 14-term
  row sums of the squared feature differences; row-sequential column means
  (``.mean(axis=0)``), pairwise 1-D means (``r[:, 10].mean()``); the BLAS
  4-term dot as a chain of fused multiply-adds.

Parity is PINNED: tests/golden/make_lod_golden.py runs the live reference
(in the build container) and stores its outputs in tests/golden/lod.npz;
tests/test_lod.py checks this module against them bit for bit, and the
Philox/choice restatement against NumPy itself.

Who may import this module: ``tests/`` only (the GPU parity tests use it as
the checker on inputs larger than the stored goldens).
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

RECORD_SIZE = 59
M64 = (1 << 64) - 1


class Philox:
    """NumPy's Philox4x64-10 bit generator with Generator's draws."""

    def __init__(self, key, counter):
        self.key = [int(k) & M64 for k in key]
        self.ctr = [int(c) & M64 for c in counter]
        self.buf = [0, 0, 0, 0]
        self.pos = 4
        self.has32 = False
        self.u32 = 0

    @classmethod
    def page(cls, seed: int, page_id: int) -> "Philox":
        return cls([seed, 1], [page_id, 0, 0, 0])  # lod.py:44-46

    def _block(self):
        c = list(self.ctr)
        k0, k1 = self.key
        for r in range(10):
            p0 = 0xD2E7470EE14C6C93 * c[0]
            p1 = 0xCA5A826395121157 * c[2]
            c = [(p1 >> 64) ^ c[1] ^ k0, p1 & M64, (p0 >> 64) ^ c[3] ^ k1, p0 & M64]
            k0 = (k0 + 0x9E3779B97F4A7C15) & M64
            k1 = (k1 + 0xBB67AE8584CAA73B) & M64
        return c

    def next64(self) -> int:
        if self.pos < 4:
            v = self.buf[self.pos]
            self.pos += 1
            return v
        for i in range(4):
            self.ctr[i] = (self.ctr[i] + 1) & M64
            if self.ctr[i]:
                break
        self.buf = self._block()
        self.pos = 1
        return self.buf[0]

    def next32(self) -> int:
        if self.has32:
            self.has32 = False
            return self.u32
        v = self.next64()
        self.has32 = True
        self.u32 = v >> 32
        return v & 0xFFFFFFFF

    def random(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def integers(self, m: int) -> int:
        rng = m - 1
        if rng == 0:
            return 0
        x = self.next32() * m
        if (x & 0xFFFFFFFF) < m:
            thr = (0xFFFFFFFF - rng) % m
            while (x & 0xFFFFFFFF) < thr:
                x = self.next32() * m
        return x >> 32

    def choice(self, p: np.ndarray) -> int:
        cdf = sequential_cumsum(p)
        cdf = cdf / cdf[-1]
        return int(np.searchsorted(cdf, self.random(), side="right"))


def pairwise_sum(a) -> float:
    """numpy/_core/src/umath/loops_utils.h.src pairwise_sum."""
    n = len(a)
    if n < 8:
        r = 0.0
        for x in a:
            r += float(x)
        return r
    if n <= 128:
        r = [float(x) for x in a[:8]]
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += float(a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:n2]) + pairwise_sum(a[n2:])


def sequential_cumsum(a) -> np.ndarray:
    out = np.empty(len(a), dtype=np.float64)
    run = 0.0
    for i, x in enumerate(a):
        run = float(x) if i == 0 else run + float(x)
        out[i] = run
    return out


def colmean(rows: np.ndarray) -> np.ndarray:
    """Column mean of a 2-D f64 array, rows added in order from the first."""
    s = rows[0].copy()
    for r in rows[1:]:
        s = s + r
    return s / len(rows)


def row_dist14(diff: np.ndarray) -> np.ndarray:
    """Pairwise sum over the last axis (length 14) of diff**2, vectorised."""
    s = diff * diff
    r = ((s[..., 0] + s[..., 1]) + (s[..., 2] + s[..., 3])) + \
        ((s[..., 4] + s[..., 5]) + (s[..., 6] + s[..., 7]))
    for j in range(8, 14):
        r = r + s[..., j]
    return r


def fdot4(q, r) -> float:
    """BLAS dot of two 4-vectors: fma chain (exact rational, then rounded)."""
    acc = float(q[0]) * float(r[0])
    for j in (1, 2, 3):
        acc = float(Fraction(float(q[j])) * Fraction(float(r[j])) + Fraction(acc))
    return acc


def features(records: np.ndarray, w) -> np.ndarray:
    """lod.py:49-59"""
    r = np.asarray(records, dtype=np.float32).astype(np.float64)
    quat = r[:, 3:7].copy()
    quat[quat[:, 0] < 0] *= -1.0
    return np.hstack([r[:, 0:3] * w[0], quat * w[1], r[:, 7:10] * w[2], r[:, 10:11] * w[3],
                      r[:, 11:14] * w[4]])


def kmeans_pp(feat: np.ndarray, k: int, rng: Philox) -> np.ndarray:
    """lod.py:62-80"""
    m = len(feat)
    centers = np.empty((k, feat.shape[1]), dtype=np.float64)
    centers[0] = feat[rng.integers(m)]
    d2 = row_dist14(feat - centers[0])
    for c in range(1, k):
        total = pairwise_sum(d2)
        idx = rng.integers(m) if total <= 0.0 else rng.choice(d2 / total)
        centers[c] = feat[idx]
        d2 = np.minimum(d2, row_dist14(feat - centers[c]))
    return centers


def cluster_page(records: np.ndarray, k: int, w=(1.0, 0.1, 0.1, 0.05, 0.1), max_iters: int = 50,
                 rng: Philox | None = None, seed: int = 0) -> np.ndarray:
    """lod.py:83-131"""
    m = len(records)
    if k >= m:
        return np.arange(m, dtype=np.int64)
    if rng is None:
        rng = Philox.page(seed, 0)
    feat = features(records, w)
    centers = kmeans_pp(feat, k, rng)
    assign = np.full(m, -1, dtype=np.int64)
    prev = np.inf
    for _ in range(max_iters):
        d2 = row_dist14(feat[:, None, :] - centers[None, :, :])
        new = d2.argmin(axis=1)
        pd2 = d2[np.arange(m), new]
        inertia = pairwise_sum(pd2)
        if inertia > prev + 1e-9 * max(1.0, prev):
            raise RuntimeError("k-means inertia increased")
        prev = inertia
        if np.array_equal(new, assign):
            break
        assign = new
        counts = np.bincount(assign, minlength=k)
        for c in np.flatnonzero(counts == 0):
            far = int(pd2.argmax())
            centers[c] = feat[far]
            counts[assign[far]] -= 1
            assign[far] = c
            counts[c] += 1
            pd2[far] = 0.0
        for c in range(k):
            if counts[c]:
                centers[c] = colmean(feat[assign == c])
    return assign


def merge_cluster(members: np.ndarray, scale_factor: float = 2.0 ** (1.0 / 3.0)) -> np.ndarray:
    """lod.py:134-154"""
    r = np.asarray(members, dtype=np.float32).reshape(-1, RECORD_SIZE).astype(np.float64)
    out = np.empty(RECORD_SIZE, dtype=np.float64)
    out[0:3] = colmean(r[:, 0:3])
    quat = r[:, 3:7].copy()
    ref = quat[0].copy()
    for i in range(len(quat)):
        if fdot4(quat[i], ref) < 0:
            quat[i] *= -1.0
    q = colmean(quat)
    norm = float(np.sqrt(fdot4(q, q)))
    out[3:7] = ref if norm < 1e-6 else q / norm
    out[7:10] = colmean(r[:, 7:10]) * scale_factor
    out[10] = pairwise_sum(r[:, 10]) / len(r)
    out[11:] = colmean(r[:, 11:])
    return out.astype(np.float32)


def build_pyramid(level0: np.ndarray, page_size: int, level_count: int = 4,
                  scale_factor: float = 2.0 ** (1.0 / 3.0), max_iters: int = 50, seed: int = 7,
                  w=(1.0, 0.1, 0.1, 0.05, 0.1)) -> list:
    """lod.py:157-226 (pages in order; each page's stream continues across
    its levels)."""
    level0 = np.asarray(level0, dtype=np.float32).reshape(-1, RECORD_SIZE)
    pages = len(level0) // page_size
    out = [level0] + [np.zeros((pages * (page_size >> k), RECORD_SIZE), np.float32)
                      for k in range(1, level_count)]
    for p in range(pages):
        rng = Philox.page(seed, p + 1)
        cur = level0[p * page_size:(p + 1) * page_size]
        for k in range(1, level_count):
            cap = page_size >> k
            live = cur[cur.any(axis=1)]
            merged = np.zeros((cap, RECORD_SIZE), np.float32)
            if len(live):
                assign = cluster_page(live, -(-len(live) // 2), w, max_iters, rng)
                n = 0
                for c in range(int(assign.max()) + 1):
                    sel = live[assign == c]
                    if len(sel):
                        merged[n] = merge_cluster(sel, scale_factor)
                        n += 1
            out[k][p * cap:(p + 1) * cap] = merged
            cur = merged
    return out
