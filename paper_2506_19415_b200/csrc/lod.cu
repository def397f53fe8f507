// SURVEY §8(f) F3, preprocessing accelerator: the weighted k-means level-of-
// detail pyramid of pkg/src/vmsplat/lod.py (features :44-59, k-means++ seeding
// :62-80, Lloyd iterations with empty-cluster reseeding :83-131, the attribute
// merge :134-154, the per-page level loop :157-176) on the GPU, one CTA per
// page, with results bit-identical to the reference's NumPy.
//
// Exactness: every FP64 operation is rounded separately (compiled with
// -fmad=false, explicit __d*_rn) and every reduction follows the order NumPy
// uses for the reference's expressions (pinned against NumPy 2.3 in
// tests/test_lod.py and oracle/lod.py):
//   * a row sum of 14 squared differences (`.sum(axis=2)` / `.sum(axis=1)` on
//     a contiguous last axis) and a 1-D sum (`d2.sum()`, `point_d2.sum()`,
//     `r[:, 10].mean()`) are NumPy's pairwise sum: blocks of <= 128 elements
//     with 8 interleaved accumulators, halves split at a multiple of 8;
//   * a column mean (`.mean(axis=0)` of a 2-D array) adds the rows in order
//     starting from the first row, then divides by the count;
//   * `np.cumsum` is sequential; `Generator.choice(m, p=...)` is
//     cdf = cumsum(p), cdf /= cdf[-1], searchsorted(cdf, random(), 'right');
//   * `np.linalg.norm` of a 4-vector and `quat @ ref` use the host BLAS dot,
//     fma(q3, r3, fma(q2, r2, fma(q1, r1, q0 * r0))) (measured; `quat @ ref`
//     only feeds a sign test).
// The random streams are NumPy's Philox4x64-10 bit generator (key, counter,
// 4-word output buffer, the split 32-bit half) with Lemire's bounded integers
// and the 53-bit double - the state is handed in and written back, so a
// caller's numpy Generator continues exactly where the reference would.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace vms {
namespace {

constexpr int kFeat = 14;        // position 3, rotation 4, scale 3, opacity 1, SH DC 3
constexpr int kRec = 59;         // record floats (gaussians.py:27)
constexpr int kThreads = 256;
constexpr int kTile = 64;        // centers per shared-memory tile in the assignment
constexpr int kMaxLeaves = 64;   // pairwise-sum leaves for n <= 4096

// ---------------------------------------------------------------------------
// NumPy Philox4x64-10 (numpy/random/src/philox/philox.h) + Generator draws
struct Philox {
  uint64_t ctr[4], key[2], buf[4];
  int pos, has32;
  uint32_t u32;
};

VMS_DEV void philox_block(Philox& s) {
  uint64_t c0 = s.ctr[0], c1 = s.ctr[1], c2 = s.ctr[2], c3 = s.ctr[3];
  uint64_t k0 = s.key[0], k1 = s.key[1];
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
    const uint64_t lo1 = 0xCA5A826395121157ull * c2, hi1 = __umul64hi(0xCA5A826395121157ull, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  s.buf[0] = c0;
  s.buf[1] = c1;
  s.buf[2] = c2;
  s.buf[3] = c3;
}

VMS_DEV uint64_t next64(Philox& s) {
  if (s.pos < 4) return s.buf[s.pos++];
  for (int i = 0; i < 4; ++i)
    if (++s.ctr[i] != 0) break;
  philox_block(s);
  s.pos = 1;
  return s.buf[0];
}

VMS_DEV uint32_t next32(Philox& s) {
  if (s.has32) {
    s.has32 = 0;
    return s.u32;
  }
  const uint64_t v = next64(s);
  s.has32 = 1;
  s.u32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

// Generator.random(): 53-bit double
VMS_DEV double next_double(Philox& s) {
  return (double)(next64(s) >> 11) * (1.0 / 9007199254740992.0);
}

// Generator.integers(m) for 1 <= m < 2^32: Lemire's bounded 32-bit draw
VMS_DEV uint32_t bounded(Philox& s, uint32_t m) {
  const uint32_t rng = m - 1;
  if (rng == 0) return 0;
  const uint32_t excl = m;
  uint64_t x = (uint64_t)next32(s) * excl;
  uint32_t left = (uint32_t)x;
  if (left < excl) {
    const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
    while (left < thr) {
      x = (uint64_t)next32(s) * excl;
      left = (uint32_t)x;
    }
  }
  return (uint32_t)(x >> 32);
}

// ---------------------------------------------------------------------------
// NumPy pairwise summation (numpy/_core/src/umath/loops_utils.h.src)
template <class F>
VMS_DEV double pw_leaf(F at, int off, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = dadd(r, at(off + i));
    return r;
  }
  double r0 = at(off), r1 = at(off + 1), r2 = at(off + 2), r3 = at(off + 3);
  double r4 = at(off + 4), r5 = at(off + 5), r6 = at(off + 6), r7 = at(off + 7);
  int i = 8;
  const int lim = n - (n % 8);
  for (; i < lim; i += 8) {
    r0 = dadd(r0, at(off + i));
    r1 = dadd(r1, at(off + i + 1));
    r2 = dadd(r2, at(off + i + 2));
    r3 = dadd(r3, at(off + i + 3));
    r4 = dadd(r4, at(off + i + 4));
    r5 = dadd(r5, at(off + i + 5));
    r6 = dadd(r6, at(off + i + 6));
    r7 = dadd(r7, at(off + i + 7));
  }
  double res = dadd(dadd(dadd(r0, r1), dadd(r2, r3)), dadd(dadd(r4, r5), dadd(r6, r7)));
  for (; i < n; ++i) res = dadd(res, at(off + i));
  return res;
}

// Whole pairwise sum on one thread (recursion depth <= log2(n / 128)).
template <class F>
__device__ double pw_sum(F at, int off, int n) {
  if (n <= 128) return pw_leaf(at, off, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  const double a = pw_sum(at, off, n2);
  return dadd(a, pw_sum(at, off + n2, n - n2));
}

// The pairwise recursion's shape for a given n, built once: the leaves (in
// order) and the internal nodes in post-order, each adding its two children
// (a child < kNodeBase is a leaf, else node child - kNodeBase).
constexpr int kNodeBase = 1 << 12;

__device__ int pw_build(int off, int n, int* lo, int* ln, int& nl, int* nleft, int* nright,
                        int& nn) {
  if (n <= 128) {
    lo[nl] = off;
    ln[nl] = n;
    return nl++;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  const int l = pw_build(off, n2, lo, ln, nl, nleft, nright, nn);
  const int r = pw_build(off + n2, n - n2, lo, ln, nl, nleft, nright, nn);
  nleft[nn] = l;
  nright[nn] = r;
  return kNodeBase + nn++;
}

// sum of the 14 squared feature differences, NumPy's pairwise order for n=14
VMS_DEV double dist14(const double* f, const double* c) {
  double s[kFeat];
#pragma unroll
  for (int j = 0; j < kFeat; ++j) {
    const double d = dsub(f[j], c[j]);
    s[j] = dmul(d, d);
  }
  double r = dadd(dadd(dadd(s[0], s[1]), dadd(s[2], s[3])), dadd(dadd(s[4], s[5]), dadd(s[6], s[7])));
#pragma unroll
  for (int j = 8; j < kFeat; ++j) r = dadd(r, s[j]);
  return r;
}

VMS_DEV double dot4(const double* q, const double* r) {
  return __fma_rn(q[3], r[3], __fma_rn(q[2], r[2], __fma_rn(q[1], r[1], dmul(q[0], r[0]))));
}

struct Shared {
  Philox rng;
  double total, u, prev_inertia;
  int idx, changed, any_empty, n_live, k, stop, leaves, nodes;
  int leaf_off[kMaxLeaves], leaf_n[kMaxLeaves], node_l[kMaxLeaves], node_r[kMaxLeaves];
  double leaf_sum[kMaxLeaves], node_sum[kMaxLeaves];
  double ctr[kFeat];
  int warp_tot[kThreads / 32];
};

// block-wide pairwise sum of a[0..n) in shared memory: the leaves on
// separate threads, then thread 0 adds the internal nodes in post-order
// (the recursion's order); result in sh.total.  The shape is built once
// per n (plan_n: thread 0's record of the n it was built for, -1 at first).
__device__ void block_pw(Shared& sh, const double* a, int n, int& plan_n) {
  if (threadIdx.x == 0) {
    if (plan_n != n) {
      int nl = 0, nn = 0;
      pw_build(0, n, sh.leaf_off, sh.leaf_n, nl, sh.node_l, sh.node_r, nn);
      sh.leaves = nl;
      sh.nodes = nn;
      plan_n = n;
    }
  }
  __syncthreads();
  auto at = [a](int i) { return a[i]; };
  for (int l = threadIdx.x; l < sh.leaves; l += blockDim.x)
    sh.leaf_sum[l] = pw_leaf(at, sh.leaf_off[l], sh.leaf_n[l]);
  __syncthreads();
  if (threadIdx.x == 0) {
    auto val = [&](int c) { return c < kNodeBase ? sh.leaf_sum[c] : sh.node_sum[c - kNodeBase]; };
    for (int j = 0; j < sh.nodes; ++j) sh.node_sum[j] = dadd(val(sh.node_l[j]), val(sh.node_r[j]));
    sh.total = sh.nodes ? sh.node_sum[sh.nodes - 1] : sh.leaf_sum[0];
  }
  __syncthreads();
}

// exclusive scan of in[0..n) into out[0..n]; out[n] = total
__device__ void block_scan(Shared& sh, const int* in, int* out, int n) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int b = threadIdx.x * per, e = min(b + per, n);
  int s = 0;
  for (int i = b; i < e; ++i) s += in[i];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = s;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh.warp_tot[w] = x;
  __syncthreads();
  int base = 0;
  for (int i = 0; i < w; ++i) base += sh.warp_tot[i];
  int run = base + x - s;
  for (int i = b; i < e; ++i) {
    out[i] = run;
    run += in[i];
  }
  if (threadIdx.x == blockDim.x - 1) out[n] = run;
  __syncthreads();
}

struct LodArgs {
  const float* in;
  uint32_t rows_in;
  float* out;
  uint32_t rows_out;
  double w[5];
  double scale_factor;
  int max_iters;
  int k_fixed;       // 0: pyramid level (padding filtered, k = ceil(live / 2), merge)
  Philox* rng;       // per page
  int32_t* assign;   // per page rows_in (cluster mode) or nullptr
  int32_t* status;   // per page: 0 ok, 1 inertia increased, 2 level overflow
  double* feat_ws;   // per page rows_in x 14
  double* cent_ws;   // per page rows_in x 14
  int* live_ws;      // per page rows_in: the live rows in order (seeding -> Lloyd)
  int* m_ws;         // per page: live row count
  uint32_t k_cap;
};

// Two launches per level: phase 1 (kSeedThreads threads, shared memory for
// the two distance arrays only, so ~5 pages share an SM and their serial
// k-means++ cumsums overlap) finds the live rows, builds the features and
// seeds the centres; phase 2 (kThreads) runs the Lloyd iterations and the
// merge.  Both phases keep the page's state in global memory (features,
// centres, live rows, the Philox state).
constexpr int kSeedThreads = 128;
__device__ int g_lod_prof = 0;  // VMSPLAT_LOD_PROF=1: per-section clocks of page 0's seeding

template <int phase>
__device__ __forceinline__ void lod_page(const LodArgs& a, Shared& sh) {
  extern __shared__ __align__(16) unsigned char smem[];
  int plan_n = -1;  // block_pw's shape cache (thread 0)
  const uint32_t page = blockIdx.x;
  const int R = (int)a.rows_in, K = (int)a.k_cap;
  double* d2 = reinterpret_cast<double*>(smem);
  double* cdf = d2 + R;  // phase 1: R + 2 doubles (also the live scan's scratch)
  double* tile = cdf;    // phase 2
  int* live = reinterpret_cast<int*>(tile + kTile * kFeat);
  int* asg = live + (R + 1);
  int* mem = asg + R;
  int* cnt = mem + (R + 1);
  int* off = cnt + (K + 1);
  const float* in = a.in + (size_t)page * R * kRec;
  double* feat = a.feat_ws + (size_t)page * R * kFeat;
  double* cent = a.cent_ws + (size_t)page * R * kFeat;
  int* glive = a.live_ws + (size_t)page * R;
  const int tid = threadIdx.x, NT = blockDim.x;

  if (phase == 1) {
    // live rows in order (is_padding: all-zero rows, gaussians.py:71-73)
    int* flag = reinterpret_cast<int*>(cdf);  // R + 1 ints
    int* pos = flag + (R + 1);                // R + 1 ints
    if (a.k_fixed == 0) {  // pyramid level: padding rows are not clustered
      for (int i = tid; i < R; i += NT) {
        bool any = false;
        for (int j = 0; j < kRec; ++j) any |= in[(size_t)i * kRec + j] != 0.0f;
        flag[i] = any ? 1 : 0;
      }
      __syncthreads();
      block_scan(sh, flag, pos, R);
      for (int i = tid; i < R; i += NT)
        if (flag[i]) glive[pos[i]] = i;
      if (tid == 0) sh.n_live = pos[R];
    } else {
      for (int i = tid; i < R; i += NT) glive[i] = i;
      if (tid == 0) sh.n_live = R;
    }
    if (tid == 0) {
      sh.rng = a.rng[page];
      a.m_ws[page] = sh.n_live;
    }
    __syncthreads();
  } else {
    if (tid == 0) {
      sh.n_live = a.m_ws[page];
      sh.rng = a.rng[page];
      sh.stop = 0;
    }
    __syncthreads();
    for (int i = tid; i < sh.n_live; i += NT) live[i] = glive[i];
  }
  const int m = sh.n_live;
  if (m == 0) return;
  const int k = a.k_fixed > 0 ? a.k_fixed : a.k_fixed == 0 ? (m + 1) / 2 : 1;
  if (phase == 2)
    for (int i = tid; i < R; i += NT) asg[i] = -1;

  if (a.k_fixed < 0) {
    // merge_cluster of all rows (lod.py:134-154)
    if constexpr (phase == 1) {
      return;
    } else {
      for (int i = tid; i < m; i += NT) asg[i] = 0;
    }
  } else if (k >= m) {
    // cluster_page: k >= m -> arange(m), no draws (lod.py:96-97)
    if constexpr (phase == 1) {
      return;
    } else {
      for (int i = tid; i < m; i += NT) asg[i] = i;
    }
  } else if (phase == 1) {
    __syncthreads();  // glive complete
    // features (lod.py:44-59)
    for (int i = tid; i < m; i += NT) {
      const float* r = in + (size_t)glive[i] * kRec;
      double* f = feat + (size_t)i * kFeat;
      for (int j = 0; j < 3; ++j) f[j] = dmul((double)r[j], a.w[0]);
      const bool flip = (double)r[3] < 0.0;
      for (int j = 0; j < 4; ++j) {
        double q = (double)r[3 + j];
        if (flip) q = dmul(q, -1.0);
        f[3 + j] = dmul(q, a.w[1]);
      }
      for (int j = 0; j < 3; ++j) f[7 + j] = dmul((double)r[7 + j], a.w[2]);
      f[10] = dmul((double)r[10], a.w[3]);
      for (int j = 0; j < 3; ++j) f[11 + j] = dmul((double)r[11 + j], a.w[4]);
    }
    // k-means++ seeding (lod.py:62-80)
    if (tid == 0) sh.idx = (int)bounded(sh.rng, (uint32_t)m);
    __syncthreads();
    long long tp[6] = {0, 0, 0, 0, 0, 0};  // VMSPLAT_LOD_PROF: clock per section
    const bool prof = g_lod_prof && blockIdx.x == 0 && tid == 0;
    long long t0 = prof ? clock64() : 0;
    auto tick = [&](int k) {
      if (prof) {
        const long long t = clock64();
        tp[k] += t - t0;
        t0 = t;
      }
    };
    for (int c = 0; c < k; ++c) {
      if (c > 0) {
        block_pw(sh, d2, m, plan_n);
        tick(0);
        const double total = sh.total;
        if (!(total > 0.0)) {
          if (tid == 0) sh.idx = (int)bounded(sh.rng, (uint32_t)m);
        } else {
          for (int i = tid; i < m; i += NT) cdf[i] = ddiv(d2[i], total);
          __syncthreads();
          tick(1);
          if (tid == 0) {
            double run = 0.0;
            int i = 0;
            // sequential cumsum; loads run ahead of the dependent adds
            for (; i + 8 <= m; i += 8) {
              double v[8];
#pragma unroll
              for (int t = 0; t < 8; ++t) v[t] = cdf[i + t];
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                run = (i + t == 0) ? v[t] : dadd(run, v[t]);
                cdf[i + t] = run;
              }
            }
            for (; i < m; ++i) {
              run = (i == 0) ? cdf[0] : dadd(run, cdf[i]);
              cdf[i] = run;
            }
            tick(2);
            // searchsorted(cdf / cdf[-1], u, 'right'): RN(x / last) is
            // monotone in x, so the first index past u is found by bisection
            const double u = next_double(sh.rng), last = run;
            int lo = 0, hi = m - 1;  // cdf[m - 1] / last == 1 > u
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (ddiv(cdf[mid], last) > u) hi = mid; else lo = mid + 1;
            }
            sh.idx = lo;
            tick(3);
          }
        }
        __syncthreads();
      }
      const int idx = sh.idx;
      if (tid < kFeat) {
        const double v = feat[(size_t)idx * kFeat + tid];
        sh.ctr[tid] = v;
        cent[(size_t)c * kFeat + tid] = v;
      }
      __syncthreads();
      for (int i = tid; i < m; i += NT) {
        double f[kFeat];
#pragma unroll
        for (int j = 0; j < kFeat; ++j) f[j] = feat[(size_t)i * kFeat + j];
        const double d = dist14(f, sh.ctr);
        d2[i] = (c == 0) ? d : fmin(d2[i], d);
      }
      __syncthreads();
      tick(4);
    }
    if (prof)
      printf("[lod seed] m %d k %d cycles: pairwise %lld, divide %lld, cumsum %lld, search %lld, "
             "distances %lld\n", m, k, tp[0], tp[1], tp[2], tp[3], tp[4]);
    if (tid == 0) a.rng[page] = sh.rng;
    return;
  } else {
    // Lloyd iterations (lod.py:106-130)
    if (tid == 0) sh.prev_inertia = __longlong_as_double(0x7FF0000000000000ll);
    for (int it = 0; it < a.max_iters; ++it) {
      if (tid == 0) sh.changed = 0;
      __syncthreads();
      for (int base = 0; base < m; base += 2 * NT) {
        const int i0 = base + tid, i1 = base + NT + tid;
        const bool v0 = i0 < m, v1 = i1 < m;
        double f0[kFeat], f1[kFeat];
#pragma unroll
        for (int j = 0; j < kFeat; ++j) {
          f0[j] = v0 ? feat[(size_t)i0 * kFeat + j] : 0.0;
          f1[j] = v1 ? feat[(size_t)i1 * kFeat + j] : 0.0;
        }
        double b0 = __longlong_as_double(0x7FF0000000000000ll), b1 = b0;
        int c0 = 0, c1 = 0;
        for (int t0 = 0; t0 < k; t0 += kTile) {
          const int tn = min(kTile, k - t0);
          __syncthreads();
          for (int x = tid; x < tn * kFeat; x += NT) tile[x] = cent[(size_t)t0 * kFeat + x];
          __syncthreads();
          for (int t = 0; t < tn; ++t) {
            const double* cc = tile + t * kFeat;
            const double d0 = dist14(f0, cc);
            const double d1 = dist14(f1, cc);
            if (d0 < b0) {
              b0 = d0;
              c0 = t0 + t;
            }
            if (d1 < b1) {
              b1 = d1;
              c1 = t0 + t;
            }
          }
        }
        if (v0) {
          if (asg[i0] != c0) sh.changed = 1;
          asg[i0] = c0;
          d2[i0] = b0;
        }
        if (v1) {
          if (asg[i1] != c1) sh.changed = 1;
          asg[i1] = c1;
          d2[i1] = b1;
        }
      }
      __syncthreads();
      block_pw(sh, d2, m, plan_n);
      if (tid == 0) {
        const double inertia = sh.total, prev = sh.prev_inertia;
        if (inertia > dadd(prev, dmul(1e-9, fmax(1.0, prev)))) {
          a.status[page] = 1;
          sh.stop = 1;
        }
        sh.prev_inertia = inertia;
      }
      __syncthreads();
      if (sh.stop) return;
      if (!sh.changed) break;
      // counts, reseed of the clusters empty now (lod.py:120-126)
      for (int c = tid; c < k; c += NT) cnt[c] = 0;
      if (tid == 0) sh.any_empty = 0;
      __syncthreads();
      for (int i = tid; i < m; i += NT) atomicAdd(&cnt[asg[i]], 1);
      __syncthreads();
      for (int c = tid; c < k; c += NT) {
        off[c] = cnt[c] == 0 ? 1 : 0;  // the fixed list of empty clusters
        if (cnt[c] == 0) sh.any_empty = 1;
      }
      __syncthreads();
      if (sh.any_empty && tid == 0) {
        for (int c = 0; c < k; ++c) {
          if (!off[c]) continue;
          int far = 0;
          double best = d2[0];
          for (int i = 1; i < m; ++i)
            if (d2[i] > best) {
              best = d2[i];
              far = i;
            }
          for (int j = 0; j < kFeat; ++j)
            cent[(size_t)c * kFeat + j] = feat[(size_t)far * kFeat + j];
          cnt[asg[far]] -= 1;
          asg[far] = c;
          cnt[c] += 1;
          d2[far] = 0.0;
        }
      }
      __syncthreads();
      // members of every cluster in index order (stable counting sort)
      block_scan(sh, cnt, off, k);
      if (tid < 32) {
        for (int b = 0; b < m; b += 32) {
          const int i = b + tid;
          const int c = i < m ? asg[i] : -1 - tid;
          const uint32_t peers = __match_any_sync(0xFFFFFFFFu, c);
          const int rank = __popc(peers & lanemask_lt());
          int pos = 0;
          if (i < m) pos = off[c] + rank;
          __syncwarp();
          if (i < m) {
            mem[pos] = i;
            if (rank == 0) off[c] += __popc(peers);
          }
          __syncwarp();
        }
      }
      __syncthreads();
      // off[c] now holds the end of c's run; the start is end - cnt[c]
      for (int t = tid; t < k * kFeat; t += NT) {
        const int c = t / kFeat, j = t - c * kFeat;
        const int n = cnt[c];
        if (!n) continue;
        const int b = off[c] - n;
        double s = feat[(size_t)mem[b] * kFeat + j];
        for (int r = 1; r < n; ++r) s = dadd(s, feat[(size_t)mem[b + r] * kFeat + j]);
        cent[(size_t)c * kFeat + j] = ddiv(s, (double)n);
      }
      __syncthreads();
    }
  }
  __syncthreads();
  if (a.k_fixed > 0) {
    int32_t* out = a.assign + (size_t)page * R;
    for (int i = tid; i < m; i += NT) out[i] = asg[i];
    if (tid == 0) a.rng[page] = sh.rng;
    return;
  }
  if (tid == 0) a.rng[page] = sh.rng;
  // merge every non-empty cluster, in cluster order (lod.py:134-154, 169-176)
  const int kk = a.k_fixed < 0 ? 1 : k >= m ? m : k;
  for (int c = tid; c < kk; c += NT) cnt[c] = 0;
  __syncthreads();
  for (int i = tid; i < m; i += NT)
    if (asg[i] >= 0) atomicAdd(&cnt[asg[i]], 1);
  __syncthreads();
  block_scan(sh, cnt, off, kk);
  if (tid < 32) {
    for (int b = 0; b < m; b += 32) {
      const int i = b + tid;
      const int c = (i < m && asg[i] >= 0) ? asg[i] : -1 - tid;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, c);
      const int rank = __popc(peers & lanemask_lt());
      int pos = 0;
      if (c >= 0) pos = off[c] + rank;
      __syncwarp();
      if (c >= 0) {
        mem[pos] = i;
        if (rank == 0) off[c] += __popc(peers);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  // members -> source rows (asg[] in member order), then the output slot of
  // cluster c = number of non-empty clusters before it (live[] is reused)
  const int placed = off[kk];
  for (int x = tid; x < placed; x += NT) asg[x] = live[mem[x]];
  __syncthreads();
  int* slot = live;
  for (int c = tid; c < kk; c += NT) slot[c] = cnt[c] > 0 ? 1 : 0;
  __syncthreads();
  block_scan(sh, slot, mem, kk);  // mem[c] = output row of cluster c
  if (tid == 0 && mem[kk] > (int)a.rows_out) a.status[page] = 2;
  __syncthreads();
  float* outp = a.out + (size_t)page * a.rows_out * kRec;
  for (int c = tid; c < kk; c += NT) {
    const int n = cnt[c];
    if (!n || mem[c] >= (int)a.rows_out) continue;
    const int b = off[c] - n;  // members asg[b .. b + n): source rows, in order
    float* o = outp + (size_t)mem[c] * kRec;
    auto row = [&](int r) { return in + (size_t)asg[b + r] * kRec; };
    auto colmean = [&](int j) {
      double s = (double)row(0)[j];
      for (int r = 1; r < n; ++r) s = dadd(s, (double)row(r)[j]);
      return ddiv(s, (double)n);
    };
    for (int j = 0; j < 3; ++j) o[j] = __double2float_rn(colmean(j));
    double ref[4], q[4];
    for (int j = 0; j < 4; ++j) ref[j] = (double)row(0)[3 + j];
    for (int r = 0; r < n; ++r) {
      double v[4];
      for (int j = 0; j < 4; ++j) v[j] = (double)row(r)[3 + j];
      const bool flip = dot4(v, ref) < 0.0;
      for (int j = 0; j < 4; ++j) {
        const double x = flip ? dmul(v[j], -1.0) : v[j];
        q[j] = r == 0 ? x : dadd(q[j], x);
      }
    }
    for (int j = 0; j < 4; ++j) q[j] = ddiv(q[j], (double)n);
    const double norm = __dsqrt_rn(dot4(q, q));
    for (int j = 0; j < 4; ++j) o[3 + j] = __double2float_rn(norm < 1e-6 ? ref[j] : ddiv(q[j], norm));
    for (int j = 7; j < 10; ++j) o[j] = __double2float_rn(dmul(colmean(j), a.scale_factor));
    auto op = [&](int r) { return (double)row(r)[10]; };
    o[10] = __double2float_rn(ddiv(pw_sum(op, 0, n), (double)n));
    for (int j = 11; j < kRec; ++j) o[j] = __double2float_rn(colmean(j));
  }
}

__global__ void __launch_bounds__(kSeedThreads) lod_seed_k(LodArgs a) {
  __shared__ Shared sh;
  lod_page<1>(a, sh);
}

__global__ void __launch_bounds__(kThreads) lod_lloyd_k(LodArgs a) {
  __shared__ Shared sh;
  lod_page<2>(a, sh);
}

}  // namespace
}  // namespace vms

extern "C" size_t vms_lod_workspace_bytes(uint32_t pages, uint32_t rows_in) {
  // features + centres (f64 x 14 per row), the live rows, the live counts
  return (size_t)pages * rows_in * (14 * sizeof(double) * 2 + sizeof(int)) +
         sizeof(int) * (size_t)pages;
}

extern "C" int32_t vms_lod_level(const float* in, uint32_t pages, uint32_t rows_in, float* out,
                                 uint32_t rows_out, const vms_lod_params* p, vms_philox* rng,
                                 int32_t* assign_out, int32_t* status, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  using namespace vms;
  if (!p || !in || !rng || !status || !workspace || rows_in < 1 || rows_in > 4096 ||
      p->max_iters < 0 || p->k < -1 || (p->k > 0 && ((uint32_t)p->k >= rows_in || !assign_out)) ||
      (p->k <= 0 && (!out || rows_out < 1)) ||
      workspace_bytes < vms_lod_workspace_bytes(pages, rows_in)) {
    set_error("lod_level: invalid arguments");
    return VMS_ERR_INVALID;
  }
  static_assert(sizeof(Philox) == sizeof(vms_philox), "Philox state layout");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  VMS_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t) * pages, s));
  if (p->k <= 0) VMS_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * kRec * rows_out * (size_t)pages, s));
  if (pages == 0) return VMS_OK;
  LodArgs a{};
  a.in = in;
  a.rows_in = rows_in;
  a.out = out;
  a.rows_out = rows_out;
  for (int i = 0; i < 5; ++i) a.w[i] = p->weights[i];
  a.scale_factor = p->scale_factor;
  a.max_iters = p->max_iters;
  a.k_fixed = p->k;
  a.rng = reinterpret_cast<Philox*>(rng);
  a.assign = assign_out;
  a.status = status;
  a.feat_ws = static_cast<double*>(workspace);
  a.cent_ws = a.feat_ws + (size_t)pages * rows_in * kFeat;
  a.live_ws = reinterpret_cast<int*>(a.cent_ws + (size_t)pages * rows_in * kFeat);
  a.m_ws = a.live_ws + (size_t)pages * rows_in;
  a.k_cap = p->k > 0 ? (uint32_t)p->k : (rows_in + 1) / 2;
  const size_t smem1 = sizeof(double) * (2 * (size_t)rows_in + 2);
  const size_t smem2 = sizeof(double) * ((size_t)rows_in + kTile * kFeat) +
                       sizeof(int) * (3 * (size_t)rows_in + 2 + 2 * ((size_t)a.k_cap + 1));
  VMS_CUDA(cudaFuncSetAttribute(lod_seed_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1));
  VMS_CUDA(cudaFuncSetAttribute(lod_lloyd_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
  static const int prof = [] {
    const char* e = getenv("VMSPLAT_LOD_PROF");
    return e && e[0] == '1' ? 1 : 0;
  }();
  if (prof) VMS_CUDA(cudaMemcpyToSymbolAsync(g_lod_prof, &prof, sizeof(int), 0,
                                             cudaMemcpyHostToDevice, s));
  lod_seed_k<<<pages, kSeedThreads, smem1, s>>>(a);
  lod_lloyd_k<<<pages, kThreads, smem2, s>>>(a);
  mark("lod_page", s);
  VMS_LAUNCH_CHECK("lod_level");
  return VMS_OK;
}
