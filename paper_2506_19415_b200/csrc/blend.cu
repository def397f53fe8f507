// Subsystems [5] + [6]: (tile, depth) ordering and per-tile compositing.
//
//   compact_k     kept splats in gather order -> (depth key, gather idx)
//   radix (32b)   stable depth sort: ties keep gather order (render.py:235-239)
//   dup_count_k   per sorted splat: tile rectangle, instance count, and the
//                 per-tile counts as a 2D difference array
//   tile_prep_k   per-tile counts -> list ranges, overflow, the tile sort's
//                 digit histograms, the blend schedule (one CTA)
//   dup_emit_k    one instance per overlapped tile, emitted in depth order
//   radix (tile)  stable sort on the tile id only -> per tile the instances
//                 are in (depth key, gather idx) order, i.e. the reference's
//                 global order restricted to the tile (SURVEY §0 finding 1)
//   blend_k       one CTA per tile, one thread per pixel; splats staged in
//                 shared memory 256 at a time; per-pixel half-open bbox test,
//                 stop test before blending, 0.99 clamp, early exit once every
//                 pixel of the tile has T < 1/255 (_core.pyx:24-78).
//
// Fast mode blends in FP32 (measured <= 2.6e-5 from the FP64 reference,
// SURVEY A16); exact mode reproduces the reference's FP64 arithmetic with
// f32 storage of T and colour.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "prims.h"
#include "render.h"

namespace vms {

int tile_size() {
  static const int ts = [] {
    const char* e = std::getenv("VMSPLAT_TILE");
    return (e && std::atoi(e) == 16) ? 16 : 32;
  }();
  return ts;
}

uint32_t tile_count(int width, int height) {
  const int t = tile_size();
  return (uint32_t)(ceil_div(width, t) * ceil_div(height, t));
}

namespace {

constexpr int kBlendThreads = 256;

template <typename T>
T* carve(char*& p, size_t n) {
  uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255);
  T* r = reinterpret_cast<T*>(a);
  p = reinterpret_cast<char*>(a + sizeof(T) * n);
  return r;
}

__global__ void compact_k(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                          const uint32_t* __restrict__ key_g, const uint32_t* n_dev, uint32_t n_host,
                          uint32_t* __restrict__ k0, uint32_t* __restrict__ v0) {
  pdl_wait();
  const uint32_t n = n_dev ? *n_dev : n_host;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
    if (!flag[g]) continue;
    const uint32_t o = pos[g];
    k0[o] = key_g[g];
    v0[o] = g;
  }
}

constexpr int kDiffSmemWords = 12288;  // 48 KB
constexpr int kMaxBands = 8;           // blend launches per frame (host-output banding)

// Per depth-sorted splat: instance count and packed tile rectangle.  The
// per-tile instance counts come for free as a 2D difference array over the
// tile grid (4 updates per splat, gx = tiles_x + 1 columns) accumulated in
// shared memory and flushed once per CTA; tile_prep_k integrates it.
__global__ void dup_count_k(const uint32_t* __restrict__ vals, const uint2* __restrict__ box,
                            const RenderCounters* __restrict__ ctr, int shift, int gx, int gy,
                            uint32_t* __restrict__ cnt, uint32_t* __restrict__ rects,
                            uint32_t* __restrict__ tdiff) {
  pdl_wait();
  extern __shared__ uint32_t sdiff[];
  const int cells = gx * gy;
  const bool local = cells <= kDiffSmemWords;
  uint32_t* d = local ? sdiff : tdiff;
  if (local) {
    for (int i = threadIdx.x; i < cells; i += blockDim.x) sdiff[i] = 0u;
    __syncthreads();
  }
  const uint32_t n = ctr->n_kept;
  // tile rectangle of the splat's clamped pixel box, inclusive tile bounds
  // packed tx0 | tx1 << 8 | ty0 << 16 | ty1 << 24 (tile grids up to 256 x 256)
  auto one = [&](uint32_t s, uint32_t bx, uint32_t by) {
    const int x0 = bx & 0xFFFF, x1 = bx >> 16, y0 = by & 0xFFFF, y1 = by >> 16;
    const int tx0 = x0 >> shift, tx1 = (x1 - 1) >> shift, ty0 = y0 >> shift, ty1 = (y1 - 1) >> shift;
    cnt[s] = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
    rects[s] = (uint32_t)tx0 | ((uint32_t)tx1 << 8) | ((uint32_t)ty0 << 16) | ((uint32_t)ty1 << 24);
    atomicAdd(&d[ty0 * gx + tx0], 1u);
    atomicAdd(&d[ty0 * gx + tx1 + 1], 0xFFFFFFFFu);
    atomicAdd(&d[(ty1 + 1) * gx + tx0], 0xFFFFFFFFu);
    atomicAdd(&d[(ty1 + 1) * gx + tx1 + 1], 1u);
  };
  // two splats per thread per step: both gathers in flight together, each an
  // 8-byte box word pair (the preprocess writes them beside the 48-byte
  // records, so this gather touches a sixth of the bytes)
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (; s + stride < n; s += 2 * stride) {
    const uint2 b0 = box[vals[s]], b1 = box[vals[s + stride]];
    one(s, b0.x, b0.y);
    one(s + stride, b1.x, b1.y);
  }
  if (s < n) {
    const uint2 b0 = box[vals[s]];
    one(s, b0.x, b0.y);
  }
  if (local) {
    __syncthreads();
    for (int i = threadIdx.x; i < cells; i += blockDim.x)
      if (sdiff[i]) atomicAdd(&tdiff[i], sdiff[i]);
  }
}

// One CTA, once per frame: integrates the difference array into per-tile
// instance counts, and from them derives everything the tile stage needs
// without touching the instances: the [start, end) range of every tile's
// list (exclusive scan), the overflow decision, the digit histograms of both
// tile-sort radix passes (their "upsweep"), and the blend schedule
// (band-major, longest list first, bucketed by floor(log2(length))).
__global__ void __launch_bounds__(1024) tile_prep_k(
    const uint32_t* __restrict__ tdiff, int tiles_x, int tiles_y, int bands, uint32_t m_cap,
    RenderCounters* __restrict__ ctr, uint32_t* __restrict__ tcount,
    uint32_t* __restrict__ ranges, uint32_t* __restrict__ order, uint32_t* __restrict__ rcounters,
    uint32_t* __restrict__ ghist, const FrameDev* __restrict__ fd) {
  pdl_wait();
  __shared__ uint32_t h[2][256];
  __shared__ uint32_t scratch[33];
  __shared__ uint32_t hist[33 * kMaxBands];
  __shared__ uint32_t base[33 * kMaxBands];
  extern __shared__ uint32_t sgrid[];  // the difference array, when it fits
  const int gx = tiles_x + 1, gy = tiles_y + 1;
  const uint32_t n_tiles = (uint32_t)tiles_x * tiles_y;
  const bool in_smem = gx * gy <= kDiffSmemWords;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) (&h[0][0])[i] = 0u;
  for (int i = threadIdx.x; i < 33 * kMaxBands; i += blockDim.x) hist[i] = 0u;
  if (threadIdx.x < 64) rcounters[threadIdx.x] = 0u;
  // integrate the difference array (rows, then columns) in shared memory
  // (global memory for tile grids too large for it), then publish tcount
  uint32_t* g = in_smem ? sgrid : const_cast<uint32_t*>(tdiff);
  if (in_smem) {
    for (int i = threadIdx.x; i < gx * gy; i += blockDim.x) sgrid[i] = tdiff[i];
    __syncthreads();
  }
  for (int y = threadIdx.x; y < tiles_y; y += blockDim.x) {
    uint32_t run = 0;
    for (int x = 0; x < tiles_x; ++x) {
      run += g[y * gx + x];
      g[y * gx + x] = run;
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < tiles_x; x += blockDim.x) {
    uint32_t run = 0;
    for (int y = 0; y < tiles_y; ++y) {
      run += g[y * gx + x];
      g[y * gx + x] = run;
    }
  }
  __syncthreads();
  for (uint32_t t = threadIdx.x; t < n_tiles; t += blockDim.x)
    tcount[t] = g[(t / tiles_x) * gx + t % tiles_x];
  __syncthreads();
  // exclusive scan over tiles -> ranges; each thread a contiguous run
  const uint32_t per = (n_tiles + blockDim.x - 1) / blockDim.x;
  const uint32_t t0 = threadIdx.x * per, t1 = min(n_tiles, t0 + per);
  uint32_t local = 0;
  for (uint32_t t = t0; t < t1; ++t) local += tcount[t];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = lane < (int)(blockDim.x / 32) ? scratch[lane] : 0u;
    uint32_t wi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    scratch[lane] = wi - v;
    if (lane == 31) scratch[32] = wi;
  }
  __syncthreads();
  uint32_t run = scratch[warp] + inc - local;
  const uint32_t total = scratch[32];
  for (uint32_t t = t0; t < t1; ++t) {
    const uint32_t c = tcount[t];
    ranges[2 * t] = run;
    ranges[2 * t + 1] = run + c;
    run += c;
    if (c) {
      atomicAdd(&h[0][t & 255u], c);
      atomicAdd(&h[1][(t >> 8) & 255u], c);
    }
  }
  if (threadIdx.x == 0) {
    // total == ctr->n_inst (the scan of per-splat counts)
    ctr->n_need = total;
    if (total > m_cap) {
      ctr->overflow = 1;
      ctr->n_inst = 0;  // no lists: blend_k takes the spill path
    }
    uint32_t* hc = fd ? fd->counters_host : nullptr;
    if (hc) {
      hc[0] = ctr->n_kept;
      hc[1] = ctr->n_inst;
      hc[2] = ctr->overflow;
      hc[3] = total;
    }
  }
  // schedule
  auto key = [&](uint32_t t) -> int {
    const uint32_t len = tcount[t];
    // the band whose rows [blend_band_row(b), blend_band_row(b + 1)) hold t
    const int band = (((int)(t / tiles_x) + 1) * bands - 1) / tiles_y;
    return band * 33 + (len ? __clz(len) : 32);  // descending length within the band
  };
  for (uint32_t t = threadIdx.x; t < n_tiles; t += blockDim.x) atomicAdd(&hist[key(t)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) ghist[i] = (&h[0][0])[i];
  if (threadIdx.x == 0) {
    uint32_t r = 0;
    for (int b = 0; b < 33 * bands; ++b) {
      base[b] = r;
      r += hist[b];
    }
  }
  __syncthreads();
  for (uint32_t t = threadIdx.x; t < n_tiles; t += blockDim.x) order[atomicAdd(&base[key(t)], 1u)] = t;
}

// Load-balanced expansion: each CTA owns contiguous runs of kEmitChunk
// output instances (depth-sorted splats emit their tile rectangles in order;
// near splats can cover thousands of tiles, so the split is by instances,
// not by splats).  The splats covering a run are found with a warp-parallel
// 32-ary search over the exclusive offsets (a handful of L2 round trips),
// staged in shared memory, and every thread writes consecutive instances
// (coalesced).  Also clears the look-back status words of the tile-sort
// passes (sized by the frame's instance count).
constexpr int kEmitChunk = 2048;
constexpr int kEmitThreads = 256;

__device__ __forceinline__ uint32_t last_le(const uint32_t* a, uint32_t n, uint32_t x) {
  // largest j < n with a[j] <= x (a ascending, a[0] <= x)
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// The same search by one warp over global memory, 32 pivots per round.
__device__ __forceinline__ uint32_t warp_last_le(const uint32_t* __restrict__ a, uint32_t n,
                                                 uint32_t x) {
  const int lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t piv = lo + (uint32_t)lane * step;
    const bool le = piv < hi && a[piv] <= x;
    const uint32_t b = __ballot_sync(0xffffffffu, le);  // a prefix of lanes (a ascending)
    const uint32_t last = 31 - __clz(b);                  // lane 0 always holds (a[lo] <= x)
    lo = lo + last * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

__global__ void __launch_bounds__(kEmitThreads) dup_emit_k(
    const uint32_t* __restrict__ vals, const uint32_t* __restrict__ rects,
    const uint32_t* __restrict__ off, const RenderCounters* __restrict__ ctr, int tiles_x,
    uint32_t* __restrict__ tk, uint32_t* __restrict__ tv, uint32_t* __restrict__ status,
    size_t pass_stride, uint32_t tile_items) {
  pdl_wait();
  __shared__ uint32_t soff[kEmitChunk + 1];
  __shared__ uint2 sinfo[kEmitChunk];  // g, tx0 | ty0 << 8 | tiles across << 16
  __shared__ uint32_t span[2];
  const uint32_t n = ctr->n_kept, m = ctr->n_inst;
  const size_t used = (size_t)((m + tile_items - 1) / tile_items) * 256;
  for (size_t i = blockIdx.x * (size_t)kEmitThreads + threadIdx.x; i < used;
       i += (size_t)gridDim.x * kEmitThreads) {
    status[i] = 0u;
    status[pass_stride + i] = 0u;
  }
  if (m == 0 || n == 0) return;  // no instances, or overflow (spill blend)
  const int warp = threadIdx.x >> 5;
  for (uint32_t i0 = blockIdx.x * kEmitChunk; i0 < m; i0 += gridDim.x * kEmitChunk) {
    const uint32_t i1 = min(m, i0 + kEmitChunk);
    if (warp < 2) {
      const uint32_t r = warp_last_le(off, n, warp == 0 ? i0 : i1 - 1);
      if ((threadIdx.x & 31) == 0) span[warp] = r;
    }
    __syncthreads();
    const uint32_t s0 = span[0], ns = span[1] - s0 + 1;  // <= kEmitChunk: each has >= 1
    for (uint32_t j = threadIdx.x; j < ns; j += kEmitThreads) {
      const uint32_t rc = rects[s0 + j];
      const uint32_t tx0 = rc & 0xFF, tx1 = (rc >> 8) & 0xFF, ty0 = (rc >> 16) & 0xFF;
      soff[j] = off[s0 + j];
      sinfo[j] = make_uint2(vals[s0 + j], tx0 | (ty0 << 8) | ((tx1 - tx0 + 1) << 16));
    }
    __syncthreads();
    for (uint32_t i = i0 + threadIdx.x; i < i1; i += kEmitThreads) {
      const uint32_t j = last_le(soff, ns, i);
      const uint2 inf = sinfo[j];
      const uint32_t k = i - soff[j], wd = inf.y >> 16;
      const uint32_t ty = ((inf.y >> 8) & 0xFF) + k / wd, tx = (inf.y & 0xFF) + k % wd;
      tk[i] = ty * (uint32_t)tiles_x + tx;
      tv[i] = inf.x;
    }
    __syncthreads();
  }
}

// Blend: one CTA per 16x16 sub-tile of a TS x TS sort tile ((TS/16)^2 CTAs
// share one tile list), one thread per pixel, each warp an 8x4 pixel block.
// Splats of the list are staged 256 at a time: each staging thread tests its
// splat against the CTA's sub-tile and a warp-ballot compaction keeps the
// overlapping ones (in list order) in shared memory.  Each warp then walks
// the staged splats 32 at a time, ballots which of them touch its own 8x4
// block, and iterates only those - warp-uniform control flow, no per-splat
// work for warps the splat misses.  Exact mode stages the splat parameters
// widened to FP64 and evaluates exp with a table-driven FP64 kernel (64-entry
// double-double table, degree-5 polynomial: <= 0.82 ulp, tested against
// libm on 2e7 points), the reference's arithmetic otherwise.
struct SplatF64 {
  double cx, cy, ca, cb2, cc, al, r, g, b;
  double skip;  // sigma below which alpha * exp(sigma) < 2^-36 (no effect on f32 T)
  int x0, xw, y0, yh;  // clamped box: [x0, x0 + xw) x [y0, y0 + yh)
  // 104-byte stride (26 banks): lanes loading the same field of different
  // staged splats (lane lists) collide only 16 splats apart, not 4 (96 B)
  int pad_[2];
};

// 2^(j/64) as double-double, j = 0..63
__constant__ double2 kExp2Tab[64];

// FP64 constants of the exact blend in the constant bank: DFMA/DMUL/DSETP
// take them as c[][] operands, where literals that do not fit an immediate
// would be rematerialised with uniform moves on every pixel-splat.
constexpr float kStopF = 0x1.010102p-8f;  // RN32(1/255) = smallest float >= 1/255
// certified fast blend: the colour error an unflagged pixel may carry (the
// contract is 1e-3 max-abs against the reference)
constexpr float kCertTol = 9e-4f;
// VMSPLAT_CERT_ALL=1: flag every pixel (tests re-blend the whole image in
// FP64 through the repair kernel)
__device__ int g_cert_all = 0;
__device__ uint32_t g_cert_why[4];
constexpr int kPairStep = 2;  // splats whose box tests and sigmas are evaluated together
// exact blend: per-pixel splat walks (VMSPLAT_LANE_LISTS: 0 off - the dense
// warp walk; 1 for groups of small splats saving more than g_lane_margin
// steps; 2, the default, every group)
__device__ int g_lane_lists = 2;
__device__ int g_lane_margin = 2;

__constant__ double kBlendC[10] = {
    0x1.71547652b82fep+6,   // 0: 64 / ln2
    0x1.8p52,               // 1: round-to-integer magic
    -0x1.62e4200000000p-7,  // 2: -ln2/64, 21 leading bits (k * kLhi exact)
    -0x1.fdf473de6af28p-28, // 3: -(ln2/64 - kLhi)
    1.0 / 120.0,            // 4
    1.0 / 24.0,             // 5
    1.0 / 6.0,              // 6
    1.0 / 255.0,            // 7: stop threshold (_core.pyx:60)
    0.99,                   // 8: weight clamp (_core.pyx:70)
    0.5,                    // 9
};

// tab[j * S] = 2^(j/64): S = 1 (one table), or S = 8 (eight interleaved
// copies, the caller passing copy lane % 8: a 128-bit shared load is served
// 8 lanes at a time, and entry j of copy c sits in banks 4c..4c+3 for every
// j, so per-lane table lookups never conflict)
template <int S = 1>
__device__ __forceinline__ double exp_tab(double x, const double2* __restrict__ tab) {
  // exp(x), x in [-700, 0]: x = (64 m + j) ln2/64 + r, |r| <= ln2/128
  const double t = __fma_rn(x, kBlendC[0], kBlendC[1]);
  const int k = __double2loint(t);
  const double kd = __dsub_rn(t, kBlendC[1]);
  double r = __fma_rn(kd, kBlendC[2], x);
  r = __fma_rn(kd, kBlendC[3], r);
  double q = __fma_rn(kBlendC[4], r, kBlendC[5]);
  q = __fma_rn(q, r, kBlendC[6]);
  q = __fma_rn(q, r, kBlendC[9]);
  q = __fma_rn(q, r, 1.0);
  const double sr = __dmul_rn(q, r);  // exp(r) - 1
  const double2 tj = tab[(k & 63) * S];
  const double v = __dadd_rn(tj.x, __fma_rn(tj.x, sr, tj.y));
  return __hiloint2double(__double2hiint(v) + ((k >> 6) << 20), __double2loint(v));
}

// The exact blend's exp, exposed for its accuracy test (vms_debug_exp).
__global__ void exp_eval_k(const double* __restrict__ x, uint64_t n, double* __restrict__ out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = exp_tab(x[i], kExp2Tab);
}

// Optional per-CTA timing trace for schedule studies (vms_debug_blend_trace):
// 8 u64 per CTA: globaltimer at start and end, SM id, list length << 32 |
// tile, then 4 zero words.
__device__ unsigned long long* g_blend_trace = nullptr;

// Tile-instance overflow (the frame needs more instances than the buffer
// holds): the tile lists were not built, and every CTA walks the whole
// depth-sorted splat list `vals` instead, filtering by its own sub-tile - the
// same per-tile order, so the image is identical, only slower.  The host
// sees the overflow counter afterwards and grows the buffer for later frames.
// kSparse (exact mode): the splats of a warp's group are processed splat-
// parallel instead of pixel-parallel - lane k evaluates the weights of splat
// k of the group over the pixels of its box inside the warp's 8x4 block
// (skipping saturated pixels) into shared memory, a ballot transpose gives
// every pixel the (list-ordered) mask of splats with a live weight for it,
// and each lane then applies only those, in list order.  Same arithmetic,
// same order per pixel - only the lanes' work assignment changes: small
// splats (the vanishing-point tiles' long lists) no longer occupy all 32
// lanes for the few pixels they touch.
constexpr int kSparseGroup = 16;   // splats per weight pass (shared-memory budget)
constexpr int kSparseRow = 33;     // padded row of doubles (bank spread)
constexpr size_t kSparseSmem = sizeof(double) * (kBlendThreads / 32) * kSparseGroup * kSparseRow;

template <bool kExact, int TS, bool kSparse = false>
__global__ void __launch_bounds__(kBlendThreads, kSparse ? 3 : 4) blend_k(const uint32_t* __restrict__ ranges,
                                                         const uint32_t* __restrict__ order,
                                                         const uint32_t* __restrict__ tv_tiles,
                                                         const uint32_t* __restrict__ vals,
                                                         const RenderCounters* __restrict__ ctr,
                                                         const BlendRec* __restrict__ rec,
                                                         int w, int h, int tiles_x,
                                                         uint32_t order_offset,
                                                         float* image_arg,
                                                         const FrameDev* __restrict__ fd,
                                                         int accumulate,
                                                         const uint32_t* __restrict__ tile_hot,
                                                         uint32_t* __restrict__ cert_cnt,
                                                         uint4* __restrict__ cert_list) {
  pdl_wait();
  constexpr int SUB = TS / 16;  // sub-tiles per tile edge
  using Staged = typename std::conditional<kExact, SplatF64, BlendRec>::type;
  __shared__ Staged sp[kBlendThreads];
  __shared__ uint32_t wsum[kBlendThreads / 32];
  __shared__ double2 tab[kExact ? 64 * 8 : 1];
  extern __shared__ double wbuf[];  // kSparse: (warps) x kSparseGroup x kSparseRow
  unsigned long long t_start = 0;
  unsigned long long* trace = g_blend_trace;
  if (trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const int tile = order[order_offset + blockIdx.x / (SUB * SUB)], sub = blockIdx.x % (SUB * SUB);
  if (tile_hot && tile_hot[tile]) return;  // blend_hot_k owns this tile's pixels
  const int sx0 = (tile % tiles_x) * TS + (sub % SUB) * 16;
  const int sy0 = (tile / tiles_x) * TS + (sub / SUB) * 16;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp w: 8x4 block at ((w & 1) * 8, (w >> 1) * 4) of the sub-tile
  const int wx0 = sx0 + (warp & 1) * 8, wy0 = sy0 + (warp >> 1) * 4;
  const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
  const bool inside = px < w && py < h;
  if (kExact)
    for (int t = threadIdx.x; t < 64 * 8; t += kBlendThreads) tab[t] = kExp2Tab[t >> 3];
  const double2* __restrict__ tabl = tab + (lane & 7);  // this lane's table copy
  const bool spill = ctr->overflow != 0u;
  const uint32_t start = spill ? 0u : ranges[2 * tile];
  const uint32_t end = spill ? ctr->n_kept : ranges[2 * tile + 1];
  const uint32_t* __restrict__ tv = spill ? vals : tv_tiles;
  float* __restrict__ image = image_arg ? image_arg : fd->image;
  // a pixel is finished once T < 1/255 (the reference's stop test, exactly:
  // for f32 T, T < 1/255 in FP64 <=> T < RN32(1/255)); pixels outside the
  // image start finished
  float cr = 0.f, cg = 0.f, cb = 0.f, T = inside ? 1.f : 0.f;
  if (accumulate && inside) {
    const float* p = image + ((size_t)py * w + px) * 3;
    cr = p[0];
    cg = p[1];
    cb = p[2];
  }
  // certified fast blend (kExact == false, cert_cnt set): E bounds the
  // relative error of T against the reference's FP64 arithmetic, C the
  // colour error; a pixel whose stop decision (T < 1/255) or colour the
  // bounds cannot certify is re-blended in FP64 by blend_repair_k
  const float cr0 = cr, cg0 = cg, cb0 = cb;
  float certE = 0.f, certC = 0.f;
  uint32_t certN = 0;
  bool certFlag = false;
  const double fx = (double)px + 0.5, fy = (double)py + 0.5;
  // the batch loop's one end-of-batch barrier also decides the early exit
  // (every pixel of the sub-tile finished); the first batch always runs
  for (uint32_t base = start; base < end; base += kBlendThreads) {
    const uint32_t i = base + threadIdx.x;
    bool hit = false;
    BlendRec r;
    if (i < end) {
      r = rec[tv[i]];
      const int x0 = r.bx & 0xFFFF, x1 = r.bx >> 16, y0 = r.by & 0xFFFF, y1 = r.by >> 16;
      hit = x0 < sx0 + 16 && x1 > sx0 && y0 < sy0 + 16 && y1 > sy0;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    uint32_t pre = 0, cnt = 0;
#pragma unroll
    for (int k = 0; k < kBlendThreads / 32; ++k) {
      const uint32_t c = wsum[k];
      pre += k < warp ? c : 0u;
      cnt += c;
    }
    if (hit) {
      const uint32_t o = pre + __popc(bal & lanemask_lt());
      if constexpr (kExact) {
        SplatF64 d;
        d.cx = r.cx;
        d.cy = r.cy;
        // sigma's -0.5 folded into the conic: power-of-two scalings are exact
        d.ca = -0.5 * (double)r.ca;
        d.cb2 = -(double)r.cb;
        d.cc = -0.5 * (double)r.cc;
        d.al = r.alpha;
        d.skip = r.skip;
        d.r = r.r;
        d.g = r.g;
        d.b = r.b;
        d.x0 = r.bx & 0xFFFF;
        d.xw = (int)(r.bx >> 16) - d.x0;
        d.y0 = r.by & 0xFFFF;
        d.yh = (int)(r.by >> 16) - d.y0;
        sp[o] = d;
      } else {
        sp[o] = r;
      }
    }
    __syncthreads();
    // this warp: the staged splats touching its 8x4 block, 32 at a time
    for (uint32_t c0 = 0; c0 < cnt && !__all_sync(0xffffffffu, T < kStopF); c0 += 32) {
      bool mine = false;
      if (c0 + lane < cnt) {
        const Staged& q = sp[c0 + lane];
        int x0, x1, y0, y1;
        if constexpr (kExact) {
          x0 = q.x0; x1 = q.x0 + q.xw; y0 = q.y0; y1 = q.y0 + q.yh;
        } else {
          x0 = q.bx & 0xFFFF; x1 = q.bx >> 16; y0 = q.by & 0xFFFF; y1 = q.by >> 16;
        }
        mine = x0 < wx0 + 8 && x1 > wx0 && y0 < wy0 + 4 && y1 > wy0;
      }
      uint32_t m = __ballot_sync(0xffffffffu, mine);
      const Staged* __restrict__ grp = sp + c0;
      if constexpr (kExact && kSparse) {
        double* __restrict__ wrow = wbuf + warp * (kSparseGroup * kSparseRow);
        for (int g0 = 0; g0 < 32 && (m >> g0); g0 += kSparseGroup) {
          const uint32_t gm = (m >> g0) & ((1u << kSparseGroup) - 1u);
          if (!gm) continue;
          // saturated (or off-image) pixels of the block: lane = pixel
          const uint32_t done = __ballot_sync(0xffffffffu, T < kStopF);
          if (done == 0xffffffffu) break;
          // weight pass: lane l owns splat g0 + (l & 15) over block rows
          // 2 (l >> 4) and 2 (l >> 4) + 1
          uint32_t pm = 0;
          const int k = lane & (kSparseGroup - 1), half = lane >> 4;
          if ((gm >> k) & 1u) {
            const Staged& q = grp[g0 + k];
            const int bx0 = max(q.x0 - wx0, 0), bx1 = min(q.x0 + q.xw - wx0, 8);
            const int by0 = max(q.y0 - wy0, 2 * half), by1 = min(q.y0 + q.yh - wy0, 2 * half + 2);
            double* __restrict__ row = wrow + k * kSparseRow;
            for (int yy = by0; yy < by1; ++yy) {
              const double fyq = (double)(wy0 + yy) + 0.5;
              const double dy = __dsub_rn(fyq, q.cy);
              const double syy = __dmul_rn(__dmul_rn(q.cc, dy), dy);
              const double sxy = __dmul_rn(q.cb2, dy);
              for (int xx = bx0; xx < bx1; ++xx) {
                const int pbit = yy * 8 + xx;
                if ((done >> pbit) & 1u) continue;
                const double dx = __dsub_rn((double)(wx0 + xx) + 0.5, q.cx);
                // the dense loop's sigma: ((a dx) dx + (2b dy) dx) + (c dy) dy
                const double sg = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(q.ca, dx), dx),
                                                      __dmul_rn(sxy, dx)),
                                            syy);
                if (sg < q.skip) continue;
                double wk = __dmul_rn(q.al, exp_tab<8>(sg, tabl));
                if (wk > kBlendC[8]) wk = kBlendC[8];
                row[pbit] = wk;
                pm |= 1u << pbit;
              }
            }
          }
          // transpose: this lane's pixel gets the mask of splats with a live
          // weight for it (bit k = splat g0 + k: list order = bit order); a
          // pixel's bits come from one half of the lanes only
          uint32_t mine_w = 0;
#pragma unroll
          for (int pbit = 0; pbit < 32; ++pbit) {
            const uint32_t b = __ballot_sync(0xffffffffu, (pm >> pbit) & 1u);
            if (lane == pbit) mine_w = (b | (b >> 16)) & 0xFFFFu;
          }
          __syncwarp();
          while (mine_w) {
            const int j = __ffs(mine_w) - 1;
            mine_w &= mine_w - 1;
            if (T < kStopF) break;
            const Staged& q = grp[g0 + j];
            const double wgt = wrow[j * kSparseRow + lane];
            const double t = (double)T;
            const double wt = __dmul_rn(wgt, t);
            cr = __double2float_rn(__dadd_rn((double)cr, __dmul_rn(wt, q.r)));
            cg = __double2float_rn(__dadd_rn((double)cg, __dmul_rn(wt, q.g)));
            cb = __double2float_rn(__dadd_rn((double)cb, __dmul_rn(wt, q.b)));
            T = __double2float_rn(__dmul_rn(t, __dsub_rn(1.0, wgt)));
          }
          __syncwarp();
        }
      } else if constexpr (kExact) {
        // two splats per step: their box tests and sigmas (independent of T)
        // are evaluated together, so rejections - most of the walk for pixels
        // that never saturate - overlap; the exp and the T/colour updates then
        // run in list order.
        auto sigma = [&](const Staged& q, bool& live) -> double {
          const bool in = ((unsigned)(px - q.x0) < (unsigned)q.xw) &
                          ((unsigned)(py - q.y0) < (unsigned)q.yh);
          const double dx = __dsub_rn(fx, q.cx);
          const double dy = __dsub_rn(fy, q.cy);
          const double sg = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(q.ca, dx), dx),
                                                __dmul_rn(__dmul_rn(q.cb2, dy), dx)),
                                      __dmul_rn(__dmul_rn(q.cc, dy), dy));
          // weight < 2^-36 (sigma below the staged threshold): T is unchanged
          // bit for bit and the colour moves by < 2^-36 - no effect
          live = in & (sg >= q.skip);
          return sg;
        };
        auto apply = [&](const Staged& q, double wgt) {
          const double t = (double)T;
          const double wt = __dmul_rn(wgt, t);
          cr = __double2float_rn(__dadd_rn((double)cr, __dmul_rn(wt, q.r)));
          cg = __double2float_rn(__dadd_rn((double)cg, __dmul_rn(wt, q.g)));
          cb = __double2float_rn(__dadd_rn((double)cb, __dmul_rn(wt, q.b)));
          T = __double2float_rn(__dmul_rn(t, __dsub_rn(1.0, wgt)));
        };
        auto blend = [&](const Staged& q, double sg) {
          // _core.pyx:56-78: FP64 arithmetic, f32 storage of T and colour
          const double t = (double)T;
          double wgt = __dmul_rn(q.al, exp_tab<8>(sg, tabl));
          if (wgt > kBlendC[8]) wgt = kBlendC[8];
          const double wt = __dmul_rn(wgt, t);
          cr = __double2float_rn(__dadd_rn((double)cr, __dmul_rn(wt, q.r)));
          cg = __double2float_rn(__dadd_rn((double)cg, __dmul_rn(wt, q.g)));
          cb = __double2float_rn(__dadd_rn((double)cb, __dmul_rn(wt, q.b)));
          T = __double2float_rn(__dmul_rn(t, __dsub_rn(1.0, wgt)));
        };
        // Lane lists for groups of small splats (the far splats of the long,
        // vanishing-point lists cover a few lanes of the 8x4 block each): the
        // group's boxes become per-pixel bit sets (8 column and 4 row
        // ballots), and every lane walks only the splats covering its pixel,
        // in list order - max over lanes of popc(own) steps instead of
        // popc(m), same arithmetic per pixel-splat, so the same image.
        if (g_lane_lists) {
          const bool in_m = (m >> lane) & 1u;
          int cl = 0, ch = 0, rl = 0, rh = 0;
          if (in_m) {
            const Staged& q = grp[lane];
            cl = max(q.x0 - wx0, 0);
            ch = min(q.x0 + q.xw - wx0, 8);
            rl = max(q.y0 - wy0, 0);
            rh = min(q.y0 + q.yh - wy0, 4);
          }
          const uint32_t area = __reduce_add_sync(0xffffffffu, (uint32_t)((ch - cl) * (rh - rl)));
          const uint32_t nm = __popc(m);
          const bool force = g_lane_lists >= 2;  // every group
          if (force || area * 4u < nm * 3u * 32u) {  // mean coverage below 3/4 of the block
            const int cx = lane & 7, ry = lane >> 3;
            uint32_t colw = 0, roww = 0;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint32_t b = __ballot_sync(0xffffffffu, cl <= c && c < ch);
              colw = cx == c ? b : colw;
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const uint32_t b = __ballot_sync(0xffffffffu, rl <= r && r < rh);
              roww = ry == r ? b : roww;
            }
            uint32_t own = colw & roww;  // group splats whose box holds this pixel
            const uint32_t steps =
                __reduce_max_sync(0xffffffffu, T >= kStopF ? (uint32_t)__popc(own) : 0u);
            if (force || steps + (uint32_t)g_lane_margin < nm) {
              auto sig = [&](const Staged& q) -> double {
                const double dx = __dsub_rn(fx, q.cx);
                const double dy = __dsub_rn(fy, q.cy);
                return __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(q.ca, dx), dx),
                                           __dmul_rn(__dmul_rn(q.cb2, dy), dx)),
                                 __dmul_rn(__dmul_rn(q.cc, dy), dy));
              };
              while (own && T >= kStopF) {
                const int j0 = __ffs(own) - 1;
                own &= own - 1;
                const bool two = own != 0u;
                const int j1 = two ? __ffs(own) - 1 : j0;
                own &= two ? own - 1 : own;
                const Staged& q0 = grp[j0];
                const Staged& q1 = grp[j1];
                const double s0 = sig(q0), s1 = sig(q1);
                const bool l0 = s0 >= q0.skip, l1 = two && s1 >= q1.skip;
                double w0 = __dmul_rn(q0.al, exp_tab<8>(l0 ? s0 : 0.0, tabl));
                double w1 = __dmul_rn(q1.al, exp_tab<8>(l1 ? s1 : 0.0, tabl));
                if (w0 > kBlendC[8]) w0 = kBlendC[8];
                if (w1 > kBlendC[8]) w1 = kBlendC[8];
                if (l0) apply(q0, w0);
                if (l1 && T >= kStopF) apply(q1, w1);
              }
              __syncwarp();
              m = 0u;
            }
          }
        }
        while (m) {
          int j[kPairStep];
          int got = 0;
#pragma unroll
          for (int k = 0; k < kPairStep; ++k) {
            j[k] = m ? __ffs(m) - 1 : 0;
            got += m ? 1 : 0;
            m &= m - 1;
          }
          bool l[kPairStep];
          double sg[kPairStep];
#pragma unroll
          for (int k = 0; k < kPairStep; ++k) sg[k] = sigma(grp[j[k]], l[k]);
          bool any = false;
#pragma unroll
          for (int k = 0; k < kPairStep; ++k) any |= k < got && l[k];
          // warp-uniform skip (no lane may leave before the vote)
          if (!__any_sync(0xffffffffu, any && T >= kStopF)) continue;
          // the step's weights (independent of T) together, branch-free
          double wv[kPairStep];
#pragma unroll
          for (int k = 0; k < kPairStep; ++k) {
            const Staged& q = grp[j[k]];
            double wk = __dmul_rn(q.al, exp_tab<8>(l[k] ? sg[k] : 0.0, tabl));
            if (wk > kBlendC[8]) wk = kBlendC[8];
            wv[k] = wk;
          }
#pragma unroll
          for (int k = 0; k < kPairStep; ++k)
            if (k < got && l[k] && T >= kStopF) apply(grp[j[k]], wv[k]);
        }
      }
      while (!kExact && m) {
        const Staged& s = grp[__ffs(m) - 1];
        m &= m - 1;
        if (T < kStopF) continue;
        if constexpr (kExact) {
          // the pixel in the splat's half-open box, as two unsigned range tests
          if (((unsigned)(px - s.x0) >= (unsigned)s.xw) | ((unsigned)(py - s.y0) >= (unsigned)s.yh))
            continue;
          // _core.pyx:56-78: FP64 arithmetic, f32 storage of T and colour
          const double t = (double)T;
          const double dx = __dsub_rn(fx, s.cx);
          const double dy = __dsub_rn(fy, s.cy);
          const double sig = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(s.ca, dx), dx),
                                                 __dmul_rn(__dmul_rn(s.cb2, dy), dx)),
                                       __dmul_rn(__dmul_rn(s.cc, dy), dy));
          // weight < 2^-36: T is unchanged bit for bit and the colour moves by
          // < 2^-36 (far tails of elongated splats) - skip the exp
          if (sig < s.skip) continue;
          double wgt = __dmul_rn(s.al, exp_tab<8>(sig, tabl));
          if (wgt > kBlendC[8]) wgt = kBlendC[8];
          const double wt = __dmul_rn(wgt, t);
          cr = __double2float_rn(__dadd_rn((double)cr, __dmul_rn(wt, s.r)));
          cg = __double2float_rn(__dadd_rn((double)cg, __dmul_rn(wt, s.g)));
          cb = __double2float_rn(__dadd_rn((double)cb, __dmul_rn(wt, s.b)));
          T = __double2float_rn(__dmul_rn(t, __dsub_rn(1.0, wgt)));
        } else {
          const int x0 = s.bx & 0xFFFF, x1 = s.bx >> 16, y0 = s.by & 0xFFFF, y1 = s.by >> 16;
          if (px < x0 || px >= x1 || py < y0 || py >= y1) continue;
          const float dx = ((float)px + 0.5f) - s.cx, dy = ((float)py + 0.5f) - s.cy;
          const float adx = s.ca * dx, bdy = s.cb * dy, cdy = s.cc * dy;
          float sig = -0.5f * __fmaf_rn(adx, dx, __fmaf_rn(2.0f * bdy, dx, cdy * dy));
          // S = 0.5 (|a dx dx| + 2 |b dx dy| + |c dy dy|): the size of sigma's
          // terms, which bounds its FP32 rounding error
          float S = 0.f;
          if (cert_cnt) {
            S = 0.5f * __fmaf_rn(fabsf(adx), fabsf(dx),
                                 __fmaf_rn(2.0f * fabsf(bdy), fabsf(dx), fabsf(cdy * dy)));
            if (S > 256.f) {
              // ill-conditioned conic (terms >> sigma: FP32 cancels): sigma
              // in FP64 as the reference evaluates it, then rounded once
              const double ddx = ((double)px + 0.5) - (double)s.cx;
              const double ddy = ((double)py + 0.5) - (double)s.cy;
              const double q = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn((double)s.ca, ddx), ddx),
                                                   __dmul_rn(__dmul_rn(2.0 * (double)s.cb, ddy), ddx)),
                                         __dmul_rn(__dmul_rn((double)s.cc, ddy), ddy));
              sig = (float)(-0.5 * q);
              S = fabsf(sig) + 1.0f;  // one f32 rounding of sigma instead of 4u S
            }
          }
          const float wgt = fminf(s.alpha * __expf(sig), 0.99f);
          const float wt = wgt * T;
          cr = __fmaf_rn(wt, s.r, cr);
          cg = __fmaf_rn(wt, s.g, cg);
          cb = __fmaf_rn(wt, s.b, cb);
          const float om = 1.0f - wgt;
          T = T * om;
          if (cert_cnt) {
            // S = 0.5 (|a dx dx| + 2 |b dx dy| + |c dy dy|) bounds the terms of
            // sigma: dx, dy are exact (Sterbenz: pixel centre and splat centre
            // within a factor of 2, |dx| < 2^12), the products and the two
            // fused sums round: |sigma' - sigma| <= 4u S; __expf adds
            // (4 + 2.4 |sigma'|) u, alpha * e and the 0.99f clamp (vs 0.99)
            // 2u -> w is within epsw = (8 S + 8) u relative (margin kept);
            // T's relative error grows by epsw w / (1 - w) + 4u per step
            const float epsw = __fmaf_rn(S, 8.0f * 0x1p-24f, 8.0f * 0x1p-24f);
            certC = __fmaf_rn(wt * fmaxf(s.r, fmaxf(s.g, s.b)), epsw + certE + 0x1p-22f, certC);
            certE = __fdividef(epsw * wgt * 1.02f, om) + (certE + 4.0f * 0x1p-24f);
            ++certN;
            // the next stop test could go the other way
            certFlag |= fabsf(T - kStopF) <= 1.02f * certE * T + 0x1p-40f;
          }
        }
      }
    }
    if (__syncthreads_and(T < kStopF)) break;
  }
  if (cert_cnt && inside) {
    // colour: the accumulated bound plus one f32 ulp per step of the final
    // value (colours are >= 0, so every partial sum is below it)
    const float cm = fmaxf(cr, fmaxf(cg, cb));
    const bool colour = __fmaf_rn((float)certN * 0x1p-23f, cm, certC) > kCertTol;
    if (g_cert_all > 1) {  // diagnostics (VMSPLAT_CERT_ALL=2): flag reasons
      if (certFlag) atomicAdd(&g_cert_why[0], 1u);
      if (colour) atomicAdd(&g_cert_why[1], 1u);
      if (certN > 2000) atomicAdd(&g_cert_why[2], 1u);
      if (certE > 1e-3f) atomicAdd(&g_cert_why[3], 1u);
    }
    certFlag |= colour;
    if (certFlag || g_cert_all == 1) {
      const uint32_t k = atomicAdd(cert_cnt, 1u);
      cert_list[k] = make_uint4((uint32_t)(py * w + px), __float_as_uint(cr0),
                                __float_as_uint(cg0), __float_as_uint(cb0));
    }
  }
  // output: the 16x16 block goes through shared memory and out as whole
  // rows of 16-byte stores (coalesced; with a zero-copy host image these are
  // full PCIe writes instead of scattered 4-byte ones)
  __shared__ __align__(16) float obuf[16][48];
  const int lx = px - sx0, ly = py - sy0;
  obuf[ly][3 * lx + 0] = cr;
  obuf[ly][3 * lx + 1] = cg;
  obuf[ly][3 * lx + 2] = cb;
  __syncthreads();
  if ((w & 3) == 0 && sx0 + 16 <= w) {
    for (int k = threadIdx.x; k < 16 * 12; k += kBlendThreads) {
      const int row = k / 12, c4 = k - row * 12, y = sy0 + row;
      if (y < h)
        *reinterpret_cast<float4*>(image + ((size_t)y * w + sx0) * 3 + 4 * c4) =
            *reinterpret_cast<const float4*>(&obuf[row][4 * c4]);
    }
  } else if (inside) {
    float* p = image + ((size_t)py * w + px) * 3;
    p[0] = cr;
    p[1] = cg;
    p[2] = cb;
  }
  if (trace) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      unsigned long long* o = trace + 8 * ((size_t)order_offset * SUB * SUB + blockIdx.x);
      o[0] = t_start;
      o[1] = t_end;
      o[2] = smid;
      o[3] = ((unsigned long long)(end - start) << 32) | (uint32_t)tile;
      o[4] = o[5] = o[6] = o[7] = 0;
    }
  }
}

// Certified fast blend, second half: every pixel the FP32 blend could not
// certify is re-blended from its initial colour with the exact kernel's
// FP64 arithmetic (the same staged values, sigma order, exp, skip and stop
// rules, in list order - so the pixel equals the exact blend's).  One warp
// per flagged pixel: the lanes take 32 list entries at a time (box test,
// sigma and weight in parallel), then every lane applies the live ones in
// list order to its own copy of the pixel state (broadcast by shuffles),
// until T < 1/255.
template <int TS>
__global__ void __launch_bounds__(kBlendThreads) blend_repair_k(
    const uint32_t* __restrict__ ranges, const uint32_t* __restrict__ tv_tiles,
    const uint32_t* __restrict__ vals, const RenderCounters* __restrict__ ctr,
    const BlendRec* __restrict__ rec, int w, int tiles_x, float* image_arg,
    const FrameDev* __restrict__ fd, const uint32_t* __restrict__ cert_cnt,
    const uint4* __restrict__ cert_list) {
  pdl_wait();
  __shared__ double2 tab[64];
  if (threadIdx.x < 64) tab[threadIdx.x] = kExp2Tab[threadIdx.x];
  __syncthreads();
  const uint32_t n = *cert_cnt;
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (kBlendThreads / 32);
  float* __restrict__ image = image_arg ? image_arg : fd->image;
  const bool spill = ctr->overflow != 0u;
  for (uint32_t k = blockIdx.x * (kBlendThreads / 32) + (threadIdx.x >> 5); k < n; k += warps) {
    const uint4 e = cert_list[k];
    const int px = (int)(e.x % (uint32_t)w), py = (int)(e.x / (uint32_t)w);
    const int tile = (py / TS) * tiles_x + px / TS;
    const uint32_t start = spill ? 0u : ranges[2 * tile];
    const uint32_t end = spill ? ctr->n_kept : ranges[2 * tile + 1];
    const uint32_t* __restrict__ tv = spill ? vals : tv_tiles;
    float cr = __uint_as_float(e.y), cg = __uint_as_float(e.z), cb = __uint_as_float(e.w);
    float T = 1.f;
    const double fx = (double)px + 0.5, fy = (double)py + 0.5;
    // the next chunk's records are in flight while this chunk is evaluated
    BlendRec nq;
    if (start + lane < end) nq = rec[tv[start + lane]];
    for (uint32_t base = start; base < end && T >= kStopF; base += 32) {
      const uint32_t i = base + lane;
      bool live = false;
      double wk = 0.0;
      float r = 0.f, g = 0.f, b = 0.f;
      const BlendRec cq = nq;
      if (base + 32 + lane < end) nq = rec[tv[base + 32 + lane]];
      if (i < end) {
        const BlendRec q = cq;
        const int x0 = q.bx & 0xFFFF, x1 = q.bx >> 16, y0 = q.by & 0xFFFF, y1 = q.by >> 16;
        if (px >= x0 && px < x1 && py >= y0 && py < y1) {
          // blend_k<exact>'s staging (-0.5 folded into the conic) and sigma
          const double ca = -0.5 * (double)q.ca, cb2 = -(double)q.cb, cc = -0.5 * (double)q.cc;
          const double dx = __dsub_rn(fx, (double)q.cx);
          const double dy = __dsub_rn(fy, (double)q.cy);
          const double sg = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(ca, dx), dx),
                                                __dmul_rn(__dmul_rn(cb2, dy), dx)),
                                      __dmul_rn(__dmul_rn(cc, dy), dy));
          if (sg >= (double)q.skip) {
            live = true;
            wk = __dmul_rn((double)q.alpha, exp_tab(sg, tab));
            if (wk > kBlendC[8]) wk = kBlendC[8];
            r = q.r;
            g = q.g;
            b = q.b;
          }
        }
      }
      uint32_t m = __ballot_sync(0xffffffffu, live);
      while (m && T >= kStopF) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const double wgt = __shfl_sync(0xffffffffu, wk, j);
        const double rr = (double)__shfl_sync(0xffffffffu, r, j);
        const double gg = (double)__shfl_sync(0xffffffffu, g, j);
        const double bb = (double)__shfl_sync(0xffffffffu, b, j);
        const double t = (double)T;
        const double wt = __dmul_rn(wgt, t);
        cr = __double2float_rn(__dadd_rn((double)cr, __dmul_rn(wt, rr)));
        cg = __double2float_rn(__dadd_rn((double)cg, __dmul_rn(wt, gg)));
        cb = __double2float_rn(__dadd_rn((double)cb, __dmul_rn(wt, bb)));
        T = __double2float_rn(__dmul_rn(t, __dsub_rn(1.0, wgt)));
      }
    }
    if (lane == 0) {
      float* p = image + ((size_t)py * w + px) * 3;
      p[0] = cr;
      p[1] = cg;
      p[2] = cb;
    }
  }
}

// ---- hot tiles: long lists (a street's vanishing point) ---------------------
// A tile whose list holds >= kHotLen instances is blended by blend_hot_k
// instead: one CTA per 8x4 pixel block (the regular kernel's warp block), so
// the tile's pixels spread over many SMs, and inside the CTA the work of
// one pixel chain is split - 7 producer warps take the list in 32-entry
// chunks (round robin), test each entry's box against the block and compute
// the FP64 weights of the hits for all 32 pixels into a shared-memory ring
// (plus a live-pixel mask per hit), while 1 consumer warp applies them in
// list order (chunk order, then hit order) to its 32 pixels.  The weight and
// the update are the regular kernel's arithmetic, in the same order per
// pixel; only the chain of T/colour updates is serial, and it no longer
// waits for the exp.
// Measured: C2's vanishing-point lists (4-12 K) blend faster in the regular
// kernel; C4's (50-560 K) twice as fast here (profiles/r2)
constexpr uint32_t kHotLen = 32768;
constexpr int kMaxHot = 64;        // tiles per frame on the hot path
constexpr int kHotRing = 6;        // chunks in flight
constexpr int kHotProducers = 7;

struct HotSlot {
  double w[32][32];  // [hit][pixel]
  float col[32][3];
  uint32_t mask[32];
  uint32_t n;
  uint32_t pad_[3];
};

struct HotSmem {
  HotSlot ring[kHotRing];
  SplatF64 stage[kHotProducers][32];
  uint32_t full_seq[kHotRing];   // chunk j in slot j % R is ready: == j + 1
  uint32_t empty_seq[kHotRing];  // chunk j consumed: == j + 1
  uint32_t done;
};
constexpr size_t kHotSmem = sizeof(HotSmem);

// The hot tiles of the frame (list length >= kHotLen, at most kMaxHot, in
// tile order) and a per-tile flag the regular blend skips them by.
__global__ void __launch_bounds__(1024) hot_list_k(const uint32_t* __restrict__ ranges,
                                                   uint32_t n_tiles, uint32_t hot_len,
                                                   const RenderCounters* __restrict__ ctr,
                                                   uint32_t* __restrict__ hot,
                                                   uint32_t* __restrict__ tile_hot) {
  pdl_wait();
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t run;
  const bool ok = ctr->overflow == 0u;
  if (threadIdx.x == 0) run = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t t0 = 0; t0 < n_tiles; t0 += 1024) {
    const uint32_t t = t0 + threadIdx.x;
    bool f = false;
    if (t < n_tiles && ok) f = ranges[2 * t + 1] - ranges[2 * t] >= hot_len;
    const uint32_t bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    uint32_t pre = 0, tot = 0;
    for (int q = 0; q < 32; ++q) {
      pre += q < warp ? wsum[q] : 0u;
      tot += wsum[q];
    }
    const uint32_t rank = run + pre + __popc(bal & lanemask_lt());
    const bool take = f && rank < (uint32_t)kMaxHot;
    if (take) hot[1 + rank] = t;
    if (t < n_tiles) tile_hot[t] = take ? 1u : 0u;
    __syncthreads();
    if (threadIdx.x == 0) run += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) hot[0] = run < (uint32_t)kMaxHot ? run : (uint32_t)kMaxHot;
}

template <int TS>
__global__ void __launch_bounds__(kBlendThreads, 2) blend_hot_k(
    const uint32_t* __restrict__ ranges, const uint32_t* __restrict__ tv,
    const BlendRec* __restrict__ rec, const uint32_t* __restrict__ hot, int w, int h,
    int tiles_x, float* image_arg, const FrameDev* __restrict__ fd, int accumulate) {
  pdl_wait();
  constexpr int SUB = TS / 16;
  constexpr int kItemsPerTile = SUB * SUB * 8;  // 8x4 blocks per tile
  extern __shared__ __align__(16) unsigned char hot_raw[];
  HotSmem& sm = *reinterpret_cast<HotSmem*>(hot_raw);
  __shared__ double2 tab[64];
  volatile uint32_t* full_seq = sm.full_seq;
  volatile uint32_t* empty_seq = sm.empty_seq;
  volatile uint32_t* done = &sm.done;
  if (threadIdx.x < 64) tab[threadIdx.x] = kExp2Tab[threadIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* __restrict__ image = image_arg ? image_arg : fd->image;
  const uint32_t items = hot[0] * (uint32_t)kItemsPerTile;
  for (uint32_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int tile = (int)hot[1 + item / kItemsPerTile];
    const int rem = (int)(item % kItemsPerTile), sub = rem / 8, blk = rem % 8;
    const int sx0 = (tile % tiles_x) * TS + (sub % SUB) * 16;
    const int sy0 = (tile / tiles_x) * TS + (sub / SUB) * 16;
    const int wx0 = sx0 + (blk & 1) * 8, wy0 = sy0 + (blk >> 1) * 4;
    const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
    const uint32_t start = ranges[2 * tile], end = ranges[2 * tile + 1];
    const uint32_t nchunks = (end - start + 31) / 32;
    if (threadIdx.x < kHotRing) {
      full_seq[threadIdx.x] = 0;
      empty_seq[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) *done = 0;
    __syncthreads();
    if (warp == 0) {
      // consumer: lane = pixel of the 8x4 block
      const bool inside = px < w && py < h;
      float cr = 0.f, cg = 0.f, cb = 0.f, T = inside ? 1.f : 0.f;
      if (accumulate && inside) {
        const float* p = image + ((size_t)py * w + px) * 3;
        cr = p[0];
        cg = p[1];
        cb = p[2];
      }
      for (uint32_t j = 0; j < nchunks; ++j) {
        if (__all_sync(0xffffffffu, T < kStopF)) {
          if (lane == 0) *done = 1;
          break;
        }
        const int slot = (int)(j % kHotRing);
        while (full_seq[slot] != j + 1) __nanosleep(32);
        __threadfence_block();
        const HotSlot& S = sm.ring[slot];
        const uint32_t n = S.n;
        for (uint32_t k = 0; k < n; ++k) {
          if (!((S.mask[k] >> lane) & 1u) || T < kStopF) continue;
          // _core.pyx:56-78: FP64 arithmetic, f32 storage of T and colour
          const double wgt = S.w[k][lane];
          const double t = (double)T;
          const double wt = __dmul_rn(wgt, t);
          cr = __double2float_rn(__dadd_rn((double)cr, __dmul_rn(wt, (double)S.col[k][0])));
          cg = __double2float_rn(__dadd_rn((double)cg, __dmul_rn(wt, (double)S.col[k][1])));
          cb = __double2float_rn(__dadd_rn((double)cb, __dmul_rn(wt, (double)S.col[k][2])));
          T = __double2float_rn(__dmul_rn(t, __dsub_rn(1.0, wgt)));
        }
        __syncwarp();
        __threadfence_block();
        if (lane == 0) empty_seq[slot] = j + 1;
      }
      if (lane == 0) *done = 1;
      if (inside) {
        float* p = image + ((size_t)py * w + px) * 3;
        p[0] = cr;
        p[1] = cg;
        p[2] = cb;
      }
    } else {
      // producer p: chunks p, p + 7, ...
      const int pw = warp - 1;
      const double fx = (double)px + 0.5, fy = (double)py + 0.5;
      SplatF64* __restrict__ st = sm.stage[pw];
      for (uint32_t j = (uint32_t)pw; j < nchunks; j += kHotProducers) {
        if (*done) break;
        const int slot = (int)(j % kHotRing);
        if (j >= (uint32_t)kHotRing) {
          bool quit = false;
          while (empty_seq[slot] < j + 1 - kHotRing) {
            if (*done) {
              quit = true;
              break;
            }
            __nanosleep(32);
          }
          if (quit) break;
          __threadfence_block();
        }
        // this chunk's entries touching the block, in list order
        const uint32_t i = start + 32 * j + lane;
        bool hit = false;
        BlendRec r;
        if (i < end) {
          r = rec[tv[i]];
          const int x0 = r.bx & 0xFFFF, x1 = r.bx >> 16, y0 = r.by & 0xFFFF, y1 = r.by >> 16;
          hit = x0 < wx0 + 8 && x1 > wx0 && y0 < wy0 + 4 && y1 > wy0;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          SplatF64 d;
          d.cx = r.cx;
          d.cy = r.cy;
          d.ca = -0.5 * (double)r.ca;
          d.cb2 = -(double)r.cb;
          d.cc = -0.5 * (double)r.cc;
          d.al = r.alpha;
          d.skip = r.skip;
          d.r = r.r;
          d.g = r.g;
          d.b = r.b;
          d.x0 = r.bx & 0xFFFF;
          d.xw = (int)(r.bx >> 16) - d.x0;
          d.y0 = r.by & 0xFFFF;
          d.yh = (int)(r.by >> 16) - d.y0;
          st[__popc(bal & lanemask_lt())] = d;
        }
        __syncwarp();
        HotSlot& S = sm.ring[slot];
        const int nh = __popc(bal);
        for (int k = 0; k < nh; ++k) {
          const SplatF64& q = st[k];
          const bool in = ((unsigned)(px - q.x0) < (unsigned)q.xw) &
                          ((unsigned)(py - q.y0) < (unsigned)q.yh);
          const double dx = __dsub_rn(fx, q.cx);
          const double dy = __dsub_rn(fy, q.cy);
          const double sg = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(q.ca, dx), dx),
                                                __dmul_rn(__dmul_rn(q.cb2, dy), dx)),
                                      __dmul_rn(__dmul_rn(q.cc, dy), dy));
          const bool live = in & (sg >= q.skip);
          const uint32_t lm = __ballot_sync(0xffffffffu, live);
          double wk = 0.0;
          if (lm) {
            wk = __dmul_rn(q.al, exp_tab(live ? sg : 0.0, tab));
            if (wk > kBlendC[8]) wk = kBlendC[8];
          }
          S.w[k][lane] = wk;
          if (lane == 0) {
            S.mask[k] = lm;
            S.col[k][0] = (float)q.r;
            S.col[k][1] = (float)q.g;
            S.col[k][2] = (float)q.b;
          }
        }
        if (lane == 0) S.n = (uint32_t)nh;
        __syncwarp();
        __threadfence_block();
        if (lane == 0) full_seq[slot] = j + 1;
        __syncwarp();
      }
    }
    __syncthreads();
  }
}

__global__ void pack_ordered_k(const float* __restrict__ centers, const float* __restrict__ conics,
                               const float* __restrict__ colors, const float* __restrict__ alphas,
                               const int32_t* __restrict__ bounds, uint32_t n, int w, int h,
                               BlendRec* __restrict__ rec, uint2* __restrict__ box,
                               uint32_t* __restrict__ vals, uint32_t* __restrict__ cnt) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x0 = max(bounds[4 * i + 0], 0), x1 = min(bounds[4 * i + 1], w);
  int y0 = max(bounds[4 * i + 2], 0), y1 = min(bounds[4 * i + 3], h);
  BlendRec o;
  o.cx = centers[2 * i];
  o.cy = centers[2 * i + 1];
  o.ca = conics[3 * i];
  o.cb = conics[3 * i + 1];
  o.cc = conics[3 * i + 2];
  o.r = colors[3 * i];
  o.g = colors[3 * i + 1];
  o.b = colors[3 * i + 2];
  o.alpha = alphas[i];
  o.skip = blend_skip(o.alpha);
  const bool empty = x1 <= x0 || y1 <= y0;
  if (empty) {
    x0 = x1 = y0 = y1 = 0;
  }
  o.bx = (uint32_t)x0 | ((uint32_t)x1 << 16);
  o.by = (uint32_t)y0 | ((uint32_t)y1 << 16);
  rec[i] = o;
  box[i] = make_uint2(o.bx, o.by);
  vals[i] = i;
  cnt[i] = empty ? 0u : 1u;
}

int tile_bits(uint32_t n_tiles) {
  int b = 1;
  while ((1u << b) < n_tiles) ++b;
  return b;
}

void record(void* const* events, int i, bool external, cudaStream_t s) {
  if (events && events[i])
    cudaEventRecordWithFlags(static_cast<cudaEvent_t>(events[i]), s,
                             external ? cudaEventRecordExternal : cudaEventRecordDefault);
}

}  // namespace

// First tile row of band b of `bands` (bands of near-equal height).
int blend_band_row(int b, int bands, int tiles_y) { return (int)((int64_t)b * tiles_y / bands); }

namespace {

// Depth-sorted splat list and tile-sorted instance list of the last render
// (the radix sorts ping-pong a fixed number of passes).
const uint32_t* sorted_vals(const RenderWs& w) { return w.v0; }  // 4 depth passes
const uint32_t* sorted_tiles(const RenderWs& w, uint32_t n_tiles) {
  return ((tile_bits(n_tiles) + 7) / 8) % 2 ? w.tv1 : w.tv0;
}

// Side stream + fork/join events of the hot-tile blend, per device (made
// outside graph capture by blend_init; a launch without them blends every
// tile with the regular kernel - the same image).
struct HotStreams {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
HotStreams g_hot[16];

bool hot_enabled() {
  static const int on = [] {
    const char* e = getenv("VMSPLAT_BLEND_HOT");
    return e && *e ? atoi(e) : 1;
  }();
  return on != 0;
}

uint32_t hot_len() {
  static const uint32_t n = [] {
    const char* e = getenv("VMSPLAT_HOT_LEN");
    return e && *e ? (uint32_t)atoi(e) : kHotLen;
  }();
  return n;
}

int blend_sparse() {
  static const int sparse = [] {
    const char* e = getenv("VMSPLAT_BLEND_SPARSE");
    return e && *e ? atoi(e) : 0;
  }();
  return sparse;
}

// Hot tiles (single-band frames, exact blend): their own kernel on a forked
// stream, concurrent with the regular blend of the other tiles.
bool hot_path(int exact, int bands) {
  int dev = 0;
  cudaGetDevice(&dev);
  return exact && !blend_sparse() && bands == 1 && hot_enabled() && g_hot[dev & 15].side;
}

int32_t launch_band(int width, int height, const uint32_t* vals, const RenderWs& w, float* image,
                    int accumulate, int exact, int band, int bands, cudaStream_t s) {
  const int ts = tile_size();
  const int tiles_x = ceil_div(width, ts), tiles_y = ceil_div(height, ts);
  const uint32_t n_tiles = (uint32_t)tiles_x * tiles_y;
  const int sparse = blend_sparse();
  auto* kern = exact ? (sparse ? (ts == 16 ? blend_k<true, 16, true> : blend_k<true, 32, true>)
                               : (ts == 16 ? blend_k<true, 16> : blend_k<true, 32>))
                     : (ts == 16 ? blend_k<false, 16> : blend_k<false, 32>);
  const uint32_t subs = (uint32_t)(ts / 16) * (ts / 16);
  const int r0 = blend_band_row(band, bands, tiles_y), r1 = blend_band_row(band + 1, bands, tiles_y);
  const uint32_t first = (uint32_t)r0 * tiles_x, count = (uint32_t)(r1 - r0) * tiles_x;
  const size_t dsmem = (exact && sparse) ? kSparseSmem : 0;
  // hot tiles: the list (hot_list_k) was built with the tile lists, so the
  // blend starts as soon as they are ready
  int dev = 0;
  cudaGetDevice(&dev);
  const HotStreams& hs = g_hot[dev & 15];
  const bool hot = hot_path(exact, bands);
  if (hot) {
    VMS_CUDA(cudaEventRecord(hs.fork, s));
    VMS_CUDA(cudaStreamWaitEvent(hs.side, hs.fork, 0));
    auto* hk = ts == 16 ? blend_hot_k<16> : blend_hot_k<32>;
    // one CTA per 8x4 block of every possible hot tile (the blocks past the
    // frame's hot count exit at once): the blocks run concurrently
    hk<<<kMaxHot * (ts / 16) * (ts / 16) * 8, kBlendThreads, kHotSmem, hs.side>>>(
        (const uint32_t*)w.ranges, sorted_tiles(w, n_tiles), (const BlendRec*)w.rec,
        (const uint32_t*)w.hot, width, height, tiles_x, image, (const FrameDev*)w.fd,
        accumulate);
    VMS_CUDA(cudaEventRecord(hs.join, hs.side));
  }
  // fast (FP32) blend: certified, with the FP64 re-blend of the pixels it
  // flags; each band's flags go to the band's own segment of the list
  uint32_t* cert_cnt = exact ? nullptr : w.cert + band;
  uint4* cert_list = exact ? nullptr : w.cert_list + (size_t)r0 * ts * width;
  if (count)
    VMS_CUDA(launch(kern, count * subs, kBlendThreads, dsmem, s, (const uint32_t*)w.ranges,
                    (const uint32_t*)w.order, sorted_tiles(w, n_tiles), vals,
                    (const RenderCounters*)w.ctr, (const BlendRec*)w.rec, width, height, tiles_x,
                    first, image, (const FrameDev*)w.fd, accumulate,
                    (const uint32_t*)(hot ? w.tile_hot : nullptr), cert_cnt, cert_list));
  mark("blend", s);
  if (hot) VMS_CUDA(cudaStreamWaitEvent(s, hs.join, 0));
  if (!exact && count) {
    auto* rk = ts == 16 ? blend_repair_k<16> : blend_repair_k<32>;
    VMS_CUDA(launch(rk, 2 * kSMs, kBlendThreads, 0, s, (const uint32_t*)w.ranges,
                    sorted_tiles(w, n_tiles), vals, (const RenderCounters*)w.ctr,
                    (const BlendRec*)w.rec, width, tiles_x, image, (const FrameDev*)w.fd,
                    (const uint32_t*)cert_cnt, (const uint4*)cert_list));
    mark("blend_repair", s);
  }
  VMS_LAUNCH_CHECK("blend");
  return VMS_OK;
}

// Tile duplication, tile sort, ranges, a band-major schedule for |bands|
// bands; then the blend as |bands| launches, unless bands < 0 (the caller
// launches them with render_band).
int32_t tiles_and_blend(int width, int height, const uint32_t* vals, const RenderWs& w,
                        float* image, int accumulate, int exact, void* const* events,
                        bool external, int bands, bool cleared, cudaStream_t s) {
  const int ts = tile_size(), shift = ts == 16 ? 4 : 5;
  const int tiles_x = ceil_div(width, ts), tiles_y = ceil_div(height, ts);
  const uint32_t n_tiles = (uint32_t)tiles_x * tiles_y;
  const int T = 256;
  const int ab = bands < 0 ? -bands : bands;
  const int nb = ab < 1 ? 1 : (ab > kMaxBands ? kMaxBands : ab);
  if (tiles_x > 256 || tiles_y > 256) {
    set_error("tiles_and_blend: more than 256 x 256 blend tiles");
    return VMS_ERR_INVALID;
  }
  const int gx = tiles_x + 1, gy = tiles_y + 1;
  if (!cleared) VMS_CUDA(cudaMemsetAsync(w.tdiff, 0, sizeof(uint32_t) * gx * gy, s));
  const size_t dsm = gx * gy <= kDiffSmemWords ? sizeof(uint32_t) * gx * gy : 0;
  VMS_CUDA(launch(dup_count_k, 2 * kSMs, T, dsm, s, vals, (const uint2*)w.box,
                  (const RenderCounters*)w.ctr, shift, gx, gy, w.cnt, w.rects, w.tdiff));
  mark("dup_count", s);
  int32_t st = scan_exclusive_u32(w.cnt, w.off, &w.ctr->n_kept, 0, w.n_cap, &w.ctr->n_inst,
                                  w.scan_ws2, s, !cleared);
  if (st) return st;
  const RadixLayout rl = radix_layout(w.radix_ws, w.n_cap > w.m_cap ? w.n_cap : w.m_cap);
  VMS_CUDA(launch(tile_prep_k, 1, 1024, dsm, s, (const uint32_t*)w.tdiff, tiles_x, tiles_y, nb,
                  w.m_cap, w.ctr, w.tcount, w.ranges, w.order, rl.counters, rl.ghist,
                  (const FrameDev*)(cleared ? w.fd : nullptr)));
  mark("tile_prep", s);
  VMS_CUDA(launch(dup_emit_k, 4 * kSMs, T, 0, s, vals, (const uint32_t*)w.rects,
                  (const uint32_t*)w.off, (const RenderCounters*)w.ctr, tiles_x, w.tk0, w.tv0,
                  rl.status, rl.pass_stride, rl.tile_items));
  mark("dup_emit", s);
  int alt = 0;
  st = radix_passes_u32(w.tk0, w.tv0, w.tk1, w.tv1, &w.ctr->n_inst,
                        w.n_cap > w.m_cap ? w.n_cap : w.m_cap, 0, tile_bits(n_tiles), &alt,
                        w.radix_ws, s);
  if (st) return st;
  const uint32_t* tv = alt ? w.tv1 : w.tv0;
  if (hot_path(exact, nb)) {
    VMS_CUDA(launch(hot_list_k, 1, 1024, 0, s, (const uint32_t*)w.ranges, n_tiles, hot_len(),
                    (const RenderCounters*)w.ctr, w.hot, w.tile_hot));
    mark("hot_list", s);
  }
  record(events, 2, external, s);
  if (bands < 0) return VMS_OK;  // the caller launches the bands
  if (tv != sorted_tiles(w, n_tiles)) {
    set_error("tiles_and_blend: tile sort parity");
    return VMS_ERR_INVARIANT;
  }
  for (int b = 0; b < nb; ++b) {
    st = launch_band(width, height, vals, w, image, accumulate, exact, b, nb, s);
    if (st) return st;
  }
  record(events, 3, external, s);
  VMS_LAUNCH_CHECK("tiles_and_blend");
  return VMS_OK;
}

}  // namespace

// One-time device setup of the blend (constant exp table).  Called outside
// any graph capture (session create, ABI entries).
int32_t blend_init() {
  static bool done = false;
  {
    // per device: the hot-tile blend's side stream and fork/join events
    int dev = 0;
    VMS_CUDA(cudaGetDevice(&dev));
    HotStreams& hs = g_hot[dev & 15];
    if (!hs.side) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(cudaStreamLegacy, &cs);
      if (cs == cudaStreamCaptureStatusNone) {
        VMS_CUDA(cudaStreamCreateWithFlags(&hs.side, cudaStreamNonBlocking));
        VMS_CUDA(cudaEventCreateWithFlags(&hs.fork, cudaEventDisableTiming));
        VMS_CUDA(cudaEventCreateWithFlags(&hs.join, cudaEventDisableTiming));
      }
    }
  }
  if (done) return VMS_OK;
  {
    const int32_t rc = preprocess_init();
    if (rc) return rc;
  }
  double2 t[64];
  for (int j = 0; j < 64; ++j) {
    const long double v = exp2l((long double)j / 64.0L);
    t[j].x = (double)v;
    t[j].y = (double)(v - (long double)t[j].x);
  }
  VMS_CUDA(cudaMemcpyToSymbol(kExp2Tab, t, sizeof(t)));
  {
    const char* e = getenv("VMSPLAT_LANE_LISTS");
    const int on = e && *e ? atoi(e) : 2;
    const char* mg = getenv("VMSPLAT_LANE_MARGIN");
    const int margin = mg && *mg ? atoi(mg) : 2;
    VMS_CUDA(cudaMemcpyToSymbol(g_lane_lists, &on, sizeof(int)));
    VMS_CUDA(cudaMemcpyToSymbol(g_lane_margin, &margin, sizeof(int)));
  }
  {
    const char* e = getenv("VMSPLAT_CERT_ALL");
    const int all = e && *e ? atoi(e) : 0;
    VMS_CUDA(cudaMemcpyToSymbol(g_cert_all, &all, sizeof(int)));
  }
  for (const void* f : {(const void*)blend_k<true, 16, true>, (const void*)blend_k<true, 32, true>})
    VMS_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kSparseSmem));
  for (const void* f : {(const void*)blend_hot_k<16>, (const void*)blend_hot_k<32>})
    VMS_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kHotSmem));
  VMS_CUDA(cudaFuncSetAttribute((const void*)tile_prep_k,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(uint32_t) * kDiffSmemWords)));
  done = true;
  return VMS_OK;
}

int32_t debug_exp(const double* x, uint64_t n, double* out, cudaStream_t s) {
  if (const int32_t rc = blend_init()) return rc;
  if (n) exp_eval_k<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, n, out);
  VMS_LAUNCH_CHECK("debug_exp");
  return VMS_OK;
}

int32_t debug_lane_lists(int on, int margin) {
  if (const int32_t rc = blend_init()) return rc;
  VMS_CUDA(cudaDeviceSynchronize());
  VMS_CUDA(cudaMemcpyToSymbol(g_lane_lists, &on, sizeof(int)));
  VMS_CUDA(cudaMemcpyToSymbol(g_lane_margin, &margin, sizeof(int)));
  return VMS_OK;
}

int32_t debug_cert_all(int on) {
  if (const int32_t rc = blend_init()) return rc;
  const int v = on ? 1 : 0;
  VMS_CUDA(cudaMemcpyToSymbol(g_cert_all, &v, sizeof(int)));
  return VMS_OK;
}

int32_t debug_cert_count(const RenderWs& w, uint32_t* out) {
  uint32_t c[16];
  VMS_CUDA(cudaDeviceSynchronize());
  VMS_CUDA(cudaMemcpy(c, w.cert, sizeof(c), cudaMemcpyDeviceToHost));
  uint32_t t = 0;
  for (int b = 0; b < kMaxBands; ++b) t += c[b];
  *out = t;
  uint32_t why[4];
  VMS_CUDA(cudaMemcpyFromSymbol(why, g_cert_why, sizeof(why)));
  if (why[0] | why[1] | why[2] | why[3]) {
    fprintf(stderr, "[cert] flagged %u: stop band %u, colour %u, >2000 steps %u, E>1e-3 %u\n", t,
            why[0], why[1], why[2], why[3]);
    const uint32_t z[4] = {0, 0, 0, 0};
    VMS_CUDA(cudaMemcpyToSymbol(g_cert_why, z, sizeof(z)));
  }
  return VMS_OK;
}

int32_t debug_blend_trace(void* dev_ptr) {
  unsigned long long* p = static_cast<unsigned long long*>(dev_ptr);
  VMS_CUDA(cudaMemcpyToSymbol(g_blend_trace, &p, sizeof(p)));
  return VMS_OK;
}

size_t render_ws_bytes(uint32_t n_cap, uint32_t m_cap, uint32_t n_tiles) {
  size_t b = 0;
  b += sizeof(uint32_t) * (size_t)n_cap * 3;   // key_g, flag, pos
  b += sizeof(BlendRec) * (size_t)n_cap;       // rec
  b += sizeof(uint2) * (size_t)n_cap;          // box
  b += sizeof(uint32_t) * (size_t)n_cap * 6;   // k0 v0 k1 v1 cnt off
  b += sizeof(uint32_t) * (size_t)m_cap * 4;   // tk0 tv0 tk1 tv1
  b += sizeof(uint32_t) * (size_t)n_cap;      // rects
  b += sizeof(uint32_t) * (4 * (size_t)n_tiles + 2);  // tcount + tdiff
  b += sizeof(uint32_t) * 3 * (size_t)n_tiles; // ranges + order
  b += sizeof(uint32_t) * (kMaxHot + 1 + (size_t)n_tiles);  // hot list + flags
  b += sizeof(RenderCounters) + sizeof(FrameDev);
  b += sizeof(uint32_t) * 16 + sizeof(uint4) * (size_t)n_tiles * tile_size() * tile_size();
  b += 2 * scan_ws_bytes(n_cap) + radix_ws_bytes(n_cap > m_cap ? n_cap : m_cap);
  return b + 256 * 26;
}

RenderWs render_carve(void* ws, uint32_t n_cap, uint32_t m_cap, uint32_t n_tiles) {
  char* p = static_cast<char*>(ws);
  RenderWs w;
  w.n_cap = n_cap;
  w.m_cap = m_cap;
  w.key_g = carve<uint32_t>(p, n_cap);
  w.flag = carve<uint32_t>(p, n_cap);
  w.pos = carve<uint32_t>(p, n_cap);
  w.rec = carve<BlendRec>(p, n_cap);
  w.box = carve<uint2>(p, n_cap);
  w.k0 = carve<uint32_t>(p, n_cap);
  w.v0 = carve<uint32_t>(p, n_cap);
  w.k1 = carve<uint32_t>(p, n_cap);
  w.v1 = carve<uint32_t>(p, n_cap);
  w.cnt = carve<uint32_t>(p, n_cap);
  w.off = carve<uint32_t>(p, n_cap);
  w.tk0 = carve<uint32_t>(p, m_cap);
  w.tv0 = carve<uint32_t>(p, m_cap);
  w.tk1 = carve<uint32_t>(p, m_cap);
  w.tv1 = carve<uint32_t>(p, m_cap);
  w.rects = carve<uint32_t>(p, n_cap);
  w.tcount = carve<uint32_t>(p, n_tiles);
  w.tdiff = carve<uint32_t>(p, 2 * (size_t)n_tiles + 2);  // >= (tx + 1)(ty + 1)
  w.ranges = carve<uint32_t>(p, 2 * (size_t)n_tiles);
  w.order = carve<uint32_t>(p, (size_t)n_tiles);
  w.hot = carve<uint32_t>(p, kMaxHot + 1);
  w.tile_hot = carve<uint32_t>(p, (size_t)n_tiles);
  w.ctr = carve<RenderCounters>(p, 1);
  w.fd = carve<FrameDev>(p, 1);
  w.cert = carve<uint32_t>(p, 16);
  w.cert_list = carve<uint4>(p, (size_t)n_tiles * tile_size() * tile_size());
  w.scan_ws = carve<char>(p, scan_ws_bytes(n_cap));
  w.scan_ws2 = carve<char>(p, scan_ws_bytes(n_cap));
  w.radix_ws = carve<char>(p, radix_ws_bytes(n_cap > m_cap ? n_cap : m_cap));
  return w;
}

int32_t render_upload_frame(const RenderWs& w, const FrameDev& f, cudaStream_t s) {
  VMS_CUDA(cudaMemcpyAsync(w.fd, &f, sizeof(FrameDev), cudaMemcpyHostToDevice, s));
  return VMS_OK;
}

int32_t render_band(int width, int height, const RenderWs& w, int exact, int band, int bands,
                    cudaStream_t s) {
  return launch_band(width, height, sorted_vals(w), w, nullptr, 0, exact, band, bands, s);
}

int32_t render_clear(int width, int height, const RenderWs& w, cudaStream_t s) {
  const int ts = tile_size();
  const size_t cells = (size_t)(ceil_div(width, ts) + 1) * (ceil_div(height, ts) + 1);
  VMS_CUDA(cudaMemsetAsync(w.ctr, 0, sizeof(RenderCounters), s));
  VMS_CUDA(cudaMemsetAsync(w.cert, 0, sizeof(uint32_t) * 16, s));
  VMS_CUDA(cudaMemsetAsync(w.scan_ws, 0, scan_ws_bytes(w.n_cap), s));
  VMS_CUDA(cudaMemsetAsync(w.scan_ws2, 0, scan_ws_bytes(w.n_cap), s));
  VMS_CUDA(cudaMemsetAsync(w.radix_ws, 0, radix_clear_bytes(), s));
  VMS_CUDA(cudaMemsetAsync(w.tdiff, 0, sizeof(uint32_t) * cells, s));
  return VMS_OK;
}

int32_t render_finish(int width, int height, const RenderWs& w, int accumulate, int exact,
                      void* const* events, bool external, int bands, cudaStream_t s) {
  // render_clear() ran before the preprocess: the kernels below chain with
  // programmatic dependent launches, no memset nodes in between
  const int T = 256;
  int32_t st = scan_exclusive_u32(w.flag, w.pos, &w.fd->n_splats, 0, w.n_cap, &w.ctr->n_kept,
                                  w.scan_ws, s, false);
  if (st) return st;
  VMS_CUDA(launch(compact_k, 8 * kSMs, T, 0, s, (const uint32_t*)w.flag, (const uint32_t*)w.pos,
                  (const uint32_t*)w.key_g, (const uint32_t*)&w.fd->n_splats, 0u, w.k0, w.v0));
  mark("compact", s);
  int alt = 0;
  // keys are IEEE bits of positive f32 depths: bit 31 is always clear
  st = radix_sort_u32(w.k0, w.v0, w.k1, w.v1, &w.ctr->n_kept, 0, w.n_cap, 0, 31, &alt,
                      w.radix_ws, s, false);
  if (st) return st;
  record(events, 1, external, s);
  if ((alt ? w.v1 : w.v0) != sorted_vals(w)) {
    set_error("render_finish: depth sort parity");
    return VMS_ERR_INVARIANT;
  }
  return tiles_and_blend(width, height, alt ? w.v1 : w.v0, w, nullptr, accumulate, exact, events,
                         external, bands, true, s);
}

int32_t composite_ordered(const float* centers, const float* conics, const float* colors,
                          const float* alphas, const int32_t* bounds, uint32_t n, float* image,
                          int h, int w, int exact, const RenderWs& ws, cudaStream_t s) {
  const int T = 256;
  VMS_CUDA(cudaMemsetAsync(ws.ctr, 0, sizeof(RenderCounters), s));
  VMS_CUDA(cudaMemsetAsync(ws.cert, 0, sizeof(uint32_t) * 16, s));
  if (n) {
    // splats with an empty clamped box are dropped; the rest keep their order
    pack_ordered_k<<<ceil_div<uint32_t>(n, T), T, 0, s>>>(centers, conics, colors, alphas, bounds,
                                                          n, w, h, ws.rec, ws.box, ws.v1,
                                                          ws.flag);
    int32_t st = scan_exclusive_u32(ws.flag, ws.pos, nullptr, n, n, &ws.ctr->n_kept, ws.scan_ws,
                                    s);
    if (st) return st;
    compact_k<<<ceil_div<uint32_t>(n, T), T, 0, s>>>(ws.flag, ws.pos, ws.v1, nullptr, n, ws.k0,
                                                     ws.v0);
  }
  return tiles_and_blend(w, h, ws.v0, ws, image, 1, exact, nullptr, false, 1, false, s);
}

}  // namespace vms
