// Count-agnostic scan and stable LSD radix sort for sm_100a.
//
// Both primitives read the element count from device memory (a frame never
// stalls on a device->host read of an intermediate size) and run as
// single-pass decoupled look-back kernels on a persistent grid: one launch
// per scan, one histogram launch + one launch per 8-bit radix pass
// (onesweep).  Tiles are claimed in order, so the sort is stable.
//
// Radix ranking: per warp, __match_any_sync groups lanes holding the same
// digit; lane rank = popc(peers & lanemask_lt) + per-warp running count.
// Warps cover consecutive sub-tiles, so (warp, item, lane) order equals
// input order.  Each tile is re-ordered in shared memory by digit before the
// scatter so the global writes of one digit run are coalesced.
#include <algorithm>

#include "common.cuh"
#include "prims.h"

#include <cstdlib>

namespace vms {

namespace {

__device__ __forceinline__ uint32_t load_n(const uint32_t* n_dev, uint32_t n_host) {
  return n_dev ? *n_dev : n_host;
}

// Block-wide exclusive scan of one value per thread; returns the block total
// through *total.  scratch: >= 32 u32 of shared memory.
template <int BLOCK>
__device__ __forceinline__ uint32_t block_exclusive(uint32_t v, uint32_t* scratch,
                                                    uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = BLOCK / 32;
    uint32_t w = lane < NW ? scratch[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < NW) scratch[lane] = wi - w;
    if (lane == 31) scratch[32] = wi;
  }
  __syncthreads();
  uint32_t res = scratch[warp] + inc - v;
  *total = scratch[32];
  __syncthreads();
  return res;
}

// ---------------------------------------------------------------- radix
constexpr int kRBlock = 256;  // threads; one per digit bin
constexpr int kRWarps = kRBlock / 32;
constexpr int kRItems = 12;
constexpr int kRTile = kRBlock * kRItems;  // 3072 pairs per tile
// sorts of up to kRSmallMax pairs (the per-frame depth sort) use half-size
// tiles: twice the CTAs on a grid that would otherwise leave SMs idle
constexpr int kRItemsSmall = 6;
constexpr int kRTileSmall = kRBlock * kRItemsSmall;
constexpr uint32_t kRSmallMax = 1u << 21;

// ------------------------------------------------ single-pass primitives
// Decoupled look-back (Merrill & Garland): tiles are claimed in order through
// an atomic counter by a persistent grid, each tile publishes its aggregate,
// walks back over its predecessors' published values until it meets an
// inclusive prefix, and publishes its own.  One launch per scan and per
// radix pass instead of reduce / scan / downsweep.  Status words: 2-bit flag
// (0 = empty, 1 = aggregate, 2 = inclusive prefix) + 30-bit value; the caller
// zeroes status + counter (one memset per primitive call).
constexpr uint32_t kFlagA = 1u << 30, kFlagP = 2u << 30, kValMask = (1u << 30) - 1u;

__device__ __forceinline__ uint32_t ld_status(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}
__device__ __forceinline__ void st_status(uint32_t* p, uint32_t v) {
  *reinterpret_cast<volatile uint32_t*>(p) = v;
}

// Exclusive prefix of tile t from the statuses of tiles t-1, t-2, ...,
// read kWindow predecessors at a time (independent loads in flight instead
// of one L2 round trip per predecessor); a window is consumed up to the first
// inclusive prefix, or up to the first predecessor that has not published
// yet, which is then re-read.
constexpr int kWindow = 8;

__device__ __forceinline__ uint32_t look_back(const uint32_t* status, uint32_t t, uint32_t stride) {
  uint32_t excl = 0;
  int64_t j = (int64_t)t - 1;
  while (j >= 0) {
    uint32_t v[kWindow];
#pragma unroll
    for (int k = 0; k < kWindow; ++k)
      v[k] = j - k >= 0 ? ld_status(status + (size_t)(j - k) * stride) : kFlagP;
    int used = 0;
    bool found = false;
#pragma unroll
    for (int k = 0; k < kWindow; ++k) {
      if (found || used < k) continue;  // stop at the first gap or prefix
      if ((v[k] & ~kValMask) == 0u) continue;
      excl += v[k] & kValMask;
      ++used;
      if (v[k] & kFlagP) found = true;
    }
    if (found) break;
    j -= used;
  }
  return excl;
}

constexpr int kLbThreads = 512;
constexpr int kLbItems = 8;
constexpr int kLbTile = kLbThreads * kLbItems;  // 4096

__global__ void __launch_bounds__(kLbThreads) scan_lb_k(const uint32_t* __restrict__ in,
                                                        uint32_t* __restrict__ out,
                                                        const uint32_t* n_dev, uint32_t n_host,
                                                        uint32_t* total, uint32_t* status,
                                                        uint32_t* counter) {
  pdl_wait();
  __shared__ uint32_t sdata[kLbTile + kLbTile / 32];
  __shared__ uint32_t scratch[33];
  __shared__ uint32_t s_tile, s_prefix;
  const uint32_t n = load_n(n_dev, n_host);
  const uint32_t n_tiles = (n + kLbTile - 1) / kLbTile;
  if (n == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && total) *total = 0;
    return;
  }
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    if (t >= n_tiles) break;
    const uint32_t base = t * kLbTile;
#pragma unroll
    for (int it = 0; it < kLbItems; ++it) {
      const uint32_t j = it * kLbThreads + threadIdx.x;
      sdata[j + (j >> 5)] = base + j < n ? in[base + j] : 0u;
    }
    __syncthreads();
    uint32_t v[kLbItems], sum = 0;
#pragma unroll
    for (int it = 0; it < kLbItems; ++it) {
      const uint32_t j = threadIdx.x * kLbItems + it;
      v[it] = sdata[j + (j >> 5)];
      sum += v[it];
    }
    uint32_t agg;
    uint32_t ex = block_exclusive<kLbThreads>(sum, scratch, &agg);
    if (threadIdx.x == 0) {
      uint32_t prefix = 0;
      if (t == 0) {
        st_status(status, kFlagP | agg);
      } else {
        st_status(status + t, kFlagA | agg);
        prefix = look_back(status, t, 1);
        st_status(status + t, kFlagP | ((prefix + agg) & kValMask));
      }
      s_prefix = prefix;
      if (t == n_tiles - 1 && total) *total = prefix + agg;
    }
    __syncthreads();
    ex += s_prefix;
#pragma unroll
    for (int it = 0; it < kLbItems; ++it) {
      const uint32_t j = threadIdx.x * kLbItems + it;
      sdata[j + (j >> 5)] = ex;
      ex += v[it];
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kLbItems; ++it) {
      const uint32_t j = it * kLbThreads + threadIdx.x;
      if (base + j < n) out[base + j] = sdata[j + (j >> 5)];
    }
    __syncthreads();
  }
}

// all passes' digit histograms in one read of the keys
// Also zeroes the look-back status words the passes will use (sized by the
// device-side count, so the host never clears a buffer sized for the worst
// case).
__global__ void __launch_bounds__(kRBlock) radix_hist_k(const uint32_t* __restrict__ keys,
                                                        const uint32_t* n_dev, uint32_t n_host,
                                                        int begin_bit, int end_bit,
                                                        uint32_t* __restrict__ ghist,
                                                        uint32_t* __restrict__ status,
                                                        size_t pass_stride, uint32_t tile_items) {
  pdl_wait();
  __shared__ uint32_t h[4][256];
  for (int i = threadIdx.x; i < 4 * 256; i += kRBlock) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t n = load_n(n_dev, n_host);
  const int passes = (end_bit - begin_bit + 7) / 8;
  const size_t used = (size_t)((n + tile_items - 1) / tile_items) * 256;
  for (int p = 0; p < passes; ++p)
    for (size_t i = blockIdx.x * (size_t)kRBlock + threadIdx.x; i < used;
         i += (size_t)gridDim.x * kRBlock)
      status[p * pass_stride + i] = 0u;
  for (uint32_t i = blockIdx.x * kRBlock + threadIdx.x; i < n; i += gridDim.x * kRBlock) {
    const uint32_t k = keys[i];
    for (int p = 0; p < passes; ++p) {
      const int b = begin_bit + 8 * p;
      const int bits = end_bit - b < 8 ? end_bit - b : 8;
      atomicAdd(&h[p][(k >> b) & ((1u << bits) - 1u)], 1u);
    }
  }
  __syncthreads();
  for (int p = 0; p < passes; ++p) {
    const uint32_t c = h[p][threadIdx.x];
    if (c) atomicAdd(&ghist[p * 256 + threadIdx.x], c);
  }
}

template <int kItems>
__global__ void __launch_bounds__(kRBlock) radix_onesweep_k(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
    uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, const uint32_t* n_dev,
    uint32_t n_host, int shift, uint32_t mask, const uint32_t* __restrict__ hist,
    uint32_t* status, uint32_t* counter) {
  pdl_wait();
  __shared__ uint32_t wcnt[kRWarps][257];
  __shared__ uint32_t skey[kRBlock * kItems];
  __shared__ uint32_t sval[kRBlock * kItems];
  __shared__ uint32_t dbase[256];
  __shared__ uint32_t run[256];
  __shared__ uint32_t tpre[256];
  __shared__ uint32_t scratch[33];
  __shared__ uint32_t s_tile;

  const uint32_t n = load_n(n_dev, n_host);
  const uint32_t n_tiles = (n + (kRBlock * kItems) - 1) / (kRBlock * kItems);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  {
    uint32_t all;
    dbase[threadIdx.x] = block_exclusive<kRBlock>(hist[threadIdx.x], scratch, &all);
  }
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    for (int i = threadIdx.x; i < kRWarps * 257; i += kRBlock) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint32_t t = s_tile;
    if (t >= n_tiles) break;
    const uint32_t base = t * (kRBlock * kItems);
    const uint32_t hi = min(n, base + (kRBlock * kItems));
    uint32_t k[kItems], v[kItems], d[kItems], rk[kItems];
    const uint32_t wbase = base + warp * 32 * kItems;
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint32_t idx = wbase + it * 32 + lane;
      const bool ok = idx < hi;
      k[it] = ok ? kin[idx] : 0u;
      v[it] = ok ? vin[idx] : 0u;
      d[it] = ok ? ((k[it] >> shift) & mask) : 256u;
    }
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint32_t peers = __match_any_sync(0xffffffffu, d[it]);
      const uint32_t before = wcnt[warp][d[it]];
      rk[it] = before + __popc(peers & lanemask_lt());
      __syncwarp();
      if (lane == __ffs(peers) - 1) wcnt[warp][d[it]] = before + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) {
      const uint32_t c = wcnt[w][threadIdx.x];
      wcnt[w][threadIdx.x] = tot;
      tot += c;
    }
    // publish this tile's digit counts, look back for the digit prefix
    uint32_t* my = status + (size_t)t * 256 + threadIdx.x;
    uint32_t excl = 0;
    if (t == 0) {
      st_status(my, kFlagP | tot);
    } else {
      st_status(my, kFlagA | tot);
      excl = look_back(status + threadIdx.x, t, 256);
      st_status(my, kFlagP | ((excl + tot) & kValMask));
    }
    run[threadIdx.x] = dbase[threadIdx.x] + excl;
    uint32_t all;
    tpre[threadIdx.x] = block_exclusive<kRBlock>(tot, scratch, &all);
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      if (d[it] < 256u) {
        const uint32_t lp = tpre[d[it]] + wcnt[warp][d[it]] + rk[it];
        skey[lp] = k[it];
        sval[lp] = v[it];
      }
    }
    __syncthreads();
    const uint32_t cnt = hi - base;
    for (uint32_t j = threadIdx.x; j < cnt; j += kRBlock) {
      const uint32_t kk = skey[j];
      const uint32_t dd = (kk >> shift) & mask;
      const uint32_t pos = run[dd] + (j - tpre[dd]);
      kout[pos] = kk;
      vout[pos] = sval[j];
    }
    __syncthreads();
  }
}

int persistent_grid(const void* kern, int threads, int cap) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = kSMs;
  }
  // occupancy per (kernel, block size), queried once (also keeps the query
  // out of graph captures)
  static const void* keys[16] = {};
  static int vals[16] = {};
  int per = 0;
  for (int i = 0; i < 16; ++i)
    if (keys[i] == kern && vals[i] >> 16 == threads) per = vals[i] & 0xFFFF;
  if (!per) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, 0);
    if (per <= 0) per = 1;
    for (int i = 0; i < 16; ++i)
      if (!keys[i]) {
        keys[i] = kern;
        vals[i] = (threads << 16) | per;
        break;
      }
  }
  const int g = sms * per;
  return cap > 0 && cap < g ? cap : g;
}

}  // namespace

size_t scan_ws_bytes(uint32_t n_max) {
  return sizeof(uint32_t) * (((size_t)n_max + kLbTile - 1) / kLbTile + 64);
}

int32_t scan_exclusive_u32(const uint32_t* in, uint32_t* out, const uint32_t* n_dev,
                           uint32_t n_host, uint32_t n_max, uint32_t* total, void* ws,
                           cudaStream_t s, bool clear) {
  const uint32_t max_tiles = (n_max + kLbTile - 1) / kLbTile;
  uint32_t* counter = static_cast<uint32_t*>(ws);
  uint32_t* status = counter + 32;
  if (clear) VMS_CUDA(cudaMemsetAsync(ws, 0, scan_ws_bytes(n_max), s));
  const int grid = persistent_grid((const void*)scan_lb_k, kLbThreads, max_tiles ? max_tiles : 1);
  VMS_CUDA(launch(scan_lb_k, grid, kLbThreads, 0, s, in, out, n_dev, n_host, total, status,
                  counter));
  mark("scan", s);
  VMS_LAUNCH_CHECK("scan_exclusive_u32");
  return VMS_OK;
}

size_t radix_clear_bytes() { return sizeof(uint32_t) * (64 + 4 * 256); }

size_t radix_ws_bytes(uint32_t n_max) {
  size_t tiles = ((size_t)n_max + kRTile - 1) / kRTile;
  const size_t small = ((size_t)std::min(n_max, kRSmallMax) + kRTileSmall - 1) / kRTileSmall;
  if (small > tiles) tiles = small;
  return sizeof(uint32_t) * (64 + 4 * 256 + 4 * 256 * tiles) + 256;
}

RadixLayout radix_layout(void* ws, uint32_t n_max) {
  RadixLayout l;
  l.counters = static_cast<uint32_t*>(ws);
  l.ghist = l.counters + 64;
  l.status = l.ghist + 4 * 256;
  l.pass_stride = 256 * (((size_t)n_max + kRTile - 1) / kRTile);
  l.tile_items = kRTile;
  return l;
}

// CTAs a onesweep pass asks for: one per tile, at most two per SM
// (VMSPLAT_RADIX_GRID overrides; 0 = up to the resident limit).  The sorts
// run beside the previous frame's blend: fewer resident look-back CTAs leave
// it more of each SM (C2 frames 5-34, same box: 2122-2141 frames/s with 3-4
// per SM, 2157-2165 with 2, 2102-2115 with 1).
int radix_grid_want(size_t tiles) {
  static const int cap = [] {
    const char* e = getenv("VMSPLAT_RADIX_GRID");
    return e && *e ? atoi(e) : 2 * kSMs;
  }();
  const int want = tiles ? (int)tiles : 1;
  return cap > 0 && cap < want ? cap : want;
}

int32_t radix_passes_u32(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1,
                         const uint32_t* n_dev, uint32_t n_max, int begin_bit, int end_bit,
                         int* in_alt, void* ws, cudaStream_t s) {
  const int passes = (end_bit - begin_bit + 7) / 8;
  if (passes > 4) {
    set_error("radix_passes_u32: at most 32 key bits");
    return VMS_ERR_INVALID;
  }
  const RadixLayout l = radix_layout(ws, n_max);
  const size_t tiles = l.pass_stride / 256;
  const int grid = persistent_grid((const void*)radix_onesweep_k<kRItems>, kRBlock,
                                   radix_grid_want(tiles));
  int alt = 0;
  for (int p = 0; p < passes; ++p) {
    const int b = begin_bit + 8 * p;
    const int bits = end_bit - b < 8 ? end_bit - b : 8;
    const uint32_t mask = (1u << bits) - 1u;
    uint32_t *ki = alt ? k1 : k0, *vi = alt ? v1 : v0;
    uint32_t *ko = alt ? k0 : k1, *vo = alt ? v0 : v1;
    VMS_CUDA(launch(radix_onesweep_k<kRItems>, grid, kRBlock, 0, s, (const uint32_t*)ki,
                    (const uint32_t*)vi, ko, vo, n_dev, 0u, b, mask,
                    (const uint32_t*)(l.ghist + p * 256), l.status + p * l.pass_stride,
                    l.counters + p));
    mark("radix_pass", s);
    alt ^= 1;
  }
  VMS_LAUNCH_CHECK("radix_passes_u32");
  *in_alt = alt;
  return VMS_OK;
}

int32_t radix_sort_u32(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1,
                       const uint32_t* n_dev, uint32_t n_host, uint32_t n_max, int begin_bit,
                       int end_bit, int* in_alt, void* ws, cudaStream_t s, bool clear) {
  const int passes = (end_bit - begin_bit + 7) / 8;
  if (passes > 4) {
    set_error("radix_sort_u32: at most 32 key bits");
    return VMS_ERR_INVALID;
  }
  const bool small = n_max <= kRSmallMax;
  const uint32_t tile_items = small ? kRTileSmall : kRTile;
  const size_t tiles = ((size_t)n_max + tile_items - 1) / tile_items;
  uint32_t* counters = static_cast<uint32_t*>(ws);  // one per pass
  uint32_t* ghist = counters + 64;                  // [passes][256]
  uint32_t* status = ghist + 4 * 256;               // [passes][tiles][256]
  if (clear) VMS_CUDA(cudaMemsetAsync(ws, 0, radix_clear_bytes(), s));
  // a few CTAs per SM: each flushes 4 x 256 bins with global atomics
  const int hgrid = persistent_grid((const void*)radix_hist_k, kRBlock,
                                    (int)std::min<size_t>(2 * 148, (n_max + 4095) / 4096 + 1));
  VMS_CUDA(launch(radix_hist_k, hgrid, kRBlock, 0, s, (const uint32_t*)k0, n_dev, n_host,
                  begin_bit, end_bit, ghist, status, (size_t)(256 * tiles), tile_items));
  mark("radix_hist", s);
  auto* kern = small ? radix_onesweep_k<kRItemsSmall> : radix_onesweep_k<kRItems>;
  const int grid = persistent_grid((const void*)kern, kRBlock, radix_grid_want(tiles));
  int alt = 0;
  for (int p = 0; p < passes; ++p) {
    const int b = begin_bit + 8 * p;
    const int bits = end_bit - b < 8 ? end_bit - b : 8;
    const uint32_t mask = (1u << bits) - 1u;
    uint32_t *ki = alt ? k1 : k0, *vi = alt ? v1 : v0;
    uint32_t *ko = alt ? k0 : k1, *vo = alt ? v0 : v1;
    VMS_CUDA(launch(kern, grid, kRBlock, 0, s, (const uint32_t*)ki,
                    (const uint32_t*)vi, ko, vo, n_dev, n_host, b, mask,
                    (const uint32_t*)(ghist + p * 256), status + (size_t)p * 256 * tiles,
                    counters + p));
    mark("radix_pass", s);
    alt ^= 1;
  }
  VMS_LAUNCH_CHECK("radix_sort_u32");
  *in_alt = alt;
  return VMS_OK;
}

}  // namespace vms
