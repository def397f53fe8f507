// Count-agnostic scan and stable LSD radix sort for sm_100a.
//
// Both primitives run on a fixed grid (kPrimGrid CTAs) and read the element
// count from device memory, so a frame never stalls on a device->host read
// of an intermediate size.  Each CTA owns one contiguous range of whole
// tiles; ranges are processed in order, which is what makes the radix sort
// stable (reduce-then-scan, Merrill-style).
//
// Radix ranking: per warp, __match_any_sync groups lanes holding the same
// digit; lane rank = popc(peers & lanemask_lt) + per-warp running count.
// Warps cover consecutive sub-tiles, so (warp, item, lane) order equals
// input order.  Each tile is re-ordered in shared memory by digit before the
// scatter so the global writes of one digit run are coalesced.
#include "common.cuh"
#include "prims.h"

namespace vms {

namespace {

constexpr int kScanBlock = 1024;

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

__device__ __forceinline__ void block_range(uint32_t n, uint32_t tile, uint32_t* lo,
                                            uint32_t* hi) {
  uint32_t tiles = (n + tile - 1) / tile;
  uint32_t per = (tiles + gridDim.x - 1) / gridDim.x;
  uint32_t a = blockIdx.x * per * tile;
  uint32_t b = a + per * tile;
  *lo = a < n ? a : n;
  *hi = b < n ? b : n;
}

// ---------------------------------------------------------------- scan
__global__ void __launch_bounds__(kScanBlock) scan_reduce_k(const uint32_t* in,
                                                             const uint32_t* n_dev,
                                                             uint32_t n_host,
                                                             uint32_t* partial) {
  __shared__ uint32_t red[33];
  uint32_t n = load_n(n_dev, n_host), lo, hi;
  block_range(n, kScanBlock, &lo, &hi);
  uint32_t s = 0;
  for (uint32_t i = lo + threadIdx.x; i < hi; i += kScanBlock) s += in[i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t t = red[threadIdx.x];
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
  }
}

// Exclusive scan of `count` values in place by one CTA (count arbitrary).
__global__ void __launch_bounds__(kScanBlock) scan_single_k(uint32_t* data, uint32_t count,
                                                             uint32_t* total) {
  __shared__ uint32_t scratch[33];
  uint32_t run = 0;
  for (uint32_t base = 0; base < count; base += kScanBlock) {
    uint32_t i = base + threadIdx.x;
    uint32_t v = i < count ? data[i] : 0u;
    uint32_t tot;
    uint32_t ex = block_exclusive<kScanBlock>(v, scratch, &tot);
    if (i < count) data[i] = run + ex;
    run += tot;
  }
  if (threadIdx.x == 0 && total) *total = run;
}

__global__ void __launch_bounds__(kScanBlock) scan_down_k(const uint32_t* in, uint32_t* out,
                                                           const uint32_t* n_dev,
                                                           uint32_t n_host,
                                                           const uint32_t* partial) {
  __shared__ uint32_t scratch[33];
  uint32_t n = load_n(n_dev, n_host), lo, hi;
  block_range(n, kScanBlock, &lo, &hi);
  uint32_t run = partial[blockIdx.x];
  for (uint32_t base = lo; base < hi; base += kScanBlock) {
    uint32_t i = base + threadIdx.x;
    uint32_t v = i < hi ? in[i] : 0u;
    uint32_t tot;
    uint32_t ex = block_exclusive<kScanBlock>(v, scratch, &tot);
    if (i < hi) out[i] = run + ex;
    run += tot;
  }
}

// ---------------------------------------------------------------- radix
constexpr int kRBlock = 256;  // threads; one per digit bin
constexpr int kRWarps = kRBlock / 32;
constexpr int kRItems = 8;
constexpr int kRTile = kRBlock * kRItems;  // 2048 pairs per tile

__global__ void __launch_bounds__(kRBlock) radix_upsweep_k(const uint32_t* keys,
                                                           const uint32_t* n_dev,
                                                           uint32_t n_host, int shift,
                                                           uint32_t mask,
                                                           uint32_t* counts) {
  __shared__ uint32_t hist[kRWarps][256];
  for (int i = threadIdx.x; i < kRWarps * 256; i += kRBlock) (&hist[0][0])[i] = 0;
  __syncthreads();
  uint32_t n = load_n(n_dev, n_host), lo, hi;
  block_range(n, kRTile, &lo, &hi);
  const int warp = threadIdx.x >> 5;
  for (uint32_t i = lo + threadIdx.x; i < hi; i += kRBlock)
    atomicAdd(&hist[warp][(keys[i] >> shift) & mask], 1u);
  __syncthreads();
  uint32_t s = 0;
#pragma unroll
  for (int w = 0; w < kRWarps; ++w) s += hist[w][threadIdx.x];
  counts[threadIdx.x * gridDim.x + blockIdx.x] = s;  // digit-major
}

__global__ void __launch_bounds__(kRBlock) radix_downsweep_k(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
    uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, const uint32_t* n_dev,
    uint32_t n_host, int shift, uint32_t mask, const uint32_t* __restrict__ offsets) {
  __shared__ uint32_t wcnt[kRWarps][257];
  __shared__ uint32_t skey[kRTile];
  __shared__ uint32_t sval[kRTile];
  __shared__ uint32_t run[256];
  __shared__ uint32_t tpre[256];
  __shared__ uint32_t scratch[33];

  uint32_t n = load_n(n_dev, n_host), lo, hi;
  block_range(n, kRTile, &lo, &hi);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  run[threadIdx.x] = offsets[threadIdx.x * gridDim.x + blockIdx.x];

  for (uint32_t base = lo; base < hi; base += kRTile) {
    for (int i = threadIdx.x; i < kRWarps * 257; i += kRBlock) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    uint32_t k[kRItems], v[kRItems], d[kRItems], rk[kRItems];
    const uint32_t wbase = base + warp * 32 * kRItems;
#pragma unroll
    for (int it = 0; it < kRItems; ++it) {
      uint32_t idx = wbase + it * 32 + lane;
      bool ok = idx < hi;
      k[it] = ok ? kin[idx] : 0u;
      v[it] = ok ? vin[idx] : 0u;
      d[it] = ok ? ((k[it] >> shift) & mask) : 256u;
    }
#pragma unroll
    for (int it = 0; it < kRItems; ++it) {
      uint32_t peers = __match_any_sync(0xffffffffu, d[it]);
      uint32_t before = wcnt[warp][d[it]];
      rk[it] = before + __popc(peers & lanemask_lt());
      __syncwarp();
      if (lane == __ffs(peers) - 1) wcnt[warp][d[it]] = before + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, tile total
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) {
      uint32_t c = wcnt[w][threadIdx.x];
      wcnt[w][threadIdx.x] = tot;
      tot += c;
    }
    uint32_t all;
    uint32_t pre = block_exclusive<kRBlock>(tot, scratch, &all);
    tpre[threadIdx.x] = pre;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kRItems; ++it) {
      if (d[it] < 256u) {
        uint32_t lp = tpre[d[it]] + wcnt[warp][d[it]] + rk[it];
        skey[lp] = k[it];
        sval[lp] = v[it];
      }
    }
    __syncthreads();
    const uint32_t cnt = min(hi - base, (uint32_t)kRTile);
    for (uint32_t j = threadIdx.x; j < cnt; j += kRBlock) {
      uint32_t kk = skey[j];
      uint32_t dd = (kk >> shift) & mask;
      uint32_t pos = run[dd] + (j - tpre[dd]);
      kout[pos] = kk;
      vout[pos] = sval[j];
    }
    __syncthreads();
    run[threadIdx.x] += tot;
    __syncthreads();
  }
}

}  // namespace

size_t scan_ws_bytes() { return sizeof(uint32_t) * (kPrimGrid + 32); }

int32_t scan_exclusive_u32(const uint32_t* in, uint32_t* out, const uint32_t* n_dev,
                           uint32_t n_host, uint32_t* total, void* ws, cudaStream_t s) {
  uint32_t* partial = static_cast<uint32_t*>(ws);
  scan_reduce_k<<<kPrimGrid, kScanBlock, 0, s>>>(in, n_dev, n_host, partial);
  mark("scan_reduce", s);
  scan_single_k<<<1, kScanBlock, 0, s>>>(partial, kPrimGrid, total);
  mark("scan_single", s);
  scan_down_k<<<kPrimGrid, kScanBlock, 0, s>>>(in, out, n_dev, n_host, partial);
  mark("scan_down", s);
  VMS_LAUNCH_CHECK("scan_exclusive_u32");
  return VMS_OK;
}

size_t radix_ws_bytes() { return sizeof(uint32_t) * (256 * kPrimGrid + 64) + scan_ws_bytes() + 256; }

int32_t radix_sort_u32(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1,
                       const uint32_t* n_dev, uint32_t n_host, int begin_bit, int end_bit,
                       int* in_alt, void* ws, cudaStream_t s) {
  uint32_t* counts = static_cast<uint32_t*>(ws);
  void* scan_ws = reinterpret_cast<char*>(ws) +
                  ((sizeof(uint32_t) * (256 * kPrimGrid + 64) + 255) & ~size_t(255));
  int alt = 0;
  for (int b = begin_bit; b < end_bit; b += 8) {
    int bits = end_bit - b < 8 ? end_bit - b : 8;
    uint32_t mask = (1u << bits) - 1u;
    uint32_t *ki = alt ? k1 : k0, *vi = alt ? v1 : v0;
    uint32_t *ko = alt ? k0 : k1, *vo = alt ? v0 : v1;
    radix_upsweep_k<<<kPrimGrid, kRBlock, 0, s>>>(ki, n_dev, n_host, b, mask, counts);
    mark("radix_up", s);
    // digit-major counts -> global (digit, block) offsets; only the digits
    // this pass can produce are scanned
    int32_t st = scan_exclusive_u32(counts, counts, nullptr, (mask + 1u) * kPrimGrid, nullptr,
                                    scan_ws, s);
    if (st) return st;
    radix_downsweep_k<<<kPrimGrid, kRBlock, 0, s>>>(ki, vi, ko, vo, n_dev, n_host, b, mask,
                                                    counts);
    mark("radix_down", s);
    alt ^= 1;
  }
  VMS_LAUNCH_CHECK("radix_sort_u32");
  *in_alt = alt;
  return VMS_OK;
}

}  // namespace vms
