// the page table / LRU residency cache resident in device
// memory - the exact semantics of runtime.PageTable + update_page_table
// (pkg/src/vmsplat/runtime.py:161-346), computed on the GPU right after the
// visibility pass, so the host no longer runs the table: it only reads the
// frame's copy plan and stats (mapped memory) to issue the page DMAs.
//
// One CTA (dpt_update_k) does the frame's update:
//   pass 1 (all threads)   every required page: resident -> refresh its
//                          entry's LRU stamp and protect it, and a class-2
//                          work item if its level differs; otherwise a
//                          class 0 (direct) / 1 (link-pulled) item
//   sort (all threads)     bitonic sort of the items by the 64-bit key
//                          (class, ~encoded depth, page id) - unique keys, so
//                          the reference's (class, -enc, pid) order exactly
//   pass 2 (thread 0)      the budgeted walk: break (never skip) on the
//                          staging budget, `continue` past a failed
//                          allocation; allocation order = first open entry of
//                          the level (bitmap + summary word find-first-set),
//                          first empty entry, then the least recently used
//                          unprotected entry (a cursor over the entries kept
//                          in (last used, index) order)
//   epilogue (all threads) missing count, the LRU order for the next frame
//                          (untouched entries keep their order, the entries
//                          touched this frame follow in index order - they
//                          all carry this frame's stamp), state write-back
// Three small kernels (dpt_chunk_sums_k, dpt_chunk_scan_k,
// dpt_chunk_emit_k: block sums, their scan, the emit) build the chunk table
// of every resident page in ascending page id (the reference's gather
// order, runtime.py:377-390) for the render.
//
// The entry metadata (level, occupancy, free-slot mask) and the bitmaps live
// in shared memory during the update: capacity <= 8192 entries and <= 6 LOD
// levels (<= 32 slots per entry).  Per-entry slot contents, LRU stamps, the
// page -> (entry, slot) map and the LRU order live in global memory.
#include <cstdint>
#include <vector>

#include "common.cuh"

struct vms_dpt {
  int32_t C, P, L, S, W, WS;  // capacity, pages, levels, max slots, bitmap words, summary words
  int8_t* level;
  uint8_t* occ;
  uint32_t* freem;
  int32_t* last;
  uint32_t* slots;   // [C * S]
  uint32_t* res;     // [P + 1]: entry << 8 | slot, or kNone
  uint32_t* bm;      // [(L + 1) * W]: open bitmaps per level, then the empty bitmap
  int32_t* lru[2];   // entries in (last used, index) order; [cur] is current
  int32_t* cur;      // [1] device: which lru buffer is current
  uint64_t* skeys;   // [P + 1] sort spill (more required pages than fit in shared memory)
  uint32_t* svals;
  int32_t* counts;   // [2 + 16]: occupied entries, resident pages, resident per level
  uint2* csums;      // chunk table: per 2048-page block (records, chunks), then their bases
  void* base;
};

namespace vms {
namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kThreads = 1024;
constexpr int kMaxCap = 8192;
constexpr int kMaxLevels = 6;
constexpr uint64_t kNoKey = ~0ull;

struct DptArgs {
  int32_t C, P, L, S, W, WS;
  int8_t* level;
  uint8_t* occ;
  uint32_t* freem;
  int32_t* last;
  uint32_t* slots;
  uint32_t* res;
  uint32_t* bm;
  int32_t* lru0;
  int32_t* lru1;
  int32_t* cur;
  uint64_t* skeys;
  uint32_t* svals;
  int32_t* counts;
  // frame inputs
  const uint32_t* pid;
  const uint32_t* enc;
  const uint8_t* direct;
  const uint8_t* lvl;
  const uint32_t* n_req;  // device count
  const vms_dpt_frame* frame;
  // outputs
  uint32_t* plan_pid;
  uint8_t* plan_level;
  int32_t* plan_entry;
  int32_t* plan_slot;
  int64_t plan_cap;
  vms_dpt_stats* stats;
  int sort_cap;  // work items sorted in shared memory (a power of two)
};

struct Bits {
  uint32_t* w;    // words
  uint32_t* sum;  // summary: bit k of sum[j] = word 32 j + k non-zero
  VMS_DEV void set(int i) {
    w[i >> 5] |= 1u << (i & 31);
    sum[i >> 10] |= 1u << ((i >> 5) & 31);
  }
  VMS_DEV void clear(int i) {
    const uint32_t v = w[i >> 5] & ~(1u << (i & 31));
    w[i >> 5] = v;
    if (!v) sum[i >> 10] &= ~(1u << ((i >> 5) & 31));
  }
  VMS_DEV bool test(int i) const { return (w[i >> 5] >> (i & 31)) & 1u; }
  // lowest set index, or -1
  VMS_DEV int first(int ws) const {
    for (int j = 0; j < ws; ++j)
      if (sum[j]) {
        const int wi = 32 * j + __ffs(sum[j]) - 1;
        return 32 * wi + __ffs(w[wi]) - 1;
      }
    return -1;
  }
};

__device__ int block_excl_scan(int v, int* warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    const int t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
    int u = t;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, u, o);
      if (lane >= o) u += y;
    }
    warp_tot[lane] = u - t;        // exclusive warp offsets
    if (lane == 31) warp_tot[32] = u;  // total
  }
  __syncthreads();
  const int r = warp_tot[w] + x - v;
  return r;
}

__global__ void __launch_bounds__(kThreads, 1) dpt_update_k(DptArgs a) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int warp_tot[33];
  __shared__ int s_np, s_missing, s_bad, s_resident, s_occupied;
  __shared__ int s_per[16];
  const int C = a.C, L = a.L, W = a.W, WS = a.WS, tid = threadIdx.x, NT = blockDim.x;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  uint32_t* vals = reinterpret_cast<uint32_t*>(keys + a.sort_cap);
  uint32_t* freem = vals + a.sort_cap;
  uint32_t* bw = freem + C;               // (L + 2) * W: open[L], empty, prot
  uint32_t* bs = bw + (L + 2) * W;        // (L + 2) * WS summaries
  int8_t* level = reinterpret_cast<int8_t*>(bs + (L + 2) * WS);
  uint8_t* occ = reinterpret_cast<uint8_t*>(level + C);
  const int n = (int)*a.n_req;
  const int64_t frame = a.frame->frame;
  const double budget = a.frame->budget;
  // state -> shared memory; prot cleared
  for (int i = tid; i < C; i += NT) {
    freem[i] = a.freem[i];
    level[i] = a.level[i];
    occ[i] = a.occ[i];
  }
  for (int i = tid; i < (L + 1) * W; i += NT) bw[i] = a.bm[i];
  for (int i = tid; i < W; i += NT) bw[(L + 1) * W + i] = 0u;
  for (int i = tid; i < (L + 2) * WS; i += NT) bs[i] = 0u;
  if (tid == 0) {
    s_np = 0;
    s_missing = 0;
    s_bad = 0;
    s_occupied = a.counts[0];
    s_resident = a.counts[1];
    for (int k = 0; k < 16; ++k) s_per[k] = a.counts[2 + k];
  }
  __syncthreads();
  for (int b = 0; b < L + 2; ++b)
    for (int i = tid; i < W; i += NT)
      if (bw[b * W + i]) atomicOr(&bs[b * WS + (i >> 5)], 1u << (i & 31));
  __syncthreads();
  Bits open[kMaxLevels], empty{bw + L * W, bs + L * WS}, prot{bw + (L + 1) * W, bs + (L + 1) * WS};
  for (int k = 0; k < L; ++k) open[k] = Bits{bw + k * W, bs + k * WS};
  // pass 1 (runtime.py:312-327): keys in shared memory up to sort_cap pages
  int N = 1;
  while (N < n) N <<= 1;
  uint64_t* K = N <= a.sort_cap ? keys : a.skeys;
  uint32_t* V = N <= a.sort_cap ? vals : a.svals;
  for (int i = tid; i < N; i += NT) {
    uint64_t key = kNoKey;
    if (i < n) {
      const uint32_t p = a.pid[i];
      const int lv = a.lvl[i];
      if (p == 0 || p > (uint32_t)a.P || lv >= L) {
        s_bad = 1;
      } else {
        const uint32_t loc = a.res[p];
        const uint64_t tail = ((uint64_t)(~a.enc[i]) << 30) | p;
        if (loc != kNone) {
          const int e = (int)(loc >> 8);
          a.last[e] = (int32_t)frame;
          atomicOr(&prot.w[e >> 5], 1u << (e & 31));
          atomicOr(&prot.sum[e >> 10], 1u << ((e >> 5) & 31));
          if (level[e] != lv) key = (2ull << 62) | tail;
        } else {
          key = ((a.direct[i] ? 0ull : 1ull) << 62) | tail;
        }
      }
    }
    K[i] = key;
    V[i] = (uint32_t)i;
  }
  __syncthreads();
  // bitonic sort (keys are unique: the page id is in them)
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < N; i += NT) {
        const int l = i ^ j;
        if (l > i) {
          const uint64_t x = K[i], y = K[l];
          const bool up = (i & k) == 0;
          if (up ? x > y : x < y) {
            K[i] = y;
            K[l] = x;
            const uint32_t t = V[i];
            V[i] = V[l];
            V[l] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  // pass 2 (runtime.py:330-343) on one thread
  if (tid == 0 && !s_bad) {
    double spent = 0.0;
    int cursor = 0;
    const int32_t* lru = *a.cur ? a.lru1 : a.lru0;
    int np = 0;
    for (int k = 0; k < n; ++k) {
      const uint64_t key = K[k];
      if (key == kNoKey) break;
      const int i = (int)V[k];
      const uint32_t p = (uint32_t)(key & 0x3FFFFFFFull);
      const int lv = a.lvl[i];
      const double cost = 1.0 / (double)(1 << lv);
      if (spent + cost > budget) break;
      const int nslot = 1 << lv;
      const uint32_t full = nslot == 32 ? 0xFFFFFFFFu : (1u << nslot) - 1u;
      // _alloc_slot (runtime.py:238-264)
      int e = open[lv].first(WS), s = 0;
      if (e >= 0) {
        s = __ffs(freem[e]) - 1;
      } else {
        e = empty.first(WS);
        if (e < 0) {
          while (cursor < C && prot.test(lru[cursor])) ++cursor;
          if (cursor == C) continue;  // every entry protected: no slot
          e = lru[cursor++];
          // _evict (runtime.py:266-271)
          const int ol = level[e];
          uint32_t used = ~freem[e] & (((1u << ol) == 32u) ? 0xFFFFFFFFu : ((1u << (1 << ol)) - 1u));
          while (used) {
            const int q = __ffs(used) - 1;
            used &= used - 1;
            const uint32_t victim = a.slots[(size_t)e * a.S + q];
            a.res[victim] = kNone;
            --s_resident;
            --s_per[ol];
          }
          if (occ[e] < (1 << ol)) open[ol].clear(e);
          --s_occupied;
        } else {
          empty.clear(e);
        }
        // activate
        level[e] = (int8_t)lv;
        occ[e] = 0;
        freem[e] = full;
        for (int q = 0; q < nslot; ++q) a.slots[(size_t)e * a.S + q] = 0u;
        open[lv].set(e);
        ++s_occupied;
        s = 0;
      }
      // _place (runtime.py:273-283)
      const uint32_t old = a.res[p];
      a.slots[(size_t)e * a.S + s] = p;
      freem[e] &= ~(1u << s);
      if (++occ[e] == nslot) open[lv].clear(e);
      a.last[e] = (int32_t)frame;
      a.res[p] = ((uint32_t)e << 8) | (uint32_t)s;
      prot.set(e);
      ++s_per[lv];
      if (old == kNone) {
        ++s_resident;
      } else {
        const int oe = (int)(old >> 8), os = (int)(old & 0xFF), ol = level[oe];
        --s_per[ol];
        a.slots[(size_t)oe * a.S + os] = 0u;
        freem[oe] |= 1u << os;
        open[ol].set(oe);
        if (--occ[oe] == 0) {  // clear()
          open[ol].clear(oe);
          level[oe] = -1;
          empty.set(oe);
          --s_occupied;
        }
      }
      if (np < a.plan_cap) {
        a.plan_pid[np] = p;
        a.plan_level[np] = (uint8_t)lv;
        a.plan_entry[np] = e;
        a.plan_slot[np] = s;
      }
      ++np;
      spent += cost;
    }
    s_np = np;
  }
  __syncthreads();
  // missing = required pages resident at no level afterwards
  int miss = 0;
  for (int i = tid; i < n; i += NT) {
    const uint32_t p = a.pid[i];
    if (p >= 1 && p <= (uint32_t)a.P && a.res[p] == kNone) ++miss;
  }
  for (int o = 16; o; o >>= 1) miss += __shfl_xor_sync(0xFFFFFFFFu, miss, o);
  if ((tid & 31) == 0 && miss) atomicAdd(&s_missing, miss);
  // LRU order for the next frame: untouched entries in their order, then the
  // entries protected (= stamped) this frame in index order
  const int32_t* lru = *a.cur ? a.lru1 : a.lru0;
  int32_t* nl = *a.cur ? a.lru0 : a.lru1;
  const int per = (C + NT - 1) / NT;
  const int b0 = tid * per, b1 = min(C, b0 + per);
  int keep = 0;
  for (int i = b0; i < b1; ++i) keep += prot.test(lru[i]) ? 0 : 1;
  int pos = block_excl_scan(keep, warp_tot);
  const int n_keep = warp_tot[32];
  for (int i = b0; i < b1; ++i)
    if (!prot.test(lru[i])) nl[pos++] = lru[i];
  __syncthreads();
  int touched = 0;
  for (int i = b0; i < b1; ++i) touched += prot.test(i) ? 1 : 0;
  pos = n_keep + block_excl_scan(touched, warp_tot);
  for (int i = b0; i < b1; ++i)
    if (prot.test(i)) nl[pos++] = i;
  // write-back
  for (int i = tid; i < C; i += NT) {
    a.freem[i] = freem[i];
    a.level[i] = level[i];
    a.occ[i] = occ[i];
  }
  for (int i = tid; i < (L + 1) * W; i += NT) a.bm[i] = bw[i];
  __syncthreads();
  if (tid == 0) {
    *a.cur = *a.cur ^ 1;
    a.counts[0] = s_occupied;
    a.counts[1] = s_resident;
    for (int k = 0; k < 16; ++k) a.counts[2 + k] = s_per[k];
    vms_dpt_stats* st = a.stats;
    st->n_req = (uint32_t)n;
    st->n_plan = (uint32_t)s_np;
    st->missing = (uint32_t)s_missing;
    st->resident = (uint32_t)s_resident;
    st->occupied = (uint32_t)s_occupied;
    st->bad = (uint32_t)s_bad;
    st->plan_overflow = s_np > a.plan_cap ? 1u : 0u;
    for (int k = 0; k < 16; ++k) st->resident_per_level[k] = (uint32_t)s_per[k];
  }
}

// chunk table of the resident pages, ascending page id (runtime.py:377-390):
// per-block sums of records and chunks over 2048-page blocks, a scan of the
// block sums, then every block emits its pages' chunks from its base
constexpr int kChunkThreads = 256;
constexpr int kChunkPages = 8;  // pages per thread
constexpr int kChunkBlock = kChunkThreads * kChunkPages;
constexpr uint32_t kChunkRecs = 128;

__device__ __forceinline__ void page_chunks(const uint32_t* res, const int8_t* level, int p,
                                            uint32_t page_size, uint32_t& r, uint32_t& c) {
  const uint32_t loc = res[p];
  r = loc == kNone ? 0u : page_size >> level[loc >> 8];
  c = (r + kChunkRecs - 1) / kChunkRecs;
}

__global__ void __launch_bounds__(kChunkThreads) dpt_chunk_sums_k(
    const uint32_t* __restrict__ res, const int8_t* __restrict__ level, int32_t P,
    uint32_t page_size, uint2* __restrict__ sums) {
  pdl_wait();
  __shared__ int warp_tot[33];
  const int p0 = 1 + blockIdx.x * kChunkBlock + threadIdx.x * kChunkPages;
  int recs = 0, chunks = 0;
  for (int p = p0; p < min(P + 1, p0 + kChunkPages); ++p) {
    uint32_t r, c;
    page_chunks(res, level, p, page_size, r, c);
    recs += (int)r;
    chunks += (int)c;
  }
  block_excl_scan(recs, warp_tot);
  const int tr = warp_tot[32];
  __syncthreads();
  block_excl_scan(chunks, warp_tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = make_uint2((uint32_t)tr, (uint32_t)warp_tot[32]);
}

__global__ void __launch_bounds__(1024) dpt_chunk_scan_k(uint2* __restrict__ sums, int nb,
                                                        vms_dpt_stats* st) {
  pdl_wait();
  __shared__ int warp_tot[33];
  int base_r = 0, base_c = 0;
  for (int b0 = 0; b0 < nb; b0 += blockDim.x) {
    const int b = b0 + threadIdx.x;
    const uint2 v = b < nb ? sums[b] : make_uint2(0u, 0u);
    const int er = block_excl_scan((int)v.x, warp_tot);
    const int tr = warp_tot[32];
    __syncthreads();
    const int ec = block_excl_scan((int)v.y, warp_tot);
    const int tc = warp_tot[32];
    __syncthreads();
    if (b < nb) sums[b] = make_uint2((uint32_t)(base_r + er), (uint32_t)(base_c + ec));
    base_r += tr;
    base_c += tc;
  }
  if (threadIdx.x == 0) {
    st->n_records = (uint32_t)base_r;
    st->n_chunks = (uint32_t)base_c;
  }
}

__global__ void __launch_bounds__(kChunkThreads) dpt_chunk_emit_k(
    const uint32_t* __restrict__ res, const int8_t* __restrict__ level, int32_t P,
    uint32_t page_size, const uint2* __restrict__ bases, vms_chunk* __restrict__ out,
    int64_t cap) {
  pdl_wait();
  __shared__ int warp_tot[33];
  const int p0 = 1 + blockIdx.x * kChunkBlock + threadIdx.x * kChunkPages;
  const int p1 = min(P + 1, p0 + kChunkPages);
  int recs = 0, chunks = 0;
  for (int p = p0; p < p1; ++p) {
    uint32_t r, c;
    page_chunks(res, level, p, page_size, r, c);
    recs += (int)r;
    chunks += (int)c;
  }
  const uint2 base = bases[blockIdx.x];
  int g = (int)base.x + block_excl_scan(recs, warp_tot);
  __syncthreads();
  int64_t c = (int64_t)base.y + block_excl_scan(chunks, warp_tot);
  for (int p = p0; p < p1; ++p) {
    const uint32_t loc = res[p];
    if (loc == kNone) continue;
    const uint32_t e = loc >> 8, sl = loc & 0xFF;
    const uint32_t r = page_size >> level[e];
    const uint32_t row = e * page_size + sl * r;
    for (uint32_t k = 0; k < r; k += kChunkRecs) {
      if (c < cap) out[c] = vms_chunk{row + k, (uint32_t)g + k, min(kChunkRecs, r - k), 0u};
      ++c;
    }
    g += (int)r;
  }
}

}  // namespace
}  // namespace vms

extern "C" {

vms_dpt* vms_dpt_create(int32_t capacity, int32_t page_count, int32_t levels) {
  using namespace vms;
  if (capacity < 1 || capacity > kMaxCap || page_count < 1 || page_count >= (1 << 30) ||
      levels < 1 || levels > kMaxLevels) {
    set_error("dpt_create: capacity 1..%d, levels 1..%d required", kMaxCap, kMaxLevels);
    return nullptr;
  }
  vms_dpt* d = new vms_dpt{};
  d->C = capacity;
  d->P = page_count;
  d->L = levels;
  d->S = 1 << (levels - 1);
  d->W = (capacity + 31) / 32;
  d->WS = (d->W + 31) / 32;
  const size_t C = capacity, P1 = (size_t)page_count + 1;
  size_t pow2 = 1;  // global bitonic buffer: a power of two >= page count
  while (pow2 < P1) pow2 <<= 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_level = take(C), o_occ = take(C), o_freem = take(4 * C), o_last = take(4 * C),
               o_slots = take(4 * C * d->S), o_res = take(4 * P1),
               o_bm = take(4 * (size_t)(levels + 1) * d->W), o_lru0 = take(4 * C),
               o_lru1 = take(4 * C), o_cur = take(4), o_sk = take(8 * pow2),
               o_sv = take(4 * pow2), o_cnt = take(4 * 18),
               o_cs = take(8 * (P1 / 2048 + 2));
  if (cudaMalloc(&d->base, off) != cudaSuccess) {
    set_error("dpt_create: device allocation of %zu bytes failed", off);
    delete d;
    return nullptr;
  }
  char* b = static_cast<char*>(d->base);
  d->level = reinterpret_cast<int8_t*>(b + o_level);
  d->occ = reinterpret_cast<uint8_t*>(b + o_occ);
  d->freem = reinterpret_cast<uint32_t*>(b + o_freem);
  d->last = reinterpret_cast<int32_t*>(b + o_last);
  d->slots = reinterpret_cast<uint32_t*>(b + o_slots);
  d->res = reinterpret_cast<uint32_t*>(b + o_res);
  d->bm = reinterpret_cast<uint32_t*>(b + o_bm);
  d->lru[0] = reinterpret_cast<int32_t*>(b + o_lru0);
  d->lru[1] = reinterpret_cast<int32_t*>(b + o_lru1);
  d->cur = reinterpret_cast<int32_t*>(b + o_cur);
  d->skeys = reinterpret_cast<uint64_t*>(b + o_sk);
  d->svals = reinterpret_cast<uint32_t*>(b + o_sv);
  d->counts = reinterpret_cast<int32_t*>(b + o_cnt);
  d->csums = reinterpret_cast<uint2*>(b + o_cs);
  // initial state: every entry empty, LRU stamp -1, order by index
  std::vector<int8_t> lv(C, -1);
  std::vector<int32_t> last(C, -1), order(C);
  std::vector<uint32_t> bm((size_t)(levels + 1) * d->W, 0u), res(P1, kNone);
  for (size_t i = 0; i < C; ++i) {
    order[i] = (int32_t)i;
    bm[(size_t)levels * d->W + i / 32] |= 1u << (i % 32);
  }
  bool ok = cudaMemset(d->base, 0, off) == cudaSuccess;
  ok = ok && cudaMemcpy(d->level, lv.data(), C, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaMemcpy(d->last, last.data(), 4 * C, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaMemcpy(d->lru[0], order.data(), 4 * C, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaMemcpy(d->bm, bm.data(), 4 * bm.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaMemcpy(d->res, res.data(), 4 * P1, cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) {
    set_error("dpt_create: initialisation failed");
    cudaFree(d->base);
    delete d;
    return nullptr;
  }
  return d;
}

void vms_dpt_destroy(vms_dpt* d) {
  if (!d) return;
  cudaFree(d->base);
  delete d;
}

namespace {
size_t dpt_fixed_smem(const vms_dpt* d) {
  return 4 * (size_t)d->C + 4 * (size_t)(d->L + 2) * (d->W + d->WS) + 2 * (size_t)d->C + 64;
}
// the sort buffer: a power of two covering every page when that fits next
// to the table state (no larger - a big shared-memory footprint would make
// the update wait for an SM the render in flight has to give up), else the
// largest that fits (more required pages spill to global memory)
int dpt_sort_cap(const vms_dpt* d) {
  const size_t avail = 227 * 1024 - 2048 - dpt_fixed_smem(d);
  int cap = 256;
  while (cap < d->P + 1 && (size_t)(2 * cap) * 12 <= avail && cap < (1 << 16)) cap *= 2;
  return cap;
}
}  // namespace

size_t vms_dpt_smem_bytes(const vms_dpt* d) {
  if (!d) return 0;
  return (size_t)dpt_sort_cap(d) * 12 + dpt_fixed_smem(d);
}

int32_t vms_dpt_update(vms_dpt* d, const uint32_t* pid, const uint32_t* enc,
                       const uint8_t* direct, const uint8_t* level, const uint32_t* n_req,
                       const vms_dpt_frame* frame, uint32_t* plan_pid, uint8_t* plan_level,
                       int32_t* plan_entry, int32_t* plan_slot, int64_t plan_cap,
                       vms_dpt_stats* stats, void* stream) {
  using namespace vms;
  if (!d || !pid || !enc || !direct || !level || !n_req || !frame || !stats || plan_cap < 0 ||
      (plan_cap > 0 && (!plan_pid || !plan_level || !plan_entry || !plan_slot))) {
    set_error("dpt_update: invalid arguments");
    return VMS_ERR_INVALID;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DptArgs a{};
  a.C = d->C;
  a.P = d->P;
  a.L = d->L;
  a.S = d->S;
  a.W = d->W;
  a.WS = d->WS;
  a.level = d->level;
  a.occ = d->occ;
  a.freem = d->freem;
  a.last = d->last;
  a.slots = d->slots;
  a.res = d->res;
  a.bm = d->bm;
  a.lru0 = d->lru[0];
  a.lru1 = d->lru[1];
  a.cur = d->cur;
  a.skeys = d->skeys;
  a.svals = d->svals;
  a.counts = d->counts;
  a.pid = pid;
  a.enc = enc;
  a.direct = direct;
  a.lvl = level;
  a.n_req = n_req;
  a.frame = frame;
  a.plan_pid = plan_pid;
  a.plan_level = plan_level;
  a.plan_entry = plan_entry;
  a.plan_slot = plan_slot;
  a.plan_cap = plan_cap;
  a.stats = stats;
  a.sort_cap = dpt_sort_cap(d);
  const size_t smem = vms_dpt_smem_bytes(d);
  VMS_CUDA(cudaFuncSetAttribute(dpt_update_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  VMS_CUDA(launch(dpt_update_k, 1, kThreads, smem, s, a));
  mark("dpt_update", s);
  VMS_LAUNCH_CHECK("dpt_update");
  return VMS_OK;
}

int32_t vms_dpt_chunks(vms_dpt* d, uint32_t page_size, vms_chunk* out, int64_t cap,
                       vms_dpt_stats* stats, void* stream) {
  using namespace vms;
  if (!d || !out || !stats || cap < 1 || page_size < 1) {
    set_error("dpt_chunks: invalid arguments");
    return VMS_ERR_INVALID;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = (d->P + kChunkBlock - 1) / kChunkBlock;
  VMS_CUDA(launch(dpt_chunk_sums_k, nb, kChunkThreads, 0, s, (const uint32_t*)d->res,
                  (const int8_t*)d->level, d->P, page_size, d->csums));
  VMS_CUDA(launch(dpt_chunk_scan_k, 1, 1024, 0, s, d->csums, nb, stats));
  VMS_CUDA(launch(dpt_chunk_emit_k, nb, kChunkThreads, 0, s, (const uint32_t*)d->res,
                  (const int8_t*)d->level, d->P, page_size, (const uint2*)d->csums, out, cap));
  mark("dpt_chunks", s);
  VMS_LAUNCH_CHECK("dpt_chunks");
  return VMS_OK;
}

int32_t vms_dpt_state(const vms_dpt* d, int32_t* level, int64_t* last_used, uint32_t* slots,
                      int32_t max_slots, uint32_t* res, void* stream) {
  using namespace vms;
  if (!d || !level || !last_used || !slots || max_slots < d->S || !res) {
    set_error("dpt_state: invalid arguments");
    return VMS_ERR_INVALID;
  }
  (void)stream;  // the table may be updated on a session's own streams
  VMS_CUDA(cudaDeviceSynchronize());
  const size_t C = d->C;
  std::vector<int8_t> lv(C);
  std::vector<int32_t> last(C);
  std::vector<uint32_t> sl(C * d->S);
  VMS_CUDA(cudaMemcpy(lv.data(), d->level, C, cudaMemcpyDeviceToHost));
  VMS_CUDA(cudaMemcpy(last.data(), d->last, 4 * C, cudaMemcpyDeviceToHost));
  VMS_CUDA(cudaMemcpy(sl.data(), d->slots, 4 * C * d->S, cudaMemcpyDeviceToHost));
  VMS_CUDA(cudaMemcpy(res, d->res, 4 * ((size_t)d->P + 1), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < C; ++i) {
    level[i] = lv[i];
    last_used[i] = last[i];
    const int n = lv[i] >= 0 ? 1 << lv[i] : 0;
    for (int q = 0; q < max_slots; ++q)
      slots[i * max_slots + q] = q < n ? sl[i * d->S + q] : 0u;
  }
  return VMS_OK;
}

}  // extern "C"
