// Subsystems [1] + [2]: proxy-mesh page-ID visibility and required-page
// extraction.  Compiled with -fmad=false: every FP64 operation below follows
// the reference's NumPy/Cython arithmetic one rounding at a time, so page-ID
// images, depths and required lists are bit-exact with the CPU reference.
//
//  K1 vis_count_k / vis_emit_k  per-face near clip + projection
//        (pkg/src/vmsplat/render.py:256-304), scan-ordered emission so the
//        triangle order is (face, clip-fan) exactly as the reference builds it.
//  K2 vis_raster_k  16x16-pixel tile per CTA; each CTA compacts the
//        triangles overlapping its tile in index order and every pixel walks
//        that list sequentially - exact first-triangle-wins ties without
//        atomics (pkg/src/vmsplat/kernels/_core.pyx:81-159).
//        Fused epilogue K3: depth encode + per-page atomicMax + direct flag
//        (pkg/src/vmsplat/runtime.py:70-89), warp-aggregated with match_any.
//  K4 vis_links_k / vis_required_k  one-hop link expansion from the
//        pre-propagation snapshot, LOD level per page, ordered compaction of
//        the required list into host-mapped memory (runtime.py:89-96,129-132).
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "prims.h"
#include "vis.h"

namespace vms {

namespace {

constexpr int kVisTile = 16;
constexpr int kVisThreads = kVisTile * kVisTile;

struct View3 {
  double x, y, z;
};

__device__ __forceinline__ View3 to_view(const VisCamera& c, const double* p) {
  const double d0 = dsub(p[0], c.pos[0]);
  const double d1 = dsub(p[1], c.pos[1]);
  const double d2 = dsub(p[2], c.pos[2]);
  View3 v;
  v.x = dot3(c.dot_mode, d0, d1, d2, c.rot[0], c.rot[3], c.rot[6]);
  v.y = dot3(c.dot_mode, d0, d1, d2, c.rot[1], c.rot[4], c.rot[7]);
  v.z = dot3(c.dot_mode, d0, d1, d2, c.rot[2], c.rot[5], c.rot[8]);
  return v;
}

__device__ __forceinline__ View3 lerp_near(const View3& a, const View3& b, double near) {
  const double t = ddiv(dsub(near, a.z), dsub(b.z, a.z));
  View3 r;
  r.x = dadd(a.x, dmul(t, dsub(b.x, a.x)));
  r.y = dadd(a.y, dmul(t, dsub(b.y, a.y)));
  r.z = dadd(a.z, dmul(t, dsub(b.z, a.z)));
  return r;
}

// Clip one view-space triangle at z = near into a polygon of 0, 3 or 4
// corners (render.py:256-276); the fan from poly[0] gives 0..2 triangles.
__device__ __forceinline__ int clip_poly(const View3* v, double near, View3* poly) {
  const bool in0 = v[0].z > near, in1 = v[1].z > near, in2 = v[2].z > near;
  const int n_in = (int)in0 + (int)in1 + (int)in2;
  if (n_in == 0) return 0;
  if (n_in == 3) {
    poly[0] = v[0];
    poly[1] = v[1];
    poly[2] = v[2];
    return 3;
  }
  const bool ins[3] = {in0, in1, in2};
  int k = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const View3& a = v[i];
    const View3& b = v[(i + 1) % 3];
    if (ins[i]) poly[k++] = a;
    if (ins[i] != ins[(i + 1) % 3]) poly[k++] = lerp_near(a, b, near);
  }
  return k;
}

__device__ __forceinline__ void face_view(const VisCamera& c, const double* verts,
                                          const int32_t* faces, uint32_t f, View3* v) {
#pragma unroll
  for (int j = 0; j < 3; ++j) v[j] = to_view(c, verts + 3 * (int64_t)faces[3 * f + j]);
}

__global__ void vis_count_k(const VisFrameDev* __restrict__ fd, const double* __restrict__ verts,
                            const int32_t* __restrict__ faces, uint32_t nf,
                            uint32_t* __restrict__ counts) {
  pdl_wait();
  __shared__ VisCamera cam;
  if (threadIdx.x == 0) cam = fd->cam;
  __syncthreads();
  uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  View3 v[3], poly[4];
  face_view(cam, verts, faces, f, v);
  int k = clip_poly(v, cam.near, poly);
  counts[f] = k >= 3 ? (uint32_t)(k - 2) : 0u;
}

// Setup of one screen-space triangle exactly as _core.pyx:105-143 does it.
__device__ __forceinline__ void setup_tri(double ax, double ay, double iza, double bx,
                                          double by, double izb, double cx, double cy,
                                          double izc, uint32_t id, int w, int h,
                                          VisTri* out) {
  double area = dsub(dmul(dsub(bx, ax), dsub(cy, ay)), dmul(dsub(by, ay), dsub(cx, ax)));
  VisTri t;
  t.id = id;
  t.x0 = 1;
  t.x1 = 0;  // empty unless proven otherwise
  t.y0 = 1;
  t.y1 = 0;
  if (area != 0.0) {
    if (area < 0.0) {
      double s;
      s = bx; bx = cx; cx = s;
      s = by; by = cy; cy = s;
      s = izb; izb = izc; izc = s;
      area = -area;
    }
    const double mnx = fmin(ax, fmin(bx, cx)), mxx = fmax(ax, fmax(bx, cx));
    const double mny = fmin(ay, fmin(by, cy)), mxy = fmax(ay, fmax(by, cy));
    double fx0 = floor(dsub(mnx, 0.5)), fx1 = ceil(dsub(mxx, 0.5));
    double fy0 = floor(dsub(mny, 0.5)), fy1 = ceil(dsub(mxy, 0.5));
    if (fx0 < 0.0) fx0 = 0.0;
    if (fy0 < 0.0) fy0 = 0.0;
    if (fx1 > (double)(w - 1)) fx1 = (double)(w - 1);
    if (fy1 > (double)(h - 1)) fy1 = (double)(h - 1);
    if (!(fx1 < fx0 || fy1 < fy0)) {
      t.x0 = (int)fx0;
      t.x1 = (int)fx1;
      t.y0 = (int)fy0;
      t.y1 = (int)fy1;
    }
  }
  t.ax = ax; t.ay = ay; t.bx = bx; t.by = by; t.cx = cx; t.cy = cy;
  t.iza = iza; t.izb = izb; t.izc = izc; t.area = area;
  *out = t;
}

__device__ __forceinline__ void to_pixels(const VisCamera& c, const View3& v, double* x,
                                          double* y, double* iz) {
  *x = dadd(ddiv(dmul(c.focal, v.x), v.z), c.half_w);
  *y = dadd(ddiv(dmul(c.focal, v.y), v.z), c.half_h);
  *iz = ddiv(1.0, v.z);
}

__global__ void vis_emit_k(const VisFrameDev* __restrict__ fd, const double* __restrict__ verts,
                           const int32_t* __restrict__ faces,
                           const uint32_t* __restrict__ face_page, uint32_t nf,
                           const uint32_t* __restrict__ offsets, VisTri* __restrict__ tris) {
  pdl_wait();
  __shared__ VisCamera cam;
  if (threadIdx.x == 0) cam = fd->cam;
  __syncthreads();
  uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  View3 v[3], poly[4];
  face_view(cam, verts, faces, f, v);
  int k = clip_poly(v, cam.near, poly);
  uint32_t o = offsets[f];
  for (int i = 1; i + 1 < k; ++i) {
    double x[3], y[3], z[3];
    to_pixels(cam, poly[0], &x[0], &y[0], &z[0]);
    to_pixels(cam, poly[i], &x[1], &y[1], &z[1]);
    to_pixels(cam, poly[i + 1], &x[2], &y[2], &z[2]);
    setup_tri(x[0], y[0], z[0], x[1], y[1], z[1], x[2], y[2], z[2], face_page[f],
              cam.width, cam.height, &tris[o + i - 1]);
  }
}

constexpr int kFrontThreads = 1024;
constexpr uint32_t kBackMaxPages = 32767;   // page depths in <= 128 KB of shared memory

__device__ __forceinline__ uint32_t block_scan_1024(uint32_t v, uint32_t* scratch,
                                                    uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t wv = scratch[lane];
    uint32_t wi = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    scratch[lane] = wi - wv;
    if (lane == 31) scratch[32] = wi;
  }
  __syncthreads();
  const uint32_t ex = scratch[warp] + inc - v;
  *total = scratch[32];
  __syncthreads();
  return ex;
}

// Single-CTA fused back end for up to kBackMaxPages pages: one-hop link
// expansion from the pre-propagation snapshot (shared-memory atomics),
// required flags, the ordered compaction and the LOD level per page -
// replacing a copy, vis_links_k, vis_flags_k, the scan and vis_required_k.
__global__ void __launch_bounds__(kFrontThreads) vis_back_k(
    const uint32_t* __restrict__ base, const uint8_t* __restrict__ direct,
    const uint32_t* __restrict__ link_off, const uint32_t* __restrict__ link_tgt,
    uint32_t page_count, const VisFrameDev* __restrict__ fd, uint32_t* __restrict__ depth_g,
    uint32_t* __restrict__ meta, RequiredOut out) {
  pdl_wait();
  extern __shared__ uint32_t dep[];  // page_count + 1 words
  __shared__ uint32_t scratch[33];
  for (uint32_t p = threadIdx.x; p <= page_count; p += kFrontThreads) dep[p] = base[p];
  __syncthreads();
  // links (runtime.py:89-96): targets pull the source's snapshot depth
  for (uint32_t p = 1 + threadIdx.x; p <= page_count; p += kFrontThreads) {
    if (!direct[p]) continue;
    const uint32_t src = base[p];
    for (uint32_t i = link_off[p - 1]; i < link_off[p]; ++i) {
      const uint32_t q = link_tgt[i];
      if (q != p && q >= 1 && q <= page_count) atomicMax(&dep[q], src);
    }
  }
  __syncthreads();
  const VisLod& lod = fd->lod;
  uint32_t run = 0;
  for (uint32_t p0 = 0; p0 <= page_count; p0 += kFrontThreads) {
    const uint32_t p = p0 + threadIdx.x;
    const uint32_t e = (p >= 1 && p <= page_count) ? dep[p] : 0u;
    if (p <= page_count) depth_g[p] = e;
    uint32_t tot;
    const uint32_t o = run + block_scan_1024(e ? 1u : 0u, scratch, &tot);
    if (e) {
      // select_lod: level = #thresholds strictly below the decoded depth
      const double d = (double)__uint_as_float(0xFFFFFFFFu - e);
      uint8_t level = 0;
      for (int k = 0; k < lod.count; ++k) level += lod.thresholds[k] < d ? 1 : 0;
      out.pid[o] = p;
      out.enc[o] = e;
      out.direct[o] = direct[p];
      out.level[o] = level;
    }
    run += tot;
  }
  if (threadIdx.x == 0) {
    meta[1] = run;  // required pages
    // the host's copy of the counts: plain stores into the mapped words (no
    // copy-engine transfer that could queue behind a frame's image copy)
    if (out.meta) {
      out.meta[0] = meta[0];
      out.meta[1] = run;
      out.meta[2] = meta[2];
      out.meta[3] = meta[3];
    }
  }
}

__global__ void vis_setup_raw_k(const double* __restrict__ raw, const uint32_t* __restrict__ ids,
                                uint32_t n, int w, int h, VisTri* __restrict__ tris) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* r = raw + 9 * (int64_t)i;
  setup_tri(r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7], r[8], ids[i], w, h, &tris[i]);
}

// Binned raster for large proxy meshes (C4: 600K faces).  Each clipped
// triangle is listed under every 16x16 raster tile its pixel box touches;
// a stable radix sort by tile keeps each tile's list in triangle order, so
// the raster walks only its own list and the first-triangle-wins rule is
// unchanged.  Triangles with an empty box (off screen) are listed nowhere.
__device__ __forceinline__ uint32_t tri_tiles(const int4 b, int* tx0, int* ty0, int* tx1,
                                              int* ty1) {
  if (b.x > b.y || b.z > b.w) return 0u;
  *tx0 = b.x / kVisTile;
  *tx1 = b.y / kVisTile;
  *ty0 = b.z / kVisTile;
  *ty1 = b.w / kVisTile;
  return (uint32_t)(*tx1 - *tx0 + 1) * (uint32_t)(*ty1 - *ty0 + 1);
}

__global__ void vis_bin_count_k(const VisTri* __restrict__ tris,
                                const uint32_t* __restrict__ n_tris, uint32_t* __restrict__ cnt) {
  pdl_wait();
  const uint32_t n = *n_tris;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int4 b = __ldg(reinterpret_cast<const int4*>(&tris[i].x0));
    int a0, a1, c0, c1;
    cnt[i] = tri_tiles(b, &a0, &c0, &a1, &c1);
  }
}

__global__ void vis_bin_emit_k(const VisTri* __restrict__ tris,
                               const uint32_t* __restrict__ n_tris,
                               const uint32_t* __restrict__ off, const uint32_t* __restrict__ n_pairs,
                               uint32_t pair_cap, int tiles_x, uint32_t* __restrict__ keys,
                               uint32_t* __restrict__ vals) {
  pdl_wait();
  const uint32_t n = *n_tris;
  if (*n_pairs > pair_cap) return;  // the raster walks every triangle instead
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int4 b = __ldg(reinterpret_cast<const int4*>(&tris[i].x0));
    int x0, y0, x1, y1;
    if (!tri_tiles(b, &x0, &y0, &x1, &y1)) continue;
    uint32_t o = off[i];
    for (int ty = y0; ty <= y1; ++ty)
      for (int tx = x0; tx <= x1; ++tx) {
        keys[o] = (uint32_t)(ty * tiles_x + tx);
        vals[o] = i;
        ++o;
      }
  }
}

// [start, end) of every tile's run in the sorted pair list.
__global__ void vis_bin_ranges_k(const uint32_t* __restrict__ keys,
                                 const uint32_t* __restrict__ n_pairs, uint32_t pair_cap,
                                 uint2* __restrict__ ranges) {
  pdl_wait();
  const uint32_t n = *n_pairs;
  if (n > pair_cap) return;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t k = keys[j];
    if (j == 0 || keys[j - 1] != k) ranges[k].x = j;
    if (j + 1 == n || keys[j + 1] != k) ranges[k].y = j + 1;
  }
}

struct VisBins {
  const uint32_t* vals;     // sorted triangle indices (nullptr: unbinned raster)
  const uint2* ranges;      // per raster tile
  const uint32_t* n_pairs;
  uint32_t pair_cap;
};

struct RasterSmem {
  VisTri stri[kVisThreads];
  uint32_t sidx[4 * kVisThreads];
  uint32_t wsum[kVisThreads / 32];
};

// The triangles [first, n) of `list` (or of the triangle array itself when
// list == nullptr) against the CTA's 16x16 tile at (tx0, ty0): each pixel
// keeps the nearest 1/z, the first triangle in order winning ties (strict >,
// _core.pyx:150-159).  CTA-uniform arguments; every thread calls it.
__device__ __forceinline__ void raster_range(const VisTri* __restrict__ tris,
                                             const uint32_t* __restrict__ list, uint32_t first,
                                             uint32_t n, int tx0, int ty0, int w, int h,
                                             RasterSmem& sm, uint32_t& best_id,
                                             double& best_z) {
  constexpr int kBoxes = 4;  // triangle boxes tested per thread per round
  const int tx1 = min(tx0 + kVisTile, w) - 1, ty1 = min(ty0 + kVisTile, h) - 1;
  const int px = tx0 + (threadIdx.x & (kVisTile - 1));
  const int py = ty0 + (threadIdx.x / kVisTile);
  const bool inside_img = px < w && py < h;
  const double fx = (double)px + 0.5, fy = (double)py + 0.5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t base = first; base < n; base += kBoxes * kVisThreads) {
    // test kBoxes 16-byte boxes per thread (loads in flight together) and
    // compact the indices of the triangles touching this tile, in order
    bool hit[kBoxes];
    uint32_t tid[kBoxes];
#pragma unroll
    for (int k = 0; k < kBoxes; ++k) {
      const uint32_t li = base + k * kVisThreads + threadIdx.x;
      hit[k] = false;
      tid[k] = li;
      if (li < n) {
        const uint32_t ti = list ? __ldg(list + li) : li;
        tid[k] = ti;
        const int4 bx = __ldg(reinterpret_cast<const int4*>(&tris[ti].x0));
        hit[k] = bx.x <= bx.y && bx.x <= tx1 && bx.y >= tx0 && bx.z <= ty1 && bx.w >= ty0;
      }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < kBoxes; ++k) {
      const uint32_t bal = __ballot_sync(0xffffffffu, hit[k]);
      if (lane == 0) sm.wsum[warp] = __popc(bal);
      __syncthreads();
      uint32_t pre = 0, tot = 0;
#pragma unroll
      for (int q = 0; q < kVisThreads / 32; ++q) {
        const uint32_t c = sm.wsum[q];
        pre += q < warp ? c : 0u;
        tot += c;
      }
      if (hit[k]) sm.sidx[cnt + pre + __popc(bal & lanemask_lt())] = tid[k];
      cnt += tot;
      __syncthreads();
    }
    // the hits, kVisThreads at a time: stage the triangles, then every pixel
    // walks them in index order (strict > keeps the first triangle on ties)
    for (uint32_t h0 = 0; h0 < cnt; h0 += kVisThreads) {
      const uint32_t m = min(cnt - h0, (uint32_t)kVisThreads);
      if (threadIdx.x < m) sm.stri[threadIdx.x] = tris[sm.sidx[h0 + threadIdx.x]];
      __syncthreads();
      if (inside_img) {
        for (uint32_t j = 0; j < m; ++j) {
          const VisTri& q = sm.stri[j];
          if (px < q.x0 || px > q.x1 || py < q.y0 || py > q.y1) continue;
          const double e0 = dsub(dmul(dsub(q.cx, q.bx), dsub(fy, q.by)),
                                 dmul(dsub(q.cy, q.by), dsub(fx, q.bx)));
          if (e0 < 0.0) continue;
          const double e1 = dsub(dmul(dsub(q.ax, q.cx), dsub(fy, q.cy)),
                                 dmul(dsub(q.ay, q.cy), dsub(fx, q.cx)));
          if (e1 < 0.0) continue;
          const double e2 = dsub(dmul(dsub(q.bx, q.ax), dsub(fy, q.ay)),
                                 dmul(dsub(q.by, q.ay), dsub(fx, q.ax)));
          if (e2 < 0.0) continue;
          const double iz =
              ddiv(dadd(dadd(dmul(e0, q.iza), dmul(e1, q.izb)), dmul(e2, q.izc)), q.area);
          if (iz > best_z) {
            best_z = iz;
            best_id = q.id;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Per-pixel outputs of the raster: the images (when asked) and K3, the fused
// depth encode + per-page max + direct flag (runtime.py:26-43,70-89,
// render.py:305-307), warp-aggregated with match_any.
__device__ __forceinline__ void raster_epilogue(int tx0, int ty0, int w, int h,
                                                uint32_t best_id, double best_z,
                                                uint32_t* __restrict__ id_image,
                                                double* __restrict__ invz_image,
                                                uint32_t page_count,
                                                uint32_t* __restrict__ page_depth,
                                                uint8_t* __restrict__ page_direct,
                                                uint32_t* __restrict__ err) {
  const int px = tx0 + (threadIdx.x & (kVisTile - 1));
  const int py = ty0 + (threadIdx.x / kVisTile);
  const bool inside_img = px < w && py < h;
  const int lane = threadIdx.x & 31;
  if (inside_img) {
    if (id_image) id_image[(int64_t)py * w + px] = best_id;
    if (invz_image) invz_image[(int64_t)py * w + px] = best_z;
  }
  if (!page_depth) return;
  uint32_t pid = inside_img ? best_id : 0u;
  if (pid > page_count) {
    atomicMax(err, pid);
    pid = 0;
  }
  uint32_t enc = 0;
  if (pid) {
    const float d32 = __double2float_rn(ddiv(1.0, best_z));
    enc = 0xFFFFFFFFu - __float_as_uint(d32);
  }
  const uint32_t peers = __match_any_sync(0xffffffffu, pid);
  if (pid) {
    const uint32_t mx = __reduce_max_sync(peers, enc);
    if (lane == __ffs(peers) - 1) {
      atomicMax(&page_depth[pid], mx);
      page_direct[pid] = 1;
    }
  }
}

// Whole-list raster: one CTA per 16x16 tile walks every triangle (small
// meshes) and writes the outputs.
__global__ void __launch_bounds__(kVisThreads) vis_raster_k(
    const VisTri* __restrict__ tris, const uint32_t* __restrict__ n_tris_dev, uint32_t n_host,
    int w, int h, uint32_t* __restrict__ id_image, double* __restrict__ invz_image,
    int init_from_images, uint32_t page_count, uint32_t* __restrict__ page_depth,
    uint8_t* __restrict__ page_direct, uint32_t* __restrict__ err) {
  pdl_wait();
  __shared__ RasterSmem sm;
  const int tx0 = blockIdx.x * kVisTile, ty0 = blockIdx.y * kVisTile;
  const int px = tx0 + (threadIdx.x & (kVisTile - 1));
  const int py = ty0 + (threadIdx.x / kVisTile);
  uint32_t best_id = 0;
  double best_z = 0.0;
  if (init_from_images && px < w && py < h) {
    best_id = id_image[(int64_t)py * w + px];
    best_z = invz_image[(int64_t)py * w + px];
  }
  const uint32_t n = n_tris_dev ? *n_tris_dev : n_host;
  raster_range(tris, nullptr, 0, n, tx0, ty0, w, h, sm, best_id, best_z);
  raster_epilogue(tx0, ty0, w, h, best_id, best_z, id_image, invz_image, page_count, page_depth,
                  page_direct, err);
}

// Binned raster, work items = (tile, chunk of <= kVisChunk of the tile's
// list entries).  The nearest-with-first-wins rule is a reduction: (z, i)
// beats (z', i') iff z > z' or (z == z' and i < i'), so a long list (the
// vanishing point of a street: 10^5 triangles in one tile) is split over many
// CTAs; a tile of one chunk writes its outputs directly, the chunks of a
// longer list write per-pixel partials that vis_merge_k folds in chunk order.
constexpr uint32_t kVisChunk = 2048;

struct VisPartial {
  double z;
  uint32_t id;
  uint32_t pad_;
};

__global__ void vis_chunk_count_k(const uint2* __restrict__ ranges, uint32_t tiles,
                                  const uint32_t* __restrict__ n_pairs, uint32_t pair_cap,
                                  uint32_t* __restrict__ nchunk, uint32_t* __restrict__ slot,
                                  uint32_t* __restrict__ slot_ctr, uint32_t slot_cap) {
  pdl_wait();
  const bool ok = *n_pairs <= pair_cap;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < tiles;
       t += gridDim.x * blockDim.x) {
    uint32_t c = 1;
    if (ok) {
      const uint2 r = ranges[t];
      const uint32_t len = r.y - r.x;
      if (len > kVisChunk) {
        c = (len + kVisChunk - 1) / kVisChunk;
        const uint32_t b = atomicAdd(slot_ctr, c);
        if (b + c > slot_cap) {
          c = 1;  // out of partial slots: this tile walks its list in one CTA
        } else {
          slot[t] = b;
        }
      }
    }
    nchunk[t] = c;
  }
}

__global__ void __launch_bounds__(kVisThreads) vis_raster_items_k(
    const VisTri* __restrict__ tris, const uint32_t* __restrict__ n_tris_dev, int w, int h,
    int tiles_x, uint32_t tiles, VisBins bins, const uint32_t* __restrict__ nchunk,
    const uint32_t* __restrict__ chunk_off, const uint32_t* __restrict__ n_items,
    const uint32_t* __restrict__ slot, VisPartial* __restrict__ partial,
    uint32_t* __restrict__ id_image, double* __restrict__ invz_image, uint32_t page_count,
    uint32_t* __restrict__ page_depth, uint8_t* __restrict__ page_direct,
    uint32_t* __restrict__ err) {
  pdl_wait();
  __shared__ RasterSmem sm;
  const bool binned = *bins.n_pairs <= bins.pair_cap;
  const uint32_t items = binned ? *n_items : tiles;
  for (uint32_t it = blockIdx.x; it < items; it += gridDim.x) {
    uint32_t t = it, c = 0;
    if (binned) {
      // the tile whose chunk range holds item `it` (chunk_off is ascending)
      uint32_t lo = 0, hi = tiles;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (chunk_off[mid] <= it) lo = mid; else hi = mid;
      }
      t = lo;
      c = it - chunk_off[t];
    }
    const int tx0 = (int)(t % tiles_x) * kVisTile, ty0 = (int)(t / tiles_x) * kVisTile;
    uint32_t best_id = 0;
    double best_z = 0.0;
    if (binned) {
      const uint2 r = bins.ranges[t];
      const uint32_t a = r.x + c * kVisChunk;
      const uint32_t b = nchunk[t] > 1 ? min(r.y, a + kVisChunk) : r.y;
      raster_range(tris, bins.vals, a, b, tx0, ty0, w, h, sm, best_id, best_z);
    } else {  // the pair list overflowed: walk every triangle
      raster_range(tris, nullptr, 0, *n_tris_dev, tx0, ty0, w, h, sm, best_id, best_z);
    }
    if (!binned || nchunk[t] == 1) {
      raster_epilogue(tx0, ty0, w, h, best_id, best_z, id_image, invz_image, page_count,
                      page_depth, page_direct, err);
    } else {
      VisPartial pt;
      pt.z = best_z;
      pt.id = best_id;
      pt.pad_ = 0;
      partial[(size_t)(slot[t] + c) * kVisThreads + threadIdx.x] = pt;
    }
  }
}

__global__ void __launch_bounds__(kVisThreads) vis_merge_k(
    int w, int h, int tiles_x, uint32_t tiles, const uint32_t* __restrict__ n_pairs,
    uint32_t pair_cap, const uint32_t* __restrict__ nchunk, const uint32_t* __restrict__ slot,
    const VisPartial* __restrict__ partial, uint32_t* __restrict__ id_image,
    double* __restrict__ invz_image, uint32_t page_count, uint32_t* __restrict__ page_depth,
    uint8_t* __restrict__ page_direct, uint32_t* __restrict__ err) {
  pdl_wait();
  if (*n_pairs > pair_cap) return;
  for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const uint32_t c = nchunk[t];
    if (c <= 1) continue;
    uint32_t best_id = 0;
    double best_z = 0.0;
    const VisPartial* p = partial + (size_t)slot[t] * kVisThreads + threadIdx.x;
    for (uint32_t k = 0; k < c; ++k) {  // chunk order: earlier chunks win ties
      const VisPartial q = p[(size_t)k * kVisThreads];
      if (q.z > best_z) {
        best_z = q.z;
        best_id = q.id;
      }
    }
    const int tx0 = (int)(t % tiles_x) * kVisTile, ty0 = (int)(t / tiles_x) * kVisTile;
    raster_epilogue(tx0, ty0, w, h, best_id, best_z, id_image, invz_image, page_count,
                    page_depth, page_direct, err);
  }
}

// Standalone reduce_visibility over given images (runtime.py:70-89).
__global__ void vis_reduce_images_k(const uint32_t* __restrict__ ids,
                                    const double* __restrict__ depth, uint64_t n_px,
                                    uint32_t page_count, uint32_t* __restrict__ page_depth,
                                    uint8_t* __restrict__ page_direct, uint32_t* __restrict__ err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_px;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t pid = ids[i];
    if (!pid) continue;
    if (pid > page_count) {
      atomicMax(err, pid);
      continue;
    }
    const uint32_t enc = 0xFFFFFFFFu - __float_as_uint(__double2float_rn(depth[i]));
    atomicMax(&page_depth[pid], enc);
    page_direct[pid] = 1;
  }
}

__global__ void vis_links_k(const uint32_t* __restrict__ base, uint32_t* __restrict__ depth,
                            const uint8_t* __restrict__ direct,
                            const uint32_t* __restrict__ link_off,
                            const uint32_t* __restrict__ link_tgt, uint32_t page_count) {
  // one warp per page; lanes stride the page's link list
  const uint32_t p = 1 + (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (p > page_count || !direct[p]) return;
  const uint32_t src = base[p];
  const uint32_t a = link_off[p - 1], b = link_off[p];
  for (uint32_t i = a + (threadIdx.x & 31); i < b; i += 32) {
    const uint32_t q = link_tgt[i];
    if (q != p && q >= 1 && q <= page_count) atomicMax(&depth[q], src);
  }
}

__global__ void vis_flags_k(const uint32_t* __restrict__ depth, uint32_t page_count,
                            uint32_t* __restrict__ flags) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > page_count) return;
  flags[p] = (p > 0 && depth[p] != 0u) ? 1u : 0u;
}

__global__ void vis_required_k(const uint32_t* __restrict__ depth,
                               const uint8_t* __restrict__ direct,
                               const uint32_t* __restrict__ pos, uint32_t page_count,
                               const VisFrameDev* __restrict__ fd, RequiredOut out) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p == 0 || p > page_count) return;
  const VisLod& lod = fd->lod;
  const uint32_t e = depth[p];
  if (!e) return;
  const uint32_t o = pos[p];
  // select_lod: level = #thresholds strictly below the decoded depth
  const double d = (double)__uint_as_float(0xFFFFFFFFu - e);
  uint8_t level = 0;
  for (int k = 0; k < lod.count; ++k) level += lod.thresholds[k] < d ? 1 : 0;
  out.pid[o] = p;
  out.enc[o] = e;
  out.direct[o] = direct[p];
  out.level[o] = level;
}

}  // namespace

// Binned raster (per-tile triangle lists) for large proxy meshes; the
// walk-everything raster is cheaper below ~64K faces (C2 2K, C3 20K).
// VMSPLAT_VIS_BIN=0/1 forces it off/on.
bool vis_binned(uint32_t n_faces) {
  static int force = -2;
  if (force == -2) {
    const char* e = getenv("VMSPLAT_VIS_BIN");
    force = (e && *e) ? (atoi(e) ? 1 : 0) : -1;
  }
  return force >= 0 ? force == 1 : n_faces >= 65536u;
}

constexpr uint32_t kVisMaxTiles = 1u << 16;  // 16-bit tile keys: 2 radix passes

uint32_t vis_pair_cap(uint32_t n_faces) {
  const uint64_t c = 8ull * n_faces;
  return (uint32_t)(c < (1u << 20) ? (1u << 20) : (c > (1ull << 30) ? (1ull << 30) : c));
}

// Partial-result slots of the chunked raster: a tile of more than one chunk
// uses one slot per chunk, so sum(slots) <= 2 * pairs / kVisChunk.
uint32_t vis_slot_cap(uint32_t n_faces) { return 2 * (vis_pair_cap(n_faces) / kVisChunk) + 64; }

size_t vis_bin_bytes(uint32_t n_faces) {
  if (!vis_binned(n_faces)) return 0;
  const uint32_t nt = 2 * n_faces + 1, cap = vis_pair_cap(n_faces);
  size_t b = sizeof(uint32_t) * (size_t)nt * 2;   // per-triangle counts + offsets
  b += sizeof(uint32_t) * 4;                       // n_pairs
  b += sizeof(uint32_t) * (size_t)cap * 4;         // keys/vals ping-pong
  b += sizeof(uint2) * kVisMaxTiles;               // tile ranges
  b += radix_ws_bytes(cap) + scan_ws_bytes(nt);
  // chunked raster: per-tile chunk counts, offsets, partial slots; partials
  b += sizeof(uint32_t) * (size_t)kVisMaxTiles * 3 + sizeof(uint32_t) * 4;
  b += scan_ws_bytes(kVisMaxTiles);
  b += sizeof(VisPartial) * kVisThreads * (size_t)vis_slot_cap(n_faces);
  return b + 16 * 256;
}

size_t vis_ws_bytes(uint32_t n_faces, uint32_t page_count) {
  size_t b = vis_bin_bytes(n_faces);
  b += sizeof(uint32_t) * (n_faces + 1) * 2;        // counts + offsets
  b += sizeof(uint32_t) * 4;                         // n_tris, n_req
  b += sizeof(VisTri) * ((size_t)n_faces * 2 + 1);   // clipped triangles
  b += sizeof(uint32_t) * (page_count + 1) * 3;      // base, depth, flags/pos
  b += sizeof(uint8_t) * (page_count + 1);           // direct
  b += scan_ws_bytes(n_faces > page_count + 1 ? n_faces : page_count + 1) + 1024;
  b += sizeof(VisFrameDev);
  return b + 8 * 256;
}

namespace {
struct VisWs {
  uint32_t *counts, *offsets, *n_tris, *n_req, *base, *depth, *pos, *err;
  VisTri* tris;
  uint8_t* direct;
  void* scan;
  VisFrameDev* fd;
  // binned raster (nullptr when the mesh is small)
  uint32_t *bcnt, *boff, *n_pairs, *k0, *v0, *k1, *v1;
  uint2* ranges;
  void *radix, *scan2;
  uint32_t pair_cap;
  uint32_t *nchunk, *chunk_off, *slot, *ictr;  // ictr: [0] items, [1] slot counter
  void* scan3;
  VisPartial* partial;
  uint32_t slot_cap;
};

template <typename T>
T* carve(char*& p, size_t n) {
  uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255);
  T* r = reinterpret_cast<T*>(a);
  p = reinterpret_cast<char*>(a + sizeof(T) * n);
  return r;
}

VisWs carve_ws(void* ws, uint32_t nf, uint32_t P) {
  char* p = static_cast<char*>(ws);
  VisWs w;
  w.counts = carve<uint32_t>(p, nf + 1);
  w.offsets = carve<uint32_t>(p, nf + 1);
  w.n_tris = carve<uint32_t>(p, 4);
  w.n_req = w.n_tris + 1;
  w.err = w.n_tris + 2;
  w.tris = carve<VisTri>(p, (size_t)nf * 2 + 1);
  w.base = carve<uint32_t>(p, P + 1);
  w.depth = carve<uint32_t>(p, P + 1);
  w.pos = carve<uint32_t>(p, P + 1);
  w.direct = carve<uint8_t>(p, P + 1);
  w.scan = carve<char>(p, scan_ws_bytes(nf > P + 1 ? nf : P + 1));
  w.fd = carve<VisFrameDev>(p, 1);
  w.bcnt = w.boff = w.n_pairs = w.k0 = w.v0 = w.k1 = w.v1 = nullptr;
  w.ranges = nullptr;
  w.radix = w.scan2 = w.scan3 = nullptr;
  w.pair_cap = w.slot_cap = 0;
  w.nchunk = w.chunk_off = w.slot = w.ictr = nullptr;
  w.partial = nullptr;
  if (vis_binned(nf)) {
    const uint32_t nt = 2 * nf + 1;
    w.pair_cap = vis_pair_cap(nf);
    w.bcnt = carve<uint32_t>(p, nt);
    w.boff = carve<uint32_t>(p, nt);
    w.n_pairs = carve<uint32_t>(p, 4);
    w.k0 = carve<uint32_t>(p, w.pair_cap);
    w.v0 = carve<uint32_t>(p, w.pair_cap);
    w.k1 = carve<uint32_t>(p, w.pair_cap);
    w.v1 = carve<uint32_t>(p, w.pair_cap);
    w.ranges = carve<uint2>(p, kVisMaxTiles);
    w.radix = carve<char>(p, radix_ws_bytes(w.pair_cap));
    w.scan2 = carve<char>(p, scan_ws_bytes(nt));
    w.nchunk = carve<uint32_t>(p, kVisMaxTiles);
    w.chunk_off = carve<uint32_t>(p, kVisMaxTiles);
    w.slot = carve<uint32_t>(p, kVisMaxTiles);
    w.ictr = carve<uint32_t>(p, 4);
    w.scan3 = carve<char>(p, scan_ws_bytes(kVisMaxTiles));
    w.slot_cap = vis_slot_cap(nf);
    w.partial = carve<VisPartial>(p, (size_t)kVisThreads * w.slot_cap);
  }
  return w;
}
}  // namespace

int32_t vis_init() {
  static bool done = false;
  if (done) return VMS_OK;
  VMS_CUDA(cudaFuncSetAttribute((const void*)vis_back_k,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(sizeof(uint32_t) * (kBackMaxPages + 1))));
  done = true;
  return VMS_OK;
}

uint32_t* vis_meta_dev(void* ws, uint32_t n_faces, uint32_t page_count) {
  return carve_ws(ws, n_faces, page_count).n_tris;
}

VisFrameDev* vis_frame_dev(void* ws, uint32_t n_faces, uint32_t page_count) {
  return carve_ws(ws, n_faces, page_count).fd;
}

int32_t vis_frame(const VisArgs& a, cudaStream_t s) {
  VisFrameDev f{};
  f.cam = a.cam;
  f.lod = a.lod;
  VMS_CUDA(cudaMemcpyAsync(vis_frame_dev(a.workspace, a.n_faces, a.page_count), &f,
                           sizeof(VisFrameDev), cudaMemcpyHostToDevice, s));
  return vis_launch(a, s);
}

int32_t vis_launch(const VisArgs& a, cudaStream_t s) {
  if (const int32_t rc = vis_init()) return rc;
  if (a.n_faces && (!a.verts || !a.faces || !a.face_page)) {
    set_error("vis_frame: null mesh pointer");
    return VMS_ERR_INVALID;
  }
  VisWs w = carve_ws(a.workspace, a.n_faces, a.page_count);
  const int T = 256;
  mark("begin", s);
  // page sets up to kBackMaxPages: a single-CTA fused back end (links,
  // flags, compaction, LOD) after the raster
  const bool back = a.page_count <= kBackMaxPages;
  // all memsets first: the kernels then chain with programmatic launches
  VMS_CUDA(cudaMemsetAsync(w.n_tris, 0, sizeof(uint32_t) * 4, s));
  VMS_CUDA(cudaMemsetAsync(w.base, 0, sizeof(uint32_t) * (a.page_count + 1), s));
  VMS_CUDA(cudaMemsetAsync(w.direct, 0, a.page_count + 1, s));
  const uint32_t scan_n = a.n_faces > a.page_count + 1 ? a.n_faces : a.page_count + 1;
  VMS_CUDA(cudaMemsetAsync(w.scan, 0, scan_ws_bytes(scan_n), s));
  if (w.bcnt && a.n_faces) {
    VMS_CUDA(cudaMemsetAsync(w.n_pairs, 0, sizeof(uint32_t) * 4, s));
    VMS_CUDA(cudaMemsetAsync(w.scan2, 0, scan_ws_bytes(2 * a.n_faces + 1), s));
    VMS_CUDA(cudaMemsetAsync(w.radix, 0, radix_clear_bytes(), s));
    VMS_CUDA(cudaMemsetAsync(w.ranges, 0, sizeof(uint2) * kVisMaxTiles, s));
    VMS_CUDA(cudaMemsetAsync(w.ictr, 0, sizeof(uint32_t) * 4, s));
    VMS_CUDA(cudaMemsetAsync(w.scan3, 0, scan_ws_bytes(kVisMaxTiles), s));
  }
  if (a.n_faces) {
    VMS_CUDA(launch(vis_count_k, ceil_div<uint32_t>(a.n_faces, T), T, 0, s,
                    (const VisFrameDev*)w.fd, a.verts, a.faces, a.n_faces, w.counts));
    mark("vis_count", s);
    int32_t st = scan_exclusive_u32(w.counts, w.offsets, nullptr, a.n_faces, a.n_faces, w.n_tris,
                                    w.scan, s, false);
    if (st) return st;
    VMS_CUDA(launch(vis_emit_k, ceil_div<uint32_t>(a.n_faces, T), T, 0, s,
                    (const VisFrameDev*)w.fd, a.verts, a.faces, a.face_page, a.n_faces,
                    (const uint32_t*)w.offsets, w.tris));
    mark("vis_emit", s);
  }
  dim3 grid(ceil_div(a.cam.width, kVisTile), ceil_div(a.cam.height, kVisTile));
  VisBins bins{nullptr, nullptr, nullptr, 0u};
  if (w.bcnt && a.n_faces) {
    // per-tile triangle lists: count tiles per triangle, scan, emit (tile,
    // triangle) pairs in triangle order, stable sort by tile, tile ranges
    const uint32_t tiles = grid.x * grid.y;
    if (tiles > kVisMaxTiles) {
      set_error("vis_frame: visibility raster larger than %u tiles", kVisMaxTiles);
      return VMS_ERR_INVALID;
    }
    const uint32_t nt_max = 2 * a.n_faces;
    const int g = 4 * kSMs;
    VMS_CUDA(launch(vis_bin_count_k, g, T, 0, s, (const VisTri*)w.tris,
                    (const uint32_t*)w.n_tris, w.bcnt));
    mark("vis_bin_count", s);
    int32_t st = scan_exclusive_u32(w.bcnt, w.boff, w.n_tris, 0, nt_max, w.n_pairs, w.scan2, s,
                                    false);
    if (st) return st;
    VMS_CUDA(launch(vis_bin_emit_k, g, T, 0, s, (const VisTri*)w.tris, (const uint32_t*)w.n_tris,
                    (const uint32_t*)w.boff, (const uint32_t*)w.n_pairs, w.pair_cap,
                    (int)grid.x, w.k0, w.v0));
    mark("vis_bin_emit", s);
    int bits = 1;
    while ((1u << bits) < tiles) ++bits;
    int alt = 0;
    // an overflowing frame sorts garbage it never reads (the emit and the
    // ranges skip it; the raster walks every triangle)
    st = radix_sort_u32(w.k0, w.v0, w.k1, w.v1, w.n_pairs, 0, w.pair_cap, 0, bits, &alt,
                        w.radix, s, false);
    if (st) return st;
    uint32_t* ks = alt ? w.k1 : w.k0;
    uint32_t* vs = alt ? w.v1 : w.v0;
    VMS_CUDA(launch(vis_bin_ranges_k, g, T, 0, s, (const uint32_t*)ks, (const uint32_t*)w.n_pairs,
                    w.pair_cap, w.ranges));
    mark("vis_bin_ranges", s);
    bins = VisBins{vs, w.ranges, w.n_pairs, w.pair_cap};
    // work items: (tile, chunk of <= kVisChunk list entries), then the
    // merge of the multi-chunk tiles
    VMS_CUDA(launch(vis_chunk_count_k, ceil_div<uint32_t>(tiles, T), T, 0, s,
                    (const uint2*)w.ranges, tiles, (const uint32_t*)w.n_pairs, w.pair_cap,
                    w.nchunk, w.slot, w.ictr + 1, w.slot_cap));
    mark("vis_chunk_count", s);
    st = scan_exclusive_u32(w.nchunk, w.chunk_off, nullptr, tiles, kVisMaxTiles, w.ictr, w.scan3,
                            s, false);
    if (st) return st;
    VMS_CUDA(launch(vis_raster_items_k, 8 * kSMs, kVisThreads, 0, s, (const VisTri*)w.tris,
                    (const uint32_t*)w.n_tris, a.cam.width, a.cam.height, (int)grid.x, tiles,
                    bins, (const uint32_t*)w.nchunk, (const uint32_t*)w.chunk_off,
                    (const uint32_t*)w.ictr, (const uint32_t*)w.slot, w.partial, a.id_image,
                    a.invz_image, a.page_count, w.base, w.direct, w.err));
    mark("vis_raster", s);
    VMS_CUDA(launch(vis_merge_k, 2 * kSMs, kVisThreads, 0, s, a.cam.width, a.cam.height,
                    (int)grid.x, tiles, (const uint32_t*)w.n_pairs, w.pair_cap,
                    (const uint32_t*)w.nchunk, (const uint32_t*)w.slot,
                    (const VisPartial*)w.partial, a.id_image, a.invz_image, a.page_count,
                    w.base, w.direct, w.err));
    mark("vis_merge", s);
  } else {
    VMS_CUDA(launch(vis_raster_k, grid, kVisThreads, 0, s, (const VisTri*)w.tris,
                    (const uint32_t*)w.n_tris, 0u, a.cam.width, a.cam.height, a.id_image,
                    a.invz_image, 0, a.page_count, w.base, w.direct, w.err));
    mark("vis_raster", s);
  }
  if (back) {
    VMS_CUDA(launch(vis_back_k, 1, kFrontThreads, sizeof(uint32_t) * (a.page_count + 1), s,
                    (const uint32_t*)w.base, (const uint8_t*)w.direct, a.link_off, a.link_tgt,
                    a.page_count, (const VisFrameDev*)w.fd, w.depth, w.n_tris, a.out));
    mark("vis_back", s);
  } else {
  VMS_CUDA(cudaMemcpyAsync(w.depth, w.base, sizeof(uint32_t) * (a.page_count + 1),
                           cudaMemcpyDeviceToDevice, s));
  if (a.page_count) {
    vis_links_k<<<ceil_div<uint32_t>(a.page_count * 32, T), T, 0, s>>>(
        w.base, w.depth, w.direct, a.link_off, a.link_tgt, a.page_count);
    mark("vis_links", s);
  }
  vis_flags_k<<<ceil_div<uint32_t>(a.page_count + 1, T), T, 0, s>>>(w.depth, a.page_count,
                                                                     w.pos);
  mark("vis_flags", s);
  int32_t st = scan_exclusive_u32(w.pos, w.pos, nullptr, a.page_count + 1, a.page_count + 1,
                                  w.n_req, w.scan, s);
  if (st) return st;
  vis_required_k<<<ceil_div<uint32_t>(a.page_count + 1, T), T, 0, s>>>(
      w.depth, w.direct, w.pos, a.page_count, w.fd, a.out);
  mark("vis_required", s);
  }
  if (a.out.meta && !back) {  // (vis_back_k stores them itself)
    VMS_CUDA(cudaMemcpyAsync(a.out.meta, w.n_tris, sizeof(uint32_t) * 4,
                             cudaMemcpyDeviceToHost, s));
  }
  if (a.depth_out) {
    VMS_CUDA(cudaMemcpyAsync(a.depth_out, w.depth, sizeof(uint32_t) * (a.page_count + 1),
                             cudaMemcpyDeviceToDevice, s));
  }
  if (a.direct_out) {
    VMS_CUDA(cudaMemcpyAsync(a.direct_out, w.direct, a.page_count + 1,
                             cudaMemcpyDeviceToDevice, s));
  }
  VMS_LAUNCH_CHECK("vis_frame");
  return VMS_OK;
}

int32_t reduce_images(const uint32_t* ids, const double* depth, uint64_t n_px,
                      uint32_t page_count, const uint32_t* link_off, const uint32_t* link_tgt,
                      uint32_t* depth_out, uint8_t* direct_out, uint32_t* err, void* ws,
                      cudaStream_t s) {
  uint32_t* base = static_cast<uint32_t*>(ws);
  const int T = 256;
  VMS_CUDA(cudaMemsetAsync(base, 0, sizeof(uint32_t) * (page_count + 1), s));
  VMS_CUDA(cudaMemsetAsync(direct_out, 0, page_count + 1, s));
  VMS_CUDA(cudaMemsetAsync(err, 0, sizeof(uint32_t), s));
  if (n_px)
    vis_reduce_images_k<<<4 * kSMs, T, 0, s>>>(ids, depth, n_px, page_count, base, direct_out,
                                               err);
  VMS_CUDA(cudaMemcpyAsync(depth_out, base, sizeof(uint32_t) * (page_count + 1),
                           cudaMemcpyDeviceToDevice, s));
  if (page_count)
    vis_links_k<<<ceil_div<uint32_t>(page_count * 32, T), T, 0, s>>>(base, depth_out, direct_out,
                                                                     link_off, link_tgt,
                                                                     page_count);
  VMS_LAUNCH_CHECK("reduce_images");
  return VMS_OK;
}

int32_t raster_triangles(const double* raw, const uint32_t* ids, uint32_t n, uint32_t* id_image,
                         double* invz_image, int w, int h, void* ws, cudaStream_t s) {
  VisTri* tris = static_cast<VisTri*>(ws);
  const int T = 256;
  if (n) vis_setup_raw_k<<<ceil_div<uint32_t>(n, T), T, 0, s>>>(raw, ids, n, w, h, tris);
  dim3 grid(ceil_div(w, kVisTile), ceil_div(h, kVisTile));
  vis_raster_k<<<grid, kVisThreads, 0, s>>>(tris, nullptr, n, w, h, id_image, invz_image, 1, 0,
                                            nullptr, nullptr, nullptr);
  VMS_LAUNCH_CHECK("raster_triangles");
  return VMS_OK;
}

}  // namespace vms
