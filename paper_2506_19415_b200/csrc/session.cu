// Per-frame orchestration in C++: VmSession.render_frame
// (pkg/src/vmsplat/runtime.py:436-489) as ONE host call per frame, pipelined
// with the previous frame's render:
//
//   vis stream  : [vis n+1 K1-K4] -> event -> host: page table n+1, copy plan,
//                 chunk table n+1                      (overlaps render n)
//   copy stream : [upload_k n+1: pinned host -> staging]  (overlaps render n)
//   main stream : [render n] ... | host waits render n, checks its counters |
//                 [scatter staging -> pool] [chunks H2D] [render n+1] ...
//
// Exactness: the visibility pass only reads the immutable mesh, the page table
// is updated strictly in frame order on the host, and pool slots are only
// rewritten (scatter) after the previous render has finished, so results are
// identical to the sequential reference order.  The host waits for render n
// before enqueueing render n+1: if render n overflowed its tile-instance
// buffer, the pool still holds frame n's pages and render n is redone with a
// larger buffer (rare slow path; the session owns and regrows its scratch).
#include <chrono>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "render.h"
#include "vis.h"

struct vms_session {
  vms_session_desc d;
  vms_pagetable* pt = nullptr;
  cudaStream_t vis_stream = nullptr, copy_stream = nullptr;
  cudaEvent_t ev_vis = nullptr, ev_copy = nullptr, ev_render = nullptr, ev_staging = nullptr;
  cudaEvent_t tev[10] = {};
  // pinned host memory
  uint32_t* req_pid = nullptr;
  uint32_t* req_enc = nullptr;
  uint8_t* req_direct = nullptr;
  uint8_t* req_level = nullptr;
  uint32_t* req_meta = nullptr;
  vms_copy* copies[2] = {nullptr, nullptr};    // host -> staging (per frame parity)
  vms_copy* scatter_h[2] = {nullptr, nullptr};  // staging -> pool offsets
  vms_chunk* chunks_h[2] = {nullptr, nullptr};
  uint32_t* counters = nullptr;  // n_kept, n_inst, overflow, n_need of the last render
  // device memory owned by the session
  vms_copy* scatter_d = nullptr;
  vms_chunk* chunks_d[2] = {nullptr, nullptr};
  void* ws = nullptr;  // render workspace
  size_t ws_bytes = 0;
  uint32_t m_cap = 0;
  int ws_w = 0, ws_h = 0;
  char* staging = nullptr;
  size_t staging_bytes = 0;
  int64_t max_chunks = 0;
  int parity = 0;
  std::vector<uint64_t> level_start;  // first row of each level block
  std::vector<uint32_t> plan_pid;
  std::vector<uint8_t> plan_level;
  std::vector<int32_t> plan_entry, plan_slot;
  // last render (for overflow recovery)
  bool have_last = false;
  vms_camera last_cam{};
  float* last_image = nullptr;
  float* last_host_image = nullptr;
  uint32_t last_chunks = 0, last_res = 0;
  int last_parity = 0;
  bool last_timing = false;
};

namespace vms {
namespace {

void free_session(vms_session* s) {
  if (!s) return;
  if (s->pt) vms_pt_destroy(s->pt);
  for (cudaStream_t x : {s->vis_stream, s->copy_stream})
    if (x) cudaStreamDestroy(x);
  for (cudaEvent_t e : {s->ev_vis, s->ev_copy, s->ev_render, s->ev_staging})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : s->tev)
    if (e) cudaEventDestroy(e);
  for (void* p : {(void*)s->req_pid, (void*)s->req_enc, (void*)s->req_direct,
                  (void*)s->req_level, (void*)s->req_meta, (void*)s->copies[0],
                  (void*)s->copies[1], (void*)s->scatter_h[0], (void*)s->scatter_h[1],
                  (void*)s->chunks_h[0], (void*)s->chunks_h[1],
                  (void*)s->counters})
    if (p) cudaFreeHost(p);
  for (void* p : {(void*)s->scatter_d, (void*)s->chunks_d[0], (void*)s->chunks_d[1], s->ws,
                  (void*)s->staging})
    if (p) cudaFree(p);
  delete s;
}

template <typename T>
cudaError_t host_alloc(T** p, size_t n) {
  return cudaHostAlloc(reinterpret_cast<void**>(p), sizeof(T) * (n ? n : 1),
                       cudaHostAllocMapped | cudaHostAllocPortable);
}

// (Re)allocate the render workspace for a resolution / instance capacity.
// Slow path only: first frame, resolution change, tile-instance overflow.
int32_t ensure_ws(vms_session* s, int w, int h, uint32_t m_cap) {
  if (s->ws && s->ws_w == w && s->ws_h == h && s->m_cap >= m_cap) return VMS_OK;
  const uint32_t n_cap = s->d.capacity * s->d.page_size;
  const size_t bytes = render_ws_bytes(n_cap, m_cap, tile_count(w, h));
  if (s->ws) {
    VMS_CUDA(cudaDeviceSynchronize());
    VMS_CUDA(cudaFree(s->ws));
    s->ws = nullptr;
  }
  VMS_CUDA(cudaMalloc(&s->ws, bytes));
  s->ws_bytes = bytes;
  s->m_cap = m_cap;
  s->ws_w = w;
  s->ws_h = h;
  return VMS_OK;
}

int32_t ensure_staging(vms_session* s, size_t bytes) {
  if (bytes <= s->staging_bytes) return VMS_OK;
  if (s->staging) {
    VMS_CUDA(cudaDeviceSynchronize());
    VMS_CUDA(cudaFree(s->staging));
    s->staging = nullptr;
  }
  const size_t want = bytes + bytes / 4;
  VMS_CUDA(cudaMalloc(&s->staging, want));
  s->staging_bytes = want;
  return VMS_OK;
}

__global__ void scatter_k(const vms_copy* __restrict__ list, int64_t n,
                          const char* __restrict__ src, char* __restrict__ dst) {
  for (int64_t c = blockIdx.y; c < n; c += gridDim.y) {
    const vms_copy cp = list[c];
    const uint4* s4 = reinterpret_cast<const uint4*>(src + cp.src_offset);
    uint4* d4 = reinterpret_cast<uint4*>(dst + cp.dst_offset);
    const uint64_t n16 = cp.nbytes / 16;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
         i += (uint64_t)gridDim.x * blockDim.x)
      d4[i] = s4[i];
    const uint32_t* s1 = reinterpret_cast<const uint32_t*>(src + cp.src_offset);
    uint32_t* d1 = reinterpret_cast<uint32_t*>(dst + cp.dst_offset);
    for (uint64_t i = n16 * 4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cp.nbytes / 4;
         i += (uint64_t)gridDim.x * blockDim.x)
      d1[i] = s1[i];
  }
}

int32_t launch_render(vms_session* s, const vms_camera& cam, float* image, int par,
                      uint32_t n_chunks, uint32_t n_res, bool timing, cudaStream_t st) {
  int32_t rc = ensure_ws(s, cam.width, cam.height, s->m_cap ? s->m_cap : s->d.m_cap);
  if (rc) return rc;
  RenderWs w = render_carve(s->ws, s->d.capacity * s->d.page_size, s->m_cap,
                            tile_count(cam.width, cam.height));
  void* ev[4] = {nullptr, nullptr, nullptr, nullptr};
  if (timing)
    for (int i = 0; i < 4; ++i) ev[i] = s->tev[4 + i];
  mark("begin", st);
  rc = render_preprocess(s->d.pool, s->chunks_d[par], n_chunks, cam, w, st);
  if (rc) return rc;
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[4], st));
  rc = render_finish(cam, n_res, w, image, 0, s->d.exact, ev, st);
  if (rc) return rc;
  VMS_CUDA(cudaMemcpyAsync(s->counters, w.ctr, sizeof(uint32_t) * 4, cudaMemcpyDeviceToHost, st));
  VMS_CUDA(cudaEventRecord(s->ev_render, st));
  s->have_last = true;
  s->last_cam = cam;
  s->last_image = image;
  s->last_chunks = n_chunks;
  s->last_res = n_res;
  s->last_parity = par;
  return VMS_OK;
}

// Wait for the last render; on tile-instance overflow grow and redo it (the
// pool still holds that frame's pages).  Returns with the render complete.
int32_t settle_last(vms_session* s, cudaStream_t st) {
  if (!s->have_last) return VMS_OK;
  VMS_CUDA(cudaEventSynchronize(s->ev_render));
  int guard = 0;
  while (s->counters[2]) {
    if (++guard > 8) {
      set_error("tile-instance buffer keeps overflowing (%u needed)", s->counters[3]);
      return VMS_ERR_NOMEM;
    }
    const uint32_t need = s->counters[3];
    int32_t rc = ensure_ws(s, s->last_cam.width, s->last_cam.height, need + need / 4 + (1u << 16));
    if (rc) return rc;
    rc = launch_render(s, s->last_cam, s->last_image, s->last_parity, s->last_chunks, s->last_res,
                       false, st);
    if (rc) return rc;
    if (s->last_host_image)
      VMS_CUDA(cudaMemcpyAsync(s->last_host_image, s->last_image,
                               sizeof(float) * 3 * (size_t)s->last_cam.width * s->last_cam.height,
                               cudaMemcpyDeviceToHost, st));
    VMS_CUDA(cudaEventSynchronize(s->ev_render));
    VMS_CUDA(cudaStreamSynchronize(st));
  }
  return VMS_OK;
}

float ms_between(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) return 0.f;
  return ms;
}

}  // namespace
}  // namespace vms

using namespace vms;

extern "C" {

size_t vms_session_render_ws_bytes(uint32_t capacity, uint32_t page_size, uint32_t m_cap,
                                   int32_t width, int32_t height) {
  return vms_render_workspace_bytes(capacity * page_size, m_cap, width, height);
}

vms_session* vms_session_create(const vms_session_desc* desc) {
  if (!desc || desc->capacity < 1 || desc->page_size < 1 || desc->lod_levels < 1 ||
      desc->lod_levels > 16 || desc->page_count < 1 || !desc->pool || !desc->vis_ws ||
      !desc->host_records) {
    set_error("session_create: invalid descriptor");
    return nullptr;
  }
  if ((uint64_t)desc->capacity * desc->page_size > 0xFFFFFFFFull) {
    set_error("session_create: pool larger than 2^32 records");
    return nullptr;
  }
  vms_session* s = new vms_session();
  s->d = *desc;
  s->pt = vms_pt_create(desc->capacity);
  const uint32_t P = desc->page_count;
  s->max_chunks = (int64_t)desc->capacity *
                  (ceil_div<uint32_t>(desc->page_size, kChunkRecords) + (1u << (desc->lod_levels - 1)));
  s->m_cap = desc->m_cap ? desc->m_cap : 16u * desc->capacity * desc->page_size;
  bool ok = s->pt != nullptr;
  ok = ok && cudaStreamCreateWithFlags(&s->vis_stream, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking) == cudaSuccess;
  for (cudaEvent_t* e : {&s->ev_vis, &s->ev_copy, &s->ev_render, &s->ev_staging})
    ok = ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
  for (cudaEvent_t& e : s->tev) ok = ok && cudaEventCreate(&e) == cudaSuccess;
  ok = ok && host_alloc(&s->req_pid, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_enc, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_direct, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_level, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_meta, 4) == cudaSuccess;
  for (int k = 0; k < 2; ++k) {
    ok = ok && host_alloc(&s->copies[k], P + 1) == cudaSuccess;
    ok = ok && host_alloc(&s->scatter_h[k], P + 1) == cudaSuccess;
  }
  ok = ok && host_alloc(&s->chunks_h[0], (size_t)s->max_chunks) == cudaSuccess;
  ok = ok && host_alloc(&s->chunks_h[1], (size_t)s->max_chunks) == cudaSuccess;
  ok = ok && host_alloc(&s->counters, 4) == cudaSuccess;
  ok = ok && cudaMalloc(&s->scatter_d, sizeof(vms_copy) * (P + 1)) == cudaSuccess;
  ok = ok && cudaMalloc(&s->chunks_d[0], sizeof(vms_chunk) * s->max_chunks) == cudaSuccess;
  ok = ok && cudaMalloc(&s->chunks_d[1], sizeof(vms_chunk) * s->max_chunks) == cudaSuccess;
  if (!ok) {
    set_error("session_create: %s", cudaGetErrorString(cudaGetLastError()));
    free_session(s);
    return nullptr;
  }
  std::memset(s->counters, 0, sizeof(uint32_t) * 4);
  s->level_start.assign(desc->lod_levels + 1, 0);
  for (uint32_t k = 0; k < desc->lod_levels; ++k)
    s->level_start[k + 1] =
        s->level_start[k] + (uint64_t)desc->page_counts[k] * (desc->page_size >> k);
  if (s->level_start[desc->lod_levels] > desc->host_rows) {
    set_error("session_create: host record section shorter than the level blocks");
    free_session(s);
    return nullptr;
  }
  s->plan_pid.resize(P + 1);
  s->plan_level.resize(P + 1);
  s->plan_entry.resize(P + 1);
  s->plan_slot.resize(P + 1);
  return s;
}

void vms_session_destroy(vms_session* s) {
  if (s) cudaDeviceSynchronize();
  free_session(s);
}

vms_pagetable* vms_session_table(vms_session* s) { return s ? s->pt : nullptr; }

int32_t vms_session_set_render_ws(vms_session* s, void* ws, uint64_t bytes, uint32_t m_cap,
                                  int32_t width, int32_t height) {
  // the session owns its scratch; this only raises the instance capacity
  (void)ws;
  (void)bytes;
  if (!s) return VMS_ERR_INVALID;
  return ensure_ws(s, width, height, m_cap);
}

int32_t vms_session_frame(vms_session* s, const vms_frame_args* a, vms_frame_stats* out,
                          void* stream) {
  if (!s || !a || !out || !a->image) {
    set_error("session_frame: invalid arguments");
    return VMS_ERR_INVALID;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::memset(out, 0, sizeof(*out));
  const bool timing = a->timing != 0;
  const uint32_t P = s->d.page_count;
  const int par = s->parity;
  s->parity ^= 1;
  // [1]+[2] visibility on its own stream (overlaps the previous render)
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[0], s->vis_stream));
  vms_vis_args v{};
  v.cam = a->vis_cam;
  v.verts = s->d.verts;
  v.faces = s->d.faces;
  v.face_page = s->d.face_page;
  v.n_faces = s->d.n_faces;
  v.page_count = P;
  v.link_off = s->d.link_off;
  v.link_tgt = s->d.link_tgt;
  v.lod = a->lod;
  v.out.pid = s->req_pid;
  v.out.enc = s->req_enc;
  v.out.direct = s->req_direct;
  v.out.level = s->req_level;
  v.out.meta = s->req_meta;
  v.workspace = s->d.vis_ws;
  int32_t rc = vis_frame(v, s->vis_stream);
  if (rc) return rc;
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[1], s->vis_stream));
  VMS_CUDA(cudaEventRecord(s->ev_vis, s->vis_stream));
  VMS_CUDA(cudaEventSynchronize(s->ev_vis));
  const uint32_t n_req = s->req_meta[1];
  out->n_tris = s->req_meta[0];
  if (s->req_meta[2]) {
    set_error("visibility page id %u out of range (page count %u)", s->req_meta[2], P);
    return VMS_ERR_INVARIANT;
  }
  const auto h0 = std::chrono::steady_clock::now();
  // [3] page table (exact update_page_table)
  int64_t n_plan = 0, missing = 0;
  rc = vms_pt_update(s->pt, s->req_pid, s->req_enc, s->req_direct, s->req_level, n_req, a->frame,
                     a->budget, s->plan_pid.data(), s->plan_level.data(), s->plan_entry.data(),
                     s->plan_slot.data(), (int64_t)s->plan_pid.size(), &n_plan, &missing);
  if (rc) return rc;
  // copy plan: scene rows -> packed staging, staging -> pool slot rows
  uint64_t bytes = 0;
  const uint64_t rb = (uint64_t)kRecordFloats * sizeof(float);
  for (int64_t i = 0; i < n_plan; ++i) {
    const uint32_t lv = s->plan_level[i];
    const uint64_t per = (uint64_t)s->d.page_size >> lv;
    const uint64_t src = s->level_start[lv] + (uint64_t)(s->plan_pid[i] - 1) * per;
    const uint64_t dst = (uint64_t)s->plan_entry[i] * s->d.page_size + (uint64_t)s->plan_slot[i] * per;
    s->copies[par][i] = vms_copy{src * rb, bytes, per * rb};
    s->scatter_h[par][i] = vms_copy{bytes, dst * rb, per * rb};
    bytes += per * rb;
  }
  // chunk table of every resident page, ascending page id (gather order)
  int64_t n_res = 0;
  const int64_t n_chunks =
      vms_pt_chunks(s->pt, s->d.page_size, s->chunks_h[par], s->max_chunks, &n_res);
  if (n_chunks < 0 || n_chunks > s->max_chunks) {
    set_error("session_frame: chunk table overflow");
    return VMS_ERR_INVARIANT;
  }
  out->host_update_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
  // uploads into staging on the copy stream (overlap the previous render)
  if (n_plan) {
    rc = ensure_staging(s, bytes);
    if (rc) return rc;
    VMS_CUDA(cudaStreamWaitEvent(s->copy_stream, s->ev_staging, 0));  // staging reuse
    if (timing) VMS_CUDA(cudaEventRecord(s->tev[2], s->copy_stream));
    rc = vms_upload_pages(s->copies[par], n_plan, s->d.host_records, s->staging, s->d.upload_mode,
                          s->copy_stream);
    if (rc) return rc;
    if (timing) VMS_CUDA(cudaEventRecord(s->tev[3], s->copy_stream));
    VMS_CUDA(cudaEventRecord(s->ev_copy, s->copy_stream));
    VMS_CUDA(cudaMemcpyAsync(s->scatter_d, s->scatter_h[par], sizeof(vms_copy) * n_plan,
                             cudaMemcpyHostToDevice, s->copy_stream));
    VMS_CUDA(cudaEventRecord(s->ev_copy, s->copy_stream));
  }
  // the previous render must be final before pool slots are rewritten
  rc = settle_last(s, st);
  if (rc) return rc;
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[8], st));
  if (n_plan) {
    VMS_CUDA(cudaStreamWaitEvent(st, s->ev_copy, 0));
    dim3 grid(64, (unsigned)(n_plan < 65535 ? n_plan : 65535));
    scatter_k<<<grid, 256, 0, st>>>(s->scatter_d, n_plan, s->staging,
                                    reinterpret_cast<char*>(s->d.pool));
    mark("scatter", st);
    VMS_CUDA(cudaEventRecord(s->ev_staging, st));
  }
  if (n_chunks)
    VMS_CUDA(cudaMemcpyAsync(s->chunks_d[par], s->chunks_h[par], sizeof(vms_chunk) * n_chunks,
                             cudaMemcpyHostToDevice, st));
  // [4]-[6] render every resident record
  rc = launch_render(s, a->cam, a->image, par, (uint32_t)n_chunks, (uint32_t)n_res, timing, st);
  if (rc) return rc;
  s->last_host_image = a->host_image;
  s->last_timing = timing;
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[9], st));
  if (a->host_image)
    VMS_CUDA(cudaMemcpyAsync(a->host_image, a->image,
                             sizeof(float) * 3 * (size_t)a->cam.width * a->cam.height,
                             cudaMemcpyDeviceToHost, st));
  // stats (runtime.py:471-481)
  out->required = n_req;
  out->resident = (uint32_t)vms_pt_resident_count(s->pt);
  out->planned = (uint32_t)n_plan;
  out->missing = (uint32_t)missing;
  out->bytes_copied = bytes;
  out->occupied_entries = (uint32_t)vms_pt_occupied(s->pt);
  out->capacity = s->d.capacity;
  out->n_chunks = (uint32_t)n_chunks;
  out->n_res = (uint32_t)n_res;
  rc = vms_pt_resident_counts(s->pt, out->resident_per_level, (int32_t)s->d.lod_levels);
  if (rc) return rc;
  if (timing || a->host_image) {
    rc = settle_last(s, st);
    if (rc) return rc;
    VMS_CUDA(cudaStreamSynchronize(st));
    out->n_kept = s->counters[0];
    out->n_inst = s->counters[1];
    out->n_need = s->counters[3];
    if (timing) {
      out->ms_vis = ms_between(s->tev[0], s->tev[1]);
      out->ms_copy = n_plan ? ms_between(s->tev[2], s->tev[3]) : 0.f;
      out->ms_preprocess = ms_between(s->tev[8], s->tev[4]);
      out->ms_sort = ms_between(s->tev[4], s->tev[5]);
      out->ms_tiles = ms_between(s->tev[5], s->tev[6]);
      out->ms_blend = ms_between(s->tev[6], s->tev[7]);
      out->ms_frame = ms_between(s->tev[8], s->tev[9]) + out->ms_vis;
    }
  }
  return VMS_OK;
}

int32_t vms_session_rerender(vms_session* s, float* host_image, void* stream) {
  if (!s || !s->have_last) {
    set_error("session_rerender: nothing to re-render");
    return VMS_ERR_INVALID;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t rc = settle_last(s, st);
  if (rc) return rc;
  rc = launch_render(s, s->last_cam, s->last_image, s->last_parity, s->last_chunks, s->last_res,
                     false, st);
  if (rc) return rc;
  if (host_image)
    VMS_CUDA(cudaMemcpyAsync(host_image, s->last_image,
                             sizeof(float) * 3 * (size_t)s->last_cam.width * s->last_cam.height,
                             cudaMemcpyDeviceToHost, st));
  s->last_host_image = host_image;
  rc = settle_last(s, st);
  if (rc) return rc;
  VMS_CUDA(cudaStreamSynchronize(st));
  return VMS_OK;
}

int32_t vms_session_counters(vms_session* s, uint32_t* out4, void* stream) {
  if (!s || !out4) return VMS_ERR_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t rc = settle_last(s, st);
  if (rc) return rc;
  VMS_CUDA(cudaStreamSynchronize(st));
  std::memcpy(out4, s->counters, sizeof(uint32_t) * 4);
  return VMS_OK;
}

}  // extern "C"
