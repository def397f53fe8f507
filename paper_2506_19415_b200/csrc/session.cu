// Per-frame orchestration in C++: VmSession.render_frame
// (pkg/src/vmsplat/runtime.py:436-489) as ONE host call per frame, so the only
// host work between the visibility readback and the render launch is the
// page-table update itself (no interpreter on the critical path).
//
//   main stream : [vis K1-K4] -event-> | host: page table, copy plan, chunk
//                 table | [chunk H2D] -wait copy- [preprocess .. blend]
//                 [counters D2H] ([image D2H])
//   copy stream : [upload_k over mapped pinned host memory]
//
// The previous frame's render is complete whenever the visibility event of
// the next frame has fired (same stream), so its counters (tile-instance
// overflow) are checked there without an extra synchronisation.
#include <chrono>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "render.h"
#include "vis.h"

struct vms_session {
  vms_session_desc d;
  vms_pagetable* pt = nullptr;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_vis = nullptr, ev_main = nullptr, ev_copy = nullptr;
  cudaEvent_t tev[10] = {};
  // pinned host memory
  uint32_t* req_pid = nullptr;
  uint32_t* req_enc = nullptr;
  uint8_t* req_direct = nullptr;
  uint8_t* req_level = nullptr;
  uint32_t* req_meta = nullptr;
  vms_copy* copies = nullptr;
  vms_chunk* chunks_h = nullptr;
  uint32_t* counters = nullptr;  // n_kept, n_inst, overflow, n_need of the last render
  // device
  vms_chunk* chunks_d = nullptr;
  int64_t max_chunks = 0;
  std::vector<uint64_t> level_start;  // first row of each level block
  // plan scratch
  std::vector<uint32_t> plan_pid;
  std::vector<uint8_t> plan_level;
  std::vector<int32_t> plan_entry, plan_slot;
  // last render (for overflow recovery)
  bool have_last = false;
  bool last_checked = true;
  vms_camera last_cam{};
  float* last_image = nullptr;
  uint32_t last_chunks = 0, last_res = 0;
};

namespace vms {
namespace {

void free_session(vms_session* s) {
  if (!s) return;
  if (s->pt) vms_pt_destroy(s->pt);
  if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
  for (cudaEvent_t e : {s->ev_vis, s->ev_main, s->ev_copy})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : s->tev)
    if (e) cudaEventDestroy(e);
  for (void* p : {(void*)s->req_pid, (void*)s->req_enc, (void*)s->req_direct,
                  (void*)s->req_level, (void*)s->req_meta, (void*)s->copies,
                  (void*)s->chunks_h, (void*)s->counters})
    if (p) cudaFreeHost(p);
  if (s->chunks_d) cudaFree(s->chunks_d);
  delete s;
}

template <typename T>
cudaError_t host_alloc(T** p, size_t n) {
  return cudaHostAlloc(reinterpret_cast<void**>(p), sizeof(T) * (n ? n : 1),
                       cudaHostAllocMapped | cudaHostAllocPortable);
}

int32_t launch_render(vms_session* s, const vms_camera& cam, float* image, uint32_t n_chunks,
                      uint32_t n_res, bool timing, cudaStream_t st) {
  const uint32_t tiles = tile_count(cam.width, cam.height);
  if (cam.width != s->d.width || cam.height != s->d.height) {
    set_error("session: render resolution %dx%d differs from the workspace's %dx%d", cam.width,
              cam.height, s->d.width, s->d.height);
    return VMS_ERR_INVALID;
  }
  RenderWs w = render_carve(s->d.render_ws, s->d.capacity * s->d.page_size, s->d.m_cap, tiles);
  void* ev[4] = {nullptr, nullptr, nullptr, nullptr};
  if (timing)
    for (int i = 0; i < 4; ++i) ev[i] = s->tev[4 + i];
  mark("begin", st);
  int32_t rc = render_preprocess(s->d.pool, s->chunks_d, n_chunks, cam, w, st);
  if (rc) return rc;
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[4], st));
  rc = render_finish(cam, n_res, w, image, 0, s->d.exact, ev, st);
  if (rc) return rc;
  VMS_CUDA(cudaMemcpyAsync(s->counters, w.ctr, sizeof(uint32_t) * 4, cudaMemcpyDeviceToHost, st));
  s->have_last = true;
  s->last_checked = false;
  s->last_cam = cam;
  s->last_image = image;
  s->last_chunks = n_chunks;
  s->last_res = n_res;
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
      !desc->render_ws || !desc->host_records) {
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
  bool ok = s->pt != nullptr;
  ok = ok && cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaEventCreateWithFlags(&s->ev_vis, cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaEventCreateWithFlags(&s->ev_main, cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaEventCreateWithFlags(&s->ev_copy, cudaEventDisableTiming) == cudaSuccess;
  for (cudaEvent_t& e : s->tev) ok = ok && cudaEventCreate(&e) == cudaSuccess;
  ok = ok && host_alloc(&s->req_pid, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_enc, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_direct, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_level, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_meta, 4) == cudaSuccess;
  ok = ok && host_alloc(&s->copies, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->chunks_h, (size_t)s->max_chunks) == cudaSuccess;
  ok = ok && host_alloc(&s->counters, 4) == cudaSuccess;
  ok = ok && cudaMalloc(&s->chunks_d, sizeof(vms_chunk) * s->max_chunks) == cudaSuccess;
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

void vms_session_destroy(vms_session* s) { free_session(s); }

vms_pagetable* vms_session_table(vms_session* s) { return s ? s->pt : nullptr; }

int32_t vms_session_set_render_ws(vms_session* s, void* ws, uint64_t bytes, uint32_t m_cap,
                                  int32_t width, int32_t height) {
  if (!s || !ws ||
      bytes < vms_session_render_ws_bytes(s->d.capacity, s->d.page_size, m_cap, width, height)) {
    set_error("session_set_render_ws: workspace too small");
    return VMS_ERR_INVALID;
  }
  s->d.render_ws = ws;
  s->d.render_ws_bytes = bytes;
  s->d.m_cap = m_cap;
  s->d.width = width;
  s->d.height = height;
  return VMS_OK;
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
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[0], st));
  // [1]+[2] visibility, required list straight into mapped pinned memory
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
  int32_t rc = vis_frame(v, st);
  if (rc) return rc;
  VMS_CUDA(cudaEventRecord(s->ev_vis, st));
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[1], st));
  VMS_CUDA(cudaEventSynchronize(s->ev_vis));
  // the previous render has completed: check its tile-instance counters
  if (s->have_last && !s->last_checked) {
    s->last_checked = true;
    if (s->counters[2]) {
      out->overflow = 2;  // 2 = the previous frame
      out->n_need = s->counters[3];
      set_error("tile-instance buffer overflow in the previous frame (%u needed, %u)",
                s->counters[3], s->d.m_cap);
      return VMS_ERR_NOMEM;
    }
  }
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
  // copy plan in bytes: source rows from the level blocks, destination slot rows
  uint64_t bytes = 0;
  const uint64_t rb = (uint64_t)kRecordFloats * sizeof(float);
  for (int64_t i = 0; i < n_plan; ++i) {
    const uint32_t lv = s->plan_level[i];
    const uint64_t per = (uint64_t)s->d.page_size >> lv;
    const uint64_t src = s->level_start[lv] + (uint64_t)(s->plan_pid[i] - 1) * per;
    const uint64_t dst = (uint64_t)s->plan_entry[i] * s->d.page_size + (uint64_t)s->plan_slot[i] * per;
    s->copies[i] = vms_copy{src * rb, dst * rb, per * rb};
    bytes += per * rb;
  }
  // chunk table of every resident page, ascending page id (gather order)
  int64_t n_res = 0;
  const int64_t n_chunks = vms_pt_chunks(s->pt, s->d.page_size, s->chunks_h, s->max_chunks, &n_res);
  if (n_chunks < 0 || n_chunks > s->max_chunks) {
    set_error("session_frame: chunk table overflow");
    return VMS_ERR_INVARIANT;
  }
  out->host_update_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
  if (n_plan) {
    VMS_CUDA(cudaEventRecord(s->ev_main, st));
    VMS_CUDA(cudaStreamWaitEvent(s->copy_stream, s->ev_main, 0));
    if (timing) VMS_CUDA(cudaEventRecord(s->tev[2], s->copy_stream));
    rc = vms_upload_pages(s->copies, n_plan, s->d.host_records, s->d.pool, s->d.upload_mode,
                          s->copy_stream);
    if (rc) return rc;
    if (timing) VMS_CUDA(cudaEventRecord(s->tev[3], s->copy_stream));
    VMS_CUDA(cudaEventRecord(s->ev_copy, s->copy_stream));
  }
  if (n_chunks)
    VMS_CUDA(cudaMemcpyAsync(s->chunks_d, s->chunks_h, sizeof(vms_chunk) * n_chunks,
                             cudaMemcpyHostToDevice, st));
  if (n_plan) VMS_CUDA(cudaStreamWaitEvent(st, s->ev_copy, 0));
  // [4]-[6] render every resident record
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[8], st));
  rc = launch_render(s, a->cam, a->image, (uint32_t)n_chunks, (uint32_t)n_res, timing, st);
  if (rc) return rc;
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[9], st));
  const bool sync_end = timing || a->host_image;
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
  if (sync_end) {
    VMS_CUDA(cudaStreamSynchronize(st));
    s->last_checked = true;
    out->n_kept = s->counters[0];
    out->n_inst = s->counters[1];
    out->overflow = s->counters[2];
    out->n_need = s->counters[3];
    if (timing) {
      out->ms_vis = ms_between(s->tev[0], s->tev[1]);
      out->ms_copy = n_plan ? ms_between(s->tev[2], s->tev[3]) : 0.f;
      out->ms_preprocess = ms_between(s->tev[8], s->tev[4]);
      out->ms_sort = ms_between(s->tev[4], s->tev[5]);
      out->ms_tiles = ms_between(s->tev[5], s->tev[6]);
      out->ms_blend = ms_between(s->tev[6], s->tev[7]);
      out->ms_frame = ms_between(s->tev[0], s->tev[9]);
    }
    if (out->overflow) {
      set_error("tile-instance buffer overflow (%u needed, %u)", out->n_need, s->d.m_cap);
      return VMS_ERR_NOMEM;
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
  int32_t rc = launch_render(s, s->last_cam, s->last_image, s->last_chunks, s->last_res, false, st);
  if (rc) return rc;
  if (host_image)
    VMS_CUDA(cudaMemcpyAsync(host_image, s->last_image,
                             sizeof(float) * 3 * (size_t)s->last_cam.width * s->last_cam.height,
                             cudaMemcpyDeviceToHost, st));
  VMS_CUDA(cudaStreamSynchronize(st));
  s->last_checked = true;
  if (s->counters[2]) {
    set_error("tile-instance buffer overflow (%u needed, %u)", s->counters[3], s->d.m_cap);
    return VMS_ERR_NOMEM;
  }
  return VMS_OK;
}

int32_t vms_session_counters(vms_session* s, uint32_t* out4, void* stream) {
  if (!s || !out4) return VMS_ERR_INVALID;
  VMS_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  std::memcpy(out4, s->counters, sizeof(uint32_t) * 4);
  if (s->have_last && !s->last_checked) {
    s->last_checked = true;
    if (s->counters[2]) {
      set_error("tile-instance buffer overflow (%u needed, %u)", s->counters[3], s->d.m_cap);
      return VMS_ERR_NOMEM;
    }
  }
  return VMS_OK;
}

}  // extern "C"
