// Per-frame orchestration in C++: VmSession.render_frame
// (pkg/src/vmsplat/runtime.py:436-489) as ONE host call per frame, pipelined
// two frames deep with the renders already in flight:
//
//   vis stream  (high priority) : [vis graph n+1] -> event -> host: page table
//                  n+1, copy plan, chunk table n+1       (overlaps render n)
//   copy stream : [upload_k n+1: pinned host -> staging] (overlaps render n)
//   main stream : [render n] [scatter staging -> pool] [frame block + chunk
//                  table H2D] [render graph n+1] [counters D2H] ...
//
// Every render kernel reads the per-frame values (camera, image pointer,
// chunk and splat counts) from a device block (FrameDev), so the whole
// render - preprocess, compaction, depth sort, tile duplication, tile sort,
// ranges, blend, ~30 launches - is captured ONCE into a CUDA graph per
// (resolution, instance capacity, timing) and replayed with one launch per
// frame; the visibility pass likewise.  The host never waits for a render
// except to recycle the pinned buffers of the frame two back.
//
// Exactness: the visibility pass only reads the immutable mesh, the page table
// is updated strictly in frame order on the host, and pool slots are only
// rewritten (scatter, main stream) after the previous render in stream order,
// so results are identical to the sequential reference order.  A frame whose
// tile instances overflow the buffer is still blended exactly (blend_k falls
// back to the depth-sorted splat list); the host sees the overflow counter
// when it recycles that frame's buffers and grows the buffer (re-capturing
// the graph) for the frames after it.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <unistd.h>

#include "common.cuh"
#include "render.h"
#include "vis.h"

namespace {
constexpr int kBands = 4;  // blend launches / image copy pieces for host output

// Streaming source (upload_mode 2): planned page rows are gathered from
// ordinary host memory (e.g. the memory-mapped .vms file, which need not fit
// in page-locked memory) into a page-locked bounce buffer by a few host
// threads, then cross PCIe as one copy.
class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { run(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // fd >= 0: the pieces' sources are byte offsets into this file, read
  // with pread (no page faults on a mapping the process has not touched)
  void set_source_fd(int fd) { fd_ = fd; }
  // Copy every piece (dst, src, bytes) and return when all are done; false
  // if a read failed.
  bool copy(const std::vector<std::tuple<char*, const char*, size_t>>& pieces) {
    if (pieces.empty()) return true;
    failed_ = false;
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &pieces;
      next_ = 0;
      pending_ = (int)workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
    return !failed_;
  }

 private:
  void run(int) {
    uint64_t seen = 0;
    for (;;) {
      const std::vector<std::tuple<char*, const char*, size_t>>* job;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        job = job_;
      }
      for (;;) {
        const size_t i = next_.fetch_add(1);
        if (i >= job->size()) break;
        const auto& pc = (*job)[i];
        if (fd_ >= 0) {
          char* dst = std::get<0>(pc);
          size_t left = std::get<2>(pc);
          off_t off = (off_t)reinterpret_cast<uintptr_t>(std::get<1>(pc));
          while (left) {
            const ssize_t got = pread(fd_, dst, left, off);
            if (got <= 0) {
              failed_ = true;
              break;
            }
            dst += got;
            off += got;
            left -= (size_t)got;
          }
        } else {
          std::memcpy(std::get<0>(pc), std::get<1>(pc), std::get<2>(pc));
        }
      }
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::vector<std::tuple<char*, const char*, size_t>>* job_ = nullptr;
  std::atomic<size_t> next_{0};
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
  int fd_ = -1;
  std::atomic<bool> failed_{false};
};
}

namespace {
struct Graph {
  cudaGraphExec_t exec = nullptr;
  int w = 0, h = 0;
  uint32_t m_cap = 0;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
  }
};
}  // namespace

// Frames in flight: frame i uses slot i % slots (its pinned host buffers,
// render workspace, graphs, events); render_frame(i) recycles frame
// i - slots.  Four slots let the host enqueue a frame while the three before
// it still render / copy to the host (VMSPLAT_SLOTS=2..8; C2 same box: 3
// slots 2112-2117 frames/s, e2e 1749-1763; 4 slots 2124-2138, e2e 1802-1804).
constexpr int kMaxSlots = 8;

struct vms_session {
  vms_session_desc d;
  int slots = 4;
  vms_pagetable* pt = nullptr;
  cudaStream_t vis_stream = nullptr, copy_stream = nullptr, cap_stream = nullptr;
  cudaStream_t d2h_stream = nullptr;  // banded image copies to the host
  cudaEvent_t ev_band[kBands] = {};
  cudaEvent_t ev_d2h = nullptr;
  cudaEvent_t ev_out[kMaxSlots] = {};  // asynchronous host copy of a frame done
  bool pending_out[kMaxSlots] = {};
  cudaEvent_t ev_vis = nullptr, ev_copy = nullptr, ev_staging = nullptr;
  cudaEvent_t ev_done[kMaxSlots] = {};
  // cross-frame overlap: frame i's front (scatter, preprocess, sorts, tile
  // lists) runs on front_stream[i & 1] while frame i - 1 blends on the
  // caller's stream; ev_pre = that parity's preprocess has read the pool,
  // ev_front = its tile lists are ready for the blend
  bool overlap = true;
  cudaStream_t front_stream[kMaxSlots] = {};
  cudaEvent_t ev_pre[kMaxSlots] = {}, ev_front[kMaxSlots] = {};
  cudaEvent_t tev[10] = {};
  // pinned host memory
  uint32_t* req_pid = nullptr;
  uint32_t* req_enc = nullptr;
  uint8_t* req_direct = nullptr;
  uint8_t* req_level = nullptr;
  uint32_t* req_meta = nullptr;
  vms::VisFrameDev* vis_fd_h = nullptr;
  vms_copy* copies[kMaxSlots] = {};    // host -> staging (per frame parity)
  vms_copy* scatter_h[kMaxSlots] = {};  // staging -> pool offsets
  vms_chunk* chunks_h[kMaxSlots] = {};
  vms::FrameDev* fd_h[kMaxSlots] = {};
  uint32_t* counters_h[kMaxSlots] = {};  // n_kept, n_inst, overflow, n_need
  bool pending[kMaxSlots] = {};
  int last_par = -1;
  // device memory owned by the session
  vms_copy* scatter_d = nullptr;
  vms_chunk* chunks_d = nullptr;
  void* ws = nullptr;  // render workspaces, one per frame parity
  size_t ws_bytes = 0, ws_stride = 0;
  uint32_t m_cap = 0, m_want = 0;
  uint32_t m_limit = 1u << 26;  // largest tile-instance buffer the session grows to
  bool trace = false;
  // VMSPLAT_TRACE=2: per-frame timeline (host clock + device events, no
  // syncs), printed every kTl frames
  static constexpr int kTl = 32;
  bool timeline = false;
  int tl_n = 0;
  // vis start, vis end, render (front) start, render end, d2h end, front end, blend start
  cudaEvent_t tl_ev[kTl][7] = {};
  double tl_host[kTl][4] = {};     // enter, vis waited, host work done, exit
  int ws_w = 0, ws_h = 0;
  char* staging = nullptr;
  size_t staging_bytes = 0;
  // upload_mode 2 (streaming source): page-locked bounce buffers per parity
  char* bounce[kMaxSlots] = {};
  size_t bounce_bytes[kMaxSlots] = {};
  CopyPool* pool = nullptr;
  std::vector<std::tuple<char*, const char*, size_t>> pieces;
  int64_t max_chunks = 0;
  int parity = 0;
  bool use_graphs = true;
  // vis: [slot] (device table); front: [slot][timing][banded]; blend: [slot][timing]
  Graph vis_graph[kMaxSlots], front_graph[kMaxSlots][2][2], blend_graph[kMaxSlots][2];
  // device page table (desc.device_table): its outputs land in mapped memory
  // (plan, stats) and per-slot device chunk tables, read in place by the
  // slot's preprocess; the next frame of the same slot waits for that
  // preprocess (ev_pre) before its update overwrites them
  vms_dpt* dpt = nullptr;
  uint32_t* dplan_pid = nullptr;
  uint8_t* dplan_level = nullptr;
  int32_t* dplan_entry = nullptr;
  int32_t* dplan_slot = nullptr;
  vms_dpt_stats* dstats = nullptr;
  vms_chunk* chunks_dev[kMaxSlots] = {};
  // the required list in device memory (the update reads it there: reads of
  // mapped host memory stall behind a concurrent image copy on the bus)
  uint32_t* dreq_pid = nullptr;
  uint32_t* dreq_enc = nullptr;
  uint8_t* dreq_direct = nullptr;
  uint8_t* dreq_level = nullptr;
  bool chunks_pending[kMaxSlots] = {};
  std::vector<uint64_t> level_start;  // first row of each level block
  std::vector<uint32_t> plan_pid;
  std::vector<int32_t> plan_order;
  std::vector<uint8_t> plan_level;
  std::vector<int32_t> plan_entry, plan_slot;
};

namespace vms {
namespace {

void reset_render_graphs(vms_session* s) {
  for (auto& gp : s->front_graph)
    for (auto& gt : gp)
      for (auto& g : gt) g.reset();
  for (auto& gp : s->blend_graph)
    for (auto& g : gp) g.reset();
}

void free_session(vms_session* s) {
  if (!s) return;
  for (auto& g : s->vis_graph) g.reset();
  if (s->dpt) vms_dpt_destroy(s->dpt);
  for (void* p : {(void*)s->dplan_pid, (void*)s->dplan_level, (void*)s->dplan_entry,
                  (void*)s->dplan_slot, (void*)s->dstats})
    if (p) cudaFreeHost(p);
  for (vms_chunk* p : s->chunks_dev)
    if (p) cudaFree(p);
  for (void* p : {(void*)s->dreq_pid, (void*)s->dreq_enc, (void*)s->dreq_direct,
                  (void*)s->dreq_level})
    if (p) cudaFree(p);
  reset_render_graphs(s);
  if (s->pt) vms_pt_destroy(s->pt);
  for (cudaStream_t x : {s->vis_stream, s->copy_stream, s->cap_stream, s->d2h_stream})
    if (x) cudaStreamDestroy(x);
  for (cudaEvent_t e : s->ev_band)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : s->ev_out)
    if (e) cudaEventDestroy(e);
  if (s->ev_d2h) cudaEventDestroy(s->ev_d2h);
  for (cudaEvent_t e : {s->ev_vis, s->ev_copy, s->ev_staging})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : s->tev)
    if (e) cudaEventDestroy(e);
  for (void* p : {(void*)s->req_pid, (void*)s->req_enc, (void*)s->req_direct,
                  (void*)s->req_level, (void*)s->req_meta, (void*)s->vis_fd_h})
    if (p) cudaFreeHost(p);
  for (int k = 0; k < kMaxSlots; ++k) {
    for (void* p : {(void*)s->copies[k], (void*)s->scatter_h[k], (void*)s->chunks_h[k],
                    (void*)s->fd_h[k], (void*)s->counters_h[k]})
      if (p) cudaFreeHost(p);
    if (s->front_stream[k]) cudaStreamDestroy(s->front_stream[k]);
    for (cudaEvent_t e : {s->ev_done[k], s->ev_pre[k], s->ev_front[k]})
      if (e) cudaEventDestroy(e);
  }
  for (void* p : {(void*)s->scatter_d, (void*)s->chunks_d, s->ws, (void*)s->staging})
    if (p) cudaFree(p);
  for (char* p : s->bounce)
    if (p) cudaFreeHost(p);
  delete s->pool;
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
  const auto t0 = std::chrono::steady_clock::now();
  const uint32_t n_cap = s->d.capacity * s->d.page_size;
  const size_t one = (render_ws_bytes(n_cap, m_cap, tile_count(w, h)) + 4095) & ~(size_t)4095;
  const size_t bytes = (size_t)s->slots * one;  // one workspace per frame in flight
  if (s->ws) {
    VMS_CUDA(cudaDeviceSynchronize());
    VMS_CUDA(cudaFree(s->ws));
    s->ws = nullptr;
  }
  reset_render_graphs(s);
  VMS_CUDA(cudaMalloc(&s->ws, bytes));
  s->ws_bytes = bytes;
  s->ws_stride = one;
  s->m_cap = m_cap;
  s->ws_w = w;
  s->ws_h = h;
  if (s->trace)
    fprintf(stderr, "[vmsplat] render workspace %dx%d, %u instances, %.1f MB: %.3f ms\n", w, h,
            m_cap, bytes / 1e6,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  return VMS_OK;
}

RenderWs ws_of(const vms_session* s, int par) {
  return render_carve(static_cast<char*>(s->ws) + (size_t)par * s->ws_stride,
                      s->d.capacity * s->d.page_size, s->m_cap, tile_count(s->ws_w, s->ws_h));
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

// A stream-ordered launch sequence, either replayed from a graph captured
// once (key: resolution + instance capacity) or enqueued directly (profiling
// mode: per-launch event marks are not capturable).
template <typename F>
int32_t run_captured(vms_session* s, Graph& g, int w, int h, uint32_t m_cap, F&& enqueue,
                     cudaStream_t st) {
  if (!s->use_graphs || g_profile) return enqueue(st, false);
  if (g.exec && (g.w != w || g.h != h || g.m_cap != m_cap)) g.reset();
  if (!g.exec) {
    const auto t0 = std::chrono::steady_clock::now();
    VMS_CUDA(cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal));
    int32_t rc = enqueue(s->cap_stream, true);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(s->cap_stream, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return cuda_status(e, "graph capture");
    e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      g.exec = nullptr;
      return cuda_status(e, "graph instantiate");
    }
    g.w = w;
    g.h = h;
    g.m_cap = m_cap;
    if (s->trace)
      fprintf(stderr, "[vmsplat] graph capture %dx%d m_cap %u: %.3f ms\n", w, h, m_cap,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count());
  }
  VMS_CUDA(cudaGraphLaunch(g.exec, st));
  return VMS_OK;
}

// The frame's front - memsets, preprocess, depth sort, tile lists - on
// stream fs (one graph per parity/timing/banded), recording ev_pre[par] once
// the preprocess has read the pool and ev_front[par] at its end.
int32_t launch_front(vms_session* s, int par, int w, int h, bool timing, bool banded,
                     cudaStream_t fs) {
  const RenderWs ws = ws_of(s, par);
  const uint32_t max_chunks = (uint32_t)s->max_chunks;
  auto enqueue = [&](cudaStream_t q, bool captured) -> int32_t {
    void* ev[4] = {nullptr, nullptr, nullptr, nullptr};
    if (timing)
      for (int i = 0; i < 4; ++i) ev[i] = s->tev[4 + i];
    const unsigned rf = captured ? cudaEventRecordExternal : cudaEventRecordDefault;
    mark("begin", q);
    int32_t rc = render_clear(w, h, ws, q);
    if (rc) return rc;
    rc = render_preprocess(s->d.pool, s->dpt ? s->chunks_dev[par] : s->chunks_d, max_chunks,
                           ws, q);
    if (rc) return rc;
    VMS_CUDA(cudaEventRecordWithFlags(s->ev_pre[par], q, rf));
    if (timing) VMS_CUDA(cudaEventRecordWithFlags(s->tev[4], q, rf));
    return render_finish(w, h, ws, 0, s->d.exact, ev, captured, banded ? -kBands : -1, q);
  };
  int32_t rc = run_captured(s, s->front_graph[par][timing ? 1 : 0][banded ? 1 : 0], w, h,
                            s->m_cap, enqueue, fs);
  if (rc) return rc;
  VMS_CUDA(cudaEventRecord(s->ev_front[par], fs));
  return VMS_OK;
}

// The frame's blend on the caller's stream st, after its front: one graph
// per parity, or (host output, banded) one launch per band, each followed
// by the event the band's image copy waits for.
int32_t launch_blend(vms_session* s, int par, int w, int h, bool timing, bool banded,
                     cudaStream_t st) {
  const RenderWs ws = ws_of(s, par);
  VMS_CUDA(cudaStreamWaitEvent(st, s->ev_front[par], 0));
  int32_t rc = VMS_OK;
  if (!banded) {
    rc = run_captured(s, s->blend_graph[par][timing ? 1 : 0], w, h, s->m_cap,
                      [&](cudaStream_t q, bool) { return render_band(w, h, ws, s->d.exact, 0, 1, q); },
                      st);
  } else {
    for (int b = 0; b < kBands && !rc; ++b) {
      rc = render_band(w, h, ws, s->d.exact, b, kBands, st);
      if (!rc) VMS_CUDA(cudaEventRecord(s->ev_band[b], st));
    }
  }
  if (rc) return rc;
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[7], st));
  return VMS_OK;
}

// The frame two back used this parity's pinned buffers: wait for its render,
// and grow the tile-instance buffer if it overflowed (it was still blended
// exactly, through the depth-sorted list).
int32_t recycle(vms_session* s, int par) {
  if (s->pending_out[par]) {
    VMS_CUDA(cudaEventSynchronize(s->ev_out[par]));
    s->pending_out[par] = false;
  }
  if (!s->pending[par]) return VMS_OK;
  VMS_CUDA(cudaEventSynchronize(s->ev_done[par]));
  s->pending[par] = false;
  const uint32_t* c = s->counters_h[par];
  if (c[2]) {
    // frames past the limit (camera inside dense geometry: tens of millions
    // of instances, blends that saturate in a few splats) keep the spill path
    const uint32_t need = c[3];
    uint64_t want = (uint64_t)need + need / 4 + (1u << 16);
    if (want > s->m_limit) want = s->m_limit;
    if (want > s->m_want) s->m_want = (uint32_t)want;
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
  if (blend_init() != VMS_OK || vis_init() != VMS_OK) return nullptr;
  vms_session* s = new vms_session();
  s->d = *desc;
  s->pt = vms_pt_create(desc->capacity);
  const uint32_t P = desc->page_count;
  s->max_chunks = (int64_t)desc->capacity *
                  (ceil_div<uint32_t>(desc->page_size, kChunkRecords) + (1u << (desc->lod_levels - 1)));
  s->m_cap = 0;
  s->m_want = desc->m_cap ? desc->m_cap : 16u * desc->capacity * desc->page_size;
  const char* g = std::getenv("VMSPLAT_GRAPHS");
  s->use_graphs = !(g && g[0] == '0');
  const char* tr = std::getenv("VMSPLAT_TRACE");
  s->trace = tr && tr[0] == '1';
  s->timeline = tr && tr[0] == '2';
  if (s->timeline)
    for (auto& r : s->tl_ev)
      for (auto& e : r) cudaEventCreate(&e);
  if (const char* ml = std::getenv("VMSPLAT_MAX_INSTANCES")) {
    const long long v = std::atoll(ml);
    if (v > 0) s->m_limit = (uint32_t)(v < 0xFFFFFFF0ll ? v : 0xFFFFFFF0ll);
  }
  if (s->m_want > s->m_limit) s->m_limit = s->m_want;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  bool ok = s->pt != nullptr;
  // visibility gates the host's page-table work: let it overtake render kernels
  ok = ok && cudaStreamCreateWithPriority(&s->vis_stream, cudaStreamNonBlocking, hi) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&s->d2h_stream, cudaStreamNonBlocking) == cudaSuccess;
  {
    // VMSPLAT_OVERLAP=0: fronts on the caller's stream (no cross-frame
    // overlap); VMSPLAT_FRONT_PRIO=0: front streams at default priority
    const char* ov = std::getenv("VMSPLAT_OVERLAP");
    s->overlap = !(ov && ov[0] == '0');
    const char* fp = std::getenv("VMSPLAT_FRONT_PRIO");
    const int prio = (fp && fp[0] == '0') ? lo : hi;
    if (const char* sl = std::getenv("VMSPLAT_SLOTS")) {
      const int v = std::atoi(sl);
      if (v >= 2 && v <= kMaxSlots) s->slots = v;
    }
    for (int k = 0; k < s->slots; ++k) {
      ok = ok && cudaStreamCreateWithPriority(&s->front_stream[k], cudaStreamNonBlocking, prio) ==
                     cudaSuccess;
      for (cudaEvent_t* e : {&s->ev_pre[k], &s->ev_front[k], &s->ev_done[k], &s->ev_out[k]})
        ok = ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
    }
  }
  for (cudaEvent_t& e : s->ev_band)
    ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaEventCreateWithFlags(&s->ev_d2h, cudaEventDisableTiming) == cudaSuccess;
  for (cudaEvent_t* e : {&s->ev_vis, &s->ev_copy, &s->ev_staging})
    ok = ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
  for (cudaEvent_t& e : s->tev) ok = ok && cudaEventCreate(&e) == cudaSuccess;
  ok = ok && host_alloc(&s->req_pid, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_enc, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_direct, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_level, P + 1) == cudaSuccess;
  ok = ok && host_alloc(&s->req_meta, 4) == cudaSuccess;
  ok = ok && host_alloc(&s->vis_fd_h, 1) == cudaSuccess;
  for (int k = 0; k < s->slots; ++k) {
    ok = ok && host_alloc(&s->copies[k], P + 1) == cudaSuccess;
    ok = ok && host_alloc(&s->scatter_h[k], P + 1) == cudaSuccess;
    ok = ok && host_alloc(&s->chunks_h[k], (size_t)s->max_chunks) == cudaSuccess;
    ok = ok && host_alloc(&s->fd_h[k], 1) == cudaSuccess;
    ok = ok && host_alloc(&s->counters_h[k], 4) == cudaSuccess;
  }
  ok = ok && cudaMalloc(&s->scatter_d, sizeof(vms_copy) * (P + 1)) == cudaSuccess;
  ok = ok && cudaMalloc(&s->chunks_d, sizeof(vms_chunk) * s->max_chunks) == cudaSuccess;
  if (ok && desc->device_table) {
    s->dpt = vms_dpt_create((int32_t)desc->capacity, (int32_t)P, (int32_t)desc->lod_levels);
    if (!s->dpt) {
      free_session(s);
      return nullptr;  // vms_dpt_create set the error
    }
    ok = ok && host_alloc(&s->dplan_pid, P + 1) == cudaSuccess;
    ok = ok && host_alloc(&s->dplan_level, P + 1) == cudaSuccess;
    ok = ok && host_alloc(&s->dplan_entry, P + 1) == cudaSuccess;
    ok = ok && host_alloc(&s->dplan_slot, P + 1) == cudaSuccess;
    ok = ok && host_alloc(&s->dstats, 1) == cudaSuccess;
    ok = ok && cudaMalloc(&s->dreq_pid, sizeof(uint32_t) * (P + 1)) == cudaSuccess;
    ok = ok && cudaMalloc(&s->dreq_enc, sizeof(uint32_t) * (P + 1)) == cudaSuccess;
    ok = ok && cudaMalloc(&s->dreq_direct, P + 1) == cudaSuccess;
    ok = ok && cudaMalloc(&s->dreq_level, P + 1) == cudaSuccess;
    for (int k = 0; k < s->slots; ++k) {
      ok = ok && cudaMalloc(&s->chunks_dev[k], sizeof(vms_chunk) * s->max_chunks) == cudaSuccess;
    }
  }
  if (!ok) {
    set_error("session_create: %s", cudaGetErrorString(cudaGetLastError()));
    free_session(s);
    return nullptr;
  }
  for (int k = 0; k < s->slots; ++k) std::memset(s->counters_h[k], 0, sizeof(uint32_t) * 4);
  s->level_start.assign(desc->lod_levels + 1, 0);
  for (uint32_t k = 0; k < desc->lod_levels; ++k)
    s->level_start[k + 1] =
        s->level_start[k] + (uint64_t)desc->page_counts[k] * (desc->page_size >> k);
  if (s->level_start[desc->lod_levels] > desc->host_rows) {
    set_error("session_create: host record section shorter than the level blocks");
    free_session(s);
    return nullptr;
  }
  if (desc->upload_mode == 2) {
    const unsigned hw = std::thread::hardware_concurrency();
    unsigned nt = std::max(1u, std::min(8u, hw ? hw / 2 : 4u));
    if (const char* e = std::getenv("VMSPLAT_COPY_THREADS")) {  // mode-2 gather threads
      const int v = std::atoi(e);
      if (v > 0 && v <= 64) nt = (unsigned)v;
    }
    s->pool = new CopyPool((int)nt);
    s->pool->set_source_fd(desc->host_fd);
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

vms_dpt* vms_session_dpt(vms_session* s) { return s ? s->dpt : nullptr; }

int32_t vms_session_cert_count(vms_session* s, uint32_t* out) {
  if (!s || !out || !s->ws) {
    set_error("session_cert_count: invalid arguments");
    return VMS_ERR_INVALID;
  }
  return debug_cert_count(ws_of(s, s->last_par < 0 ? 0 : s->last_par), out);
}

int32_t vms_session_prepare(vms_session* s, int32_t width, int32_t height) {
  if (!s || width < 1 || height < 1) {
    set_error("session_prepare: invalid arguments");
    return VMS_ERR_INVALID;
  }
  return ensure_ws(s, width, height, s->m_cap > s->m_want ? s->m_cap : s->m_want);
}

int32_t vms_session_set_render_ws(vms_session* s, void* ws, uint64_t bytes, uint32_t m_cap,
                                  int32_t width, int32_t height) {
  // the session owns its scratch; this only raises the instance capacity
  (void)ws;
  (void)bytes;
  (void)width;
  (void)height;
  if (!s) return VMS_ERR_INVALID;
  if (m_cap > s->m_want) s->m_want = m_cap;
  return VMS_OK;
}

int32_t vms_session_frame(vms_session* s, const vms_frame_args* a, vms_frame_stats* out,
                          void* stream) {
  if (!s || !a || !out || !a->image || a->cam.width < 1 || a->cam.height < 1 ||
      a->vis_cam.width < 1 || a->vis_cam.height < 1 || a->lod.count < 0 || a->lod.count > 8) {
    set_error("session_frame: invalid arguments");
    return VMS_ERR_INVALID;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::memset(out, 0, sizeof(*out));
  const bool timing = a->timing != 0;
  const int tl = s->timeline ? s->tl_n % vms_session::kTl : -1;
  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  if (tl >= 0) s->tl_host[tl][0] = now_us();
  const uint32_t P = s->d.page_count;
  const int par = s->parity;
  int32_t rc = VMS_OK;
  s->parity = (par + 1) % s->slots;
  // [1]+[2] visibility on its own high-priority stream (overlaps the renders
  // in flight); the compacted required list lands in mapped pinned memory.
  // It touches no per-parity buffer, so it starts before the frame two back
  // (same parity) is recycled: that frame's image copy to the host and the
  // visibility pass, which queues behind the render in flight for SM slots,
  // then overlap instead of adding up.
  if (s->dpt) {
    // this parity's device chunk table is free once the frame two back copied it
    if (s->chunks_pending[par]) VMS_CUDA(cudaStreamWaitEvent(s->vis_stream, s->ev_pre[par], 0));
  }
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[0], s->vis_stream));
  if (tl >= 0) VMS_CUDA(cudaEventRecord(s->tl_ev[tl][0], s->vis_stream));
  s->vis_fd_h->cam = a->vis_cam;
  s->vis_fd_h->lod = a->lod;
  s->vis_fd_h->dpt.frame = a->frame;
  s->vis_fd_h->dpt.budget = a->budget;
  VMS_CUDA(cudaMemcpyAsync(vis_frame_dev(s->d.vis_ws, s->d.n_faces, P), s->vis_fd_h,
                           sizeof(VisFrameDev), cudaMemcpyHostToDevice, s->vis_stream));
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
  // the host table reads the required list from mapped memory; the device
  // table from device memory (its counts and frame inputs too)
  v.out.pid = s->dpt ? s->dreq_pid : s->req_pid;
  v.out.enc = s->dpt ? s->dreq_enc : s->req_enc;
  v.out.direct = s->dpt ? s->dreq_direct : s->req_direct;
  v.out.level = s->dpt ? s->dreq_level : s->req_level;
  v.out.meta = s->req_meta;
  v.workspace = s->d.vis_ws;
  rc = run_captured(s, s->vis_graph[s->dpt ? par : 0], v.cam.width, v.cam.height, 0,
                    [&](cudaStream_t q, bool) {
                      int32_t r = vis_launch(v, q);
                      if (r || !s->dpt) return r;
                      // [3] on the device: update_page_table, then the chunk table
                      r = vms_dpt_update(s->dpt, s->dreq_pid, s->dreq_enc, s->dreq_direct,
                                         s->dreq_level, vis_meta_dev(s->d.vis_ws, s->d.n_faces, P) + 1,
                                         &vis_frame_dev(s->d.vis_ws, s->d.n_faces, P)->dpt,
                                         s->dplan_pid,
                                         s->dplan_level, s->dplan_entry, s->dplan_slot,
                                         (int64_t)P + 1, s->dstats, q);
                      if (r) return r;
                      return vms_dpt_chunks(s->dpt, s->d.page_size, s->chunks_dev[par],
                                            s->max_chunks, s->dstats, q);
                    },
                    s->vis_stream);
  if (rc) return rc;
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[1], s->vis_stream));
  if (tl >= 0) VMS_CUDA(cudaEventRecord(s->tl_ev[tl][1], s->vis_stream));
  VMS_CUDA(cudaEventRecord(s->ev_vis, s->vis_stream));
  VMS_CUDA(cudaEventSynchronize(s->ev_vis));
  if (tl >= 0) s->tl_host[tl][1] = now_us();
  const uint32_t n_req = s->req_meta[1];
  out->n_tris = s->req_meta[0];
  if (s->req_meta[2]) {
    set_error("visibility page id %u out of range (page count %u)", s->req_meta[2], P);
    return VMS_ERR_INVARIANT;
  }
  const auto h0 = std::chrono::steady_clock::now();
  // [3] page table (exact update_page_table): on the host, or already done
  // on the device (read its plan and stats)
  int64_t n_plan = 0, missing = 0;
  const uint32_t* plan_pid = s->plan_pid.data();
  const uint8_t* plan_level = s->plan_level.data();
  const int32_t* plan_entry = s->plan_entry.data();
  const int32_t* plan_slot = s->plan_slot.data();
  if (s->dpt) {
    if (s->dstats->bad || s->dstats->plan_overflow) {
      set_error("device page table: required page id / level out of range or plan overflow");
      return VMS_ERR_INVARIANT;
    }
    n_plan = s->dstats->n_plan;
    missing = s->dstats->missing;
    plan_pid = s->dplan_pid;
    plan_level = s->dplan_level;
    plan_entry = s->dplan_entry;
    plan_slot = s->dplan_slot;
  } else {
    rc = vms_pt_update(s->pt, s->req_pid, s->req_enc, s->req_direct, s->req_level, n_req,
                       a->frame, a->budget, s->plan_pid.data(), s->plan_level.data(),
                       s->plan_entry.data(), s->plan_slot.data(), (int64_t)s->plan_pid.size(),
                       &n_plan, &missing);
    if (rc) return rc;
  }
  // the frame two back (this parity): its host copies, counters, image
  rc = recycle(s, par);
  if (rc) return rc;
  // copy plan: scene rows -> packed staging, staging -> pool slot rows
  // (packed into staging in scene order, so pages adjacent in the scene
  // file become one copy)
  uint64_t bytes = 0;
  const uint64_t rb = (uint64_t)kRecordFloats * sizeof(float);
  auto src_row = [&](int64_t i) {
    const uint32_t lv = plan_level[i];
    return s->level_start[lv] + (uint64_t)(plan_pid[i] - 1) * ((uint64_t)s->d.page_size >> lv);
  };
  s->plan_order.resize(n_plan);
  for (int64_t i = 0; i < n_plan; ++i) s->plan_order[i] = (int32_t)i;
  std::sort(s->plan_order.begin(), s->plan_order.end(),
            [&](int32_t x, int32_t y) { return src_row(x) < src_row(y); });
  for (int64_t k = 0; k < n_plan; ++k) {
    const int64_t i = s->plan_order[k];
    const uint32_t lv = plan_level[i];
    const uint64_t per = (uint64_t)s->d.page_size >> lv;
    const uint64_t src = src_row(i);
    const uint64_t dst = (uint64_t)plan_entry[i] * s->d.page_size + (uint64_t)plan_slot[i] * per;
    s->copies[par][k] = vms_copy{src * rb, bytes, per * rb};
    s->scatter_h[par][k] = vms_copy{bytes, dst * rb, per * rb};
    bytes += per * rb;
  }
  // chunk table of every resident page, ascending page id (gather order)
  int64_t n_res = 0;
  const int64_t n_chunks =
      s->dpt ? (n_res = s->dstats->n_records, (int64_t)s->dstats->n_chunks)
             : vms_pt_chunks(s->pt, s->d.page_size, s->chunks_h[par], s->max_chunks, &n_res);
  if (n_chunks < 0 || n_chunks > s->max_chunks) {
    set_error("session_frame: chunk table overflow");
    return VMS_ERR_INVARIANT;
  }
  out->host_update_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
  // uploads into staging on the copy stream (overlap the renders in flight)
  // the most a plan can move: the budget in level-0 pages, plus the page that
  // crosses it (update_page_table's break-on-budget)
  const size_t budget_bytes =
      (size_t)(std::ceil(std::max(0.0, (double)a->budget)) + 1.0) * s->d.page_size * rb;
  if (n_plan) {
    rc = ensure_staging(s, std::max<size_t>(bytes, budget_bytes));
    if (rc) return rc;
    VMS_CUDA(cudaStreamWaitEvent(s->copy_stream, s->ev_staging, 0));  // staging reuse
    if (timing) VMS_CUDA(cudaEventRecord(s->tev[2], s->copy_stream));
    if (s->d.upload_mode == 2) {
      // gather the planned rows into page-locked memory on host threads, then
      // one PCIe copy (the bounce buffer of this parity was released when the
      // frame two back was recycled)
      if (s->bounce_bytes[par] < bytes) {
        if (s->bounce[par]) VMS_CUDA(cudaFreeHost(s->bounce[par]));
        s->bounce[par] = nullptr;
        // page-locking is slow and synchronising: size each slot's buffer
        // once for the largest plan the staging budget allows
        const size_t want = std::max<size_t>(bytes + bytes / 4, budget_bytes);
        VMS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->bounce[par]), want,
                               cudaHostAllocPortable));
        s->bounce_bytes[par] = want;
      }
      s->pieces.clear();
      // from the file (pread at the record section's offset) or the mapping
      const char* src = s->d.host_fd >= 0
                            ? reinterpret_cast<const char*>((uintptr_t)s->d.host_fd_offset)
                            : reinterpret_cast<const char*>(s->d.host_records);
      constexpr size_t kPiece = 1u << 20;
      for (int64_t i = 0; i < n_plan; ++i) {
        const vms_copy& c = s->copies[par][i];
        for (size_t o = 0; o < c.nbytes; o += kPiece)
          s->pieces.emplace_back(s->bounce[par] + c.dst_offset + o, src + c.src_offset + o,
                                 std::min<size_t>(kPiece, c.nbytes - o));
      }
      const auto g0 = std::chrono::steady_clock::now();
      const bool read_ok = s->pool->copy(s->pieces);
      out->ms_host_gather = (float)(std::chrono::duration<double, std::milli>(
                                std::chrono::steady_clock::now() - g0).count());
      if (!read_ok) {
        set_error("session_frame: reading page rows from the scene file failed");
        return VMS_ERR_CUDA;
      }
      VMS_CUDA(cudaMemcpyAsync(s->staging, s->bounce[par], bytes, cudaMemcpyHostToDevice,
                               s->copy_stream));
    } else {
      rc = vms_upload_pages(s->copies[par], n_plan, s->d.host_records, s->staging,
                            s->d.upload_mode, s->copy_stream);
      if (rc) return rc;
    }
    if (timing) VMS_CUDA(cudaEventRecord(s->tev[3], s->copy_stream));
    VMS_CUDA(cudaMemcpyAsync(s->scatter_d, s->scatter_h[par], sizeof(vms_copy) * n_plan,
                             cudaMemcpyHostToDevice, s->copy_stream));
    VMS_CUDA(cudaEventRecord(s->ev_copy, s->copy_stream));
  }
  // [4]-[6] the frame's front on this parity's front stream (the caller's
  // stream in timing mode): pool slots are rewritten only after the previous
  // frame's preprocess has read them (ev_pre), then the frame block, chunk
  // table and the front graph.  Its workspace was last used by the frame two
  // back, whose blend recycle() has waited for.
  const int W = a->cam.width, H = a->cam.height;
  rc = ensure_ws(s, W, H, s->m_cap > s->m_want ? s->m_cap : s->m_want);
  if (rc) return rc;
  cudaStream_t fs = (timing || !s->overlap) ? st : s->front_stream[par];
  if (fs != st)
    VMS_CUDA(cudaStreamWaitEvent(fs, s->ev_pre[(par + s->slots - 1) % s->slots], 0));
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[8], fs));
  if (tl >= 0) {
    s->tl_host[tl][2] = now_us();
    VMS_CUDA(cudaEventRecord(s->tl_ev[tl][2], fs));
  }
  if (n_plan) {
    VMS_CUDA(cudaStreamWaitEvent(fs, s->ev_copy, 0));
    dim3 grid(64, (unsigned)(n_plan < 65535 ? n_plan : 65535));
    scatter_k<<<grid, 256, 0, fs>>>(s->scatter_d, n_plan, s->staging,
                                    reinterpret_cast<char*>(s->d.pool));
    mark("scatter", fs);
    VMS_CUDA(cudaEventRecord(s->ev_staging, fs));
  }
  RenderWs ws = ws_of(s, par);
  FrameDev* f = s->fd_h[par];
  f->cam = a->cam;
  f->image = a->image;
  f->n_chunks = (uint32_t)n_chunks;
  f->n_splats = (uint32_t)n_res;
  f->counters_host = s->counters_h[par];  // mapped: written by tile_prep_k
  VMS_CUDA(cudaMemcpyAsync(ws.fd, f, sizeof(FrameDev), cudaMemcpyHostToDevice, fs));
  // the device table's chunk table is read in place (this slot's buffer);
  // the host table's goes up with the frame block
  if (n_chunks && !s->dpt)
    VMS_CUDA(cudaMemcpyAsync(s->chunks_d, s->chunks_h[par], sizeof(vms_chunk) * n_chunks,
                             cudaMemcpyHostToDevice, fs));
  // host output: the blend runs as kBands launches over bands of tile rows
  // and each band's rows go to the host as soon as that band is blended
  // host output, synchronous call: the blend runs as kBands launches and each
  // band's rows are copied while the next band blends.  Asynchronous call
  // (sync = 0): one blend, then one copy on the d2h stream that overlaps the
  // NEXT frame's render (the image buffer is recycled only after the copy).
  const bool async_out = a->host_image != nullptr && !a->sync && !timing;
  const bool banded = a->host_image != nullptr && !async_out;
  rc = launch_front(s, par, W, H, timing, banded, fs);
  if (rc) return rc;
  s->chunks_pending[par] = s->dpt != nullptr;  // ev_pre[par]: its preprocess read them
  if (tl >= 0) {
    VMS_CUDA(cudaEventRecord(s->tl_ev[tl][5], fs));
    VMS_CUDA(cudaStreamWaitEvent(st, s->ev_front[par], 0));
    VMS_CUDA(cudaEventRecord(s->tl_ev[tl][6], st));
  }
  rc = launch_blend(s, par, W, H, timing, banded, st);
  if (rc) return rc;
  if (async_out) {
    VMS_CUDA(cudaEventRecord(s->ev_band[0], st));
    VMS_CUDA(cudaStreamWaitEvent(s->d2h_stream, s->ev_band[0], 0));
    // in row bands: page uploads (host -> device) queued on the copy engines
    // meanwhile go between two bands instead of after the whole 25 MB frame
    // (C2 frames 5-64 under a per-frame image copy: 1609 frames/s as one
    // copy, 1717 as 8 bands)
    static const int bands = [] {
      const char* e = std::getenv("VMSPLAT_D2H_BANDS");
      const int v = e && *e ? std::atoi(e) : 8;
      return v < 1 ? 1 : (v > 64 ? 64 : v);
    }();
    const size_t row_bytes = sizeof(float) * 3 * (size_t)W;
    for (int b = 0; b < bands; ++b) {
      const int y0 = (int)((int64_t)H * b / bands), y1 = (int)((int64_t)H * (b + 1) / bands);
      if (y1 > y0)
        VMS_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(a->host_image) + row_bytes * y0,
                                 reinterpret_cast<const char*>(a->image) + row_bytes * y0,
                                 row_bytes * (y1 - y0), cudaMemcpyDeviceToHost, s->d2h_stream));
    }
    VMS_CUDA(cudaEventRecord(s->ev_out[par], s->d2h_stream));
    if (tl >= 0) VMS_CUDA(cudaEventRecord(s->tl_ev[tl][4], s->d2h_stream));
    s->pending_out[par] = true;
  }
  if (banded) {
    const int ts = tile_size(), tiles_y = ceil_div(H, ts);
    const size_t row_bytes = sizeof(float) * 3 * (size_t)W;
    for (int b = 0; b < kBands; ++b) {
      const int y0 = blend_band_row(b, kBands, tiles_y) * ts;
      const int y1 = std::min(blend_band_row(b + 1, kBands, tiles_y) * ts, H);
      VMS_CUDA(cudaStreamWaitEvent(s->d2h_stream, s->ev_band[b], 0));
      if (y1 > y0)
        VMS_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(a->host_image) + row_bytes * y0,
                                 reinterpret_cast<const char*>(a->image) + row_bytes * y0,
                                 row_bytes * (y1 - y0), cudaMemcpyDeviceToHost, s->d2h_stream));
    }
    VMS_CUDA(cudaEventRecord(s->ev_d2h, s->d2h_stream));
    VMS_CUDA(cudaStreamWaitEvent(st, s->ev_d2h, 0));
  }
  VMS_CUDA(cudaEventRecord(s->ev_done[par], st));
  if (tl >= 0) {
    VMS_CUDA(cudaEventRecord(s->tl_ev[tl][3], st));
    s->tl_host[tl][3] = now_us();
    if (++s->tl_n % vms_session::kTl == 0) {
      // frame k: host enter / vis waited / enqueue start / exit (us, relative to
      // frame 0 enter) and device vis start-end, render start-end (us, relative
      // to frame 0 vis start)
      VMS_CUDA(cudaEventSynchronize(s->tl_ev[tl][3]));
      const double h0 = 0.0;
      for (int k = 0; k < vms_session::kTl; ++k) {
        float d[7] = {0, 0, 0, 0, 0, 0, 0};
        for (int j = 0; j < 7; ++j) cudaEventElapsedTime(&d[j], s->tl_ev[0][0], s->tl_ev[k][j]);
        fprintf(stderr,
                "[tl] %2d host %12.1f %12.1f %12.1f %12.1f  dev vis %8.1f %8.1f render %8.1f %8.1f"
                " d2h end %8.1f front end %8.1f blend start %8.1f\n",
                k, s->tl_host[k][0] - h0, s->tl_host[k][1] - h0, s->tl_host[k][2] - h0,
                s->tl_host[k][3] - h0, 1e3 * d[0], 1e3 * d[1], 1e3 * d[2], 1e3 * d[3], 1e3 * d[4],
                1e3 * d[5], 1e3 * d[6]);
      }
      (void)cudaGetLastError();  // frames without a host copy never recorded their d2h event
    }
  }
  s->pending[par] = true;
  s->last_par = par;
  if (timing) VMS_CUDA(cudaEventRecord(s->tev[9], st));
  // stats (runtime.py:471-481)
  out->required = n_req;
  out->resident = s->dpt ? s->dstats->resident : (uint32_t)vms_pt_resident_count(s->pt);
  out->planned = (uint32_t)n_plan;
  out->missing = (uint32_t)missing;
  out->bytes_copied = bytes;
  out->occupied_entries = s->dpt ? s->dstats->occupied : (uint32_t)vms_pt_occupied(s->pt);
  out->capacity = s->d.capacity;
  out->n_chunks = (uint32_t)n_chunks;
  out->n_res = (uint32_t)n_res;
  if (s->dpt) {
    for (uint32_t k = 0; k < s->d.lod_levels && k < 16; ++k)
      out->resident_per_level[k] = s->dstats->resident_per_level[k];
  } else {
    rc = vms_pt_resident_counts(s->pt, out->resident_per_level, (int32_t)s->d.lod_levels);
    if (rc) return rc;
  }
  if (timing || a->sync || (a->host_image && !async_out)) {
    VMS_CUDA(cudaStreamSynchronize(st));
    const uint32_t* c = s->counters_h[par];
    out->n_kept = c[0];
    out->n_inst = c[1];
    out->overflow = c[2];
    out->n_need = c[3];
    rc = recycle(s, par);
    if (rc) return rc;
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

int32_t vms_session_wait(vms_session* s, int32_t back) {
  if (!s || back < 0 || back >= s->slots) {
    set_error("session_wait: invalid arguments");
    return VMS_ERR_INVALID;
  }
  if (s->last_par < 0) return VMS_OK;
  return recycle(s, (s->last_par + s->slots - back) % s->slots);
}

int32_t vms_session_slots(const vms_session* s) { return s ? s->slots : 0; }

int32_t vms_session_counters(vms_session* s, uint32_t* out4, void* stream) {
  if (!s || !out4) return VMS_ERR_INVALID;
  (void)stream;
  std::memset(out4, 0, sizeof(uint32_t) * 4);
  if (s->last_par < 0) return VMS_OK;
  const int par = s->last_par;
  const bool was_pending = s->pending[par];
  if (was_pending) {
    VMS_CUDA(cudaEventSynchronize(s->ev_done[par]));
  }
  std::memcpy(out4, s->counters_h[par], sizeof(uint32_t) * 4);
  return recycle(s, par);
}

}  // extern "C"
